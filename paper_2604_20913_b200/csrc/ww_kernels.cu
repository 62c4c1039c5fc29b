// sm_100a kernels of the fused ternary widely-linear GEMV (FairyFuse, arXiv 2604.20913)
// and the device packer, plus their C-ABI launchers (include/ww.h).
//
// Hot path per output row i (Alg. 1, re-designed for B200):
//   * weights: one 16-byte COL4 chunk (16 columns x 4 planes, 2 bits per code) per lane per
//     step, 128-bit coalesced non-allocating loads straight from HBM (a4);
//   * activations: x staged once per CTA in shared memory with cp.async (a3; O2),
//     16-byte granules XOR-swizzled so the 32 lanes (32 different chunks) read conflict-free;
//   * decode (a5; Eqs. 4-5, O1 P:1033): byte k of a chunk holds the 8 code bits of
//     column k; each bit predicates one packed-fp32 add (FADD2) of the pair (x_re, x_im) or
//     its negation into that plane's pair accumulator (Eqs. 6-7), so one decoded
//     code drives both the real and the imaginary path;
//   * accumulate (a6; O4 P:1041): 4 pair accumulators per row and vector in registers,
//     acc_p = (sum_j t_pj x_re,j , sum_j t_pj x_im,j), no multiplies;
//   * reduce (a7): warp transpose-reduce of the 8B partial sums, then
//   * epilogue (a8; P:1002-1011 / P:1435): 8 scale multiplies per row and vector, EQ1 or
//     ALG1 signs, one complex64 store.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "ww.h"
#include "ww_internal.h"

namespace {

// warps per CTA: 16 while the B accumulators leave room, 8 (255-register cap) above
template <int B>
__host__ __device__ constexpr int warps_for() { return B <= 4 ? 16 : 8; }
constexpr int kXBudgetBytes = 184 * 1024;  // x tile per CTA (one CTA per SM)

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }

struct Params {
    const uint4* packed;  // COL4 chunks, row-major n x W
    const float* scales;  // n x 4 or 4
    const float* X;       // B x ldx complex64
    float* Y;             // B x ldy complex64
    int64_t n, m, W, ldx, ldy;
    int32_t per_row_scales, conv, tile_chunks, ntiles, aligned16;
};

__host__ __device__ constexpr int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// mbarrier helpers (one barrier per 32-chunk x slice; completes once per launch, phase 0)
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait0(uint32_t bar) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar)
            : "memory");
    } while (!done);
}

// Issue the cp.async copies of x columns of chunks [c0 + tc_lo, c0 + tc_hi) for all B vectors
// into the swizzled tile: granule g (columns 2g, 2g+1) of tile chunk tc lives at
// ((b*TC + tc)*8 + (g ^ (tc&7)))*16, so 32 lanes reading 32 consecutive chunks hit 32 banks.
// Columns >= m are zero-filled (R6).
template <int B>
__device__ __forceinline__ void stage_x(const Params& p, uint32_t xs, int64_t c0, int tc_lo,
                                        int tc_hi) {
    const int TC = p.tile_chunks;
    const int span8 = (tc_hi - tc_lo) * 8;
#pragma unroll 1
    for (int b = 0; b < B; ++b) {
        const float* xb = p.X + 2 * (b * p.ldx + (c0 + tc_lo) * 16);
        const int64_t left0 = p.m - (c0 + tc_lo) * 16;  // valid columns from the slice start
        const uint32_t base = xs + (uint32_t)((b * TC + tc_lo) * 128);
        for (int g = threadIdx.x; g < span8; g += blockDim.x) {
            const int tcl = g >> 3, gg = g & 7;  // tile chunk (relative), granule
            const int64_t valid = left0 - 2 * g;   // columns left at this granule
            const float* src = xb + 4 * g;
            const uint32_t dst = base + (uint32_t)((tcl * 8 + (gg ^ ((tc_lo + tcl) & 7))) * 16);
            if (p.aligned16) {
                const int bytes = valid >= 2 ? 16 : (valid == 1 ? 8 : 0);
                cp_async16(dst, bytes ? (const void*)src : (const void*)p.X, bytes);
            } else {
                cp_async8(dst, valid >= 1 ? (const void*)src : (const void*)p.X, valid >= 1 ? 8 : 0);
                cp_async8(dst + 8, valid >= 2 ? (const void*)(src + 2) : (const void*)p.X,
                          valid >= 2 ? 8 : 0);
            }
        }
    }
}

// Accumulators: S column-parity sets of B x 4 pair sums.  For B <= 2 even and odd columns
// feed separate sets (more independent FADD2 chains per warp, half-length fp32 chains);
// larger B has ILP across vectors.  N = 2 would keep separate positive / negative sums
// (acc = pos - neg); measured no faster on B200, so N = 1.
template <int B>
struct Acc {
    static constexpr int S = B <= 2 ? 2 : 1;  // column-parity sets
    static constexpr int N = 1;
    float2 a[S][N][B][4];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int k = 0; k < N; ++k)
#pragma unroll
                for (int b = 0; b < B; ++b)
#pragma unroll
                    for (int q = 0; q < 4; ++q) a[s][k][b][q] = make_float2(0.f, 0.f);
    }
    // sum over sets of plane q, vector b: pos - neg
    __device__ __forceinline__ float2 total(int b, int q) const {
        float2 t = a[0][0][b][q];
        if (S == 2) t = fadd2(t, a[S - 1][0][b][q]);
        if (N == 2) {
            float2 n = a[0][N - 1][b][q];
            if (S == 2) n = fadd2(n, a[S - 1][N - 1][b][q]);
            t = fadd2(t, make_float2(-n.x, -n.y));
        }
        return t;
    }
};

// One column (8 code bits = 4 planes) against one activation pair: Eq. 6 (bit 2p+1, add)
// and Eq. 7 (bit 2p, subtract) for each plane p.
template <int N>
__device__ __forceinline__ void column(float2 (&pos)[4], float2 (&neg)[4], uint32_t bits, float2 x) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (bits & (2u << (2 * q))) pos[q] = fadd2(pos[q], x);
        if (N == 2) {
            if (bits & (1u << (2 * q))) neg[q] = fadd2(neg[q], x);
        } else {
            if (bits & (1u << (2 * q))) pos[q] = fadd2(pos[q], make_float2(-x.x, -x.y));
        }
    }
}

// One 16-column chunk of one row (its 16-byte COL4 word w) against the staged x of that
// chunk: 64 codes x B vectors, 2 predicated FADD2 per code and vector.  xc = smem address of
// the chunk's x for vector 0 (vector b at xc + b*bstride); off[kk] = swizzled offset of
// column pair kk ((kk ^ (lane & 7)) * 16: the chunk index's low bits are the lane's).
template <int B>
__device__ __forceinline__ void chunk(Acc<B>& acc, const uint4 w, uint32_t xc, uint32_t bstride,
                                      const uint32_t (&off)[8]) {
    constexpr int S = Acc<B>::S, N = Acc<B>::N;
    const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {  // column pair (2kk, 2kk+1)
        const uint32_t word = w4[kk >> 1];
        const uint32_t sh = (kk & 1) * 16;
        const uint32_t bits_a = (word >> sh) & 0xffu, bits_b = (word >> (sh + 8)) & 0xffu;
#pragma unroll
        for (int b = 0; b < B; ++b) {  // each decoded code drives all B vectors (a9)
            const float4 v = lds128(xc + b * bstride + off[kk]);
            column<N>(acc.a[0][0][b], acc.a[0][N - 1][b], bits_a, make_float2(v.x, v.y));
            column<N>(acc.a[S - 1][0][b], acc.a[S - 1][N - 1][b], bits_b, make_float2(v.z, v.w));
        }
    }
}

// Transpose-reduce NV (power of 2) partial sums across the warp: after the halving rounds
// lane l holds NV>>H totals starting at index (bit4(l) bit3(l) ...)_2 * (NV>>H).
template <int NV>
__device__ __forceinline__ void warp_transpose_reduce(float (&v)[NV]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const int off = 16 >> r;
        const int cur = NV >> r;
        if (cur > 1) {
            const int half = cur / 2;
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int i = 0; i < half; ++i) {
                const float send = up ? v[i] : v[i + half];
                const float keep = up ? v[i + half] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
        }
    }
}

// Warp reduction of this warp's 8B partial sums (a7): writes the NV = next_pow2(8B) totals
// [A0.re A0.im A1.re A1.im A2.re A2.im A3.re A3.im] x B to smem `dst` (only the lanes that
// hold them write).  Ends with __syncwarp.
template <int B>
__device__ __forceinline__ void reduce_to(const Acc<B>& acc, float* dst) {
    const int lane = threadIdx.x & 31;
    constexpr int NV = next_pow2(8 * B);
    float v[NV];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 t = acc.total(b, q);
            v[8 * b + 2 * q] = t.x;
            v[8 * b + 2 * q + 1] = t.y;
        }
#pragma unroll
    for (int i = 8 * B; i < NV; ++i) v[i] = 0.f;
    warp_transpose_reduce<NV>(v);
    constexpr int H = NV >= 32 ? 5 : (NV >= 16 ? 4 : 3);
    constexpr int C = NV >> H;
    int idx = 0;
#pragma unroll
    for (int r = 0; r < H; ++r) idx = (idx << 1) | ((lane >> (4 - r)) & 1);
    if ((lane & ((1 << (5 - H)) - 1)) == 0) {
#pragma unroll
        for (int s = 0; s < C; ++s) dst[idx * C + s] = v[s];
    }
    __syncwarp();
}

// Epilogue (a8): lane b < B applies the row's 8 scales once to the totals T
// of vector b and stores y.
template <int B>
__device__ __forceinline__ void epilogue(const Params& p, const float* T0, int64_t row) {
    const int lane = threadIdx.x & 31;
    if (lane < B) {
        const float* T = T0 + 8 * lane;
        const float* s = p.scales + (p.per_row_scales ? 4 * row : 0);
        const float sUr = s[0], sUi = s[1], sWr = s[2], sWi = s[3];
        const float yre = sUr * T[0] - sUi * T[3] + sWr * T[4] + sWi * T[7];          // Eq. 2
        const float yim = p.conv == WW_CONV_EQ1
                              ? sUr * T[1] + sUi * T[2] - sWr * T[5] + sWi * T[6]   // Eq. 1
                              : sUr * T[1] + sUi * T[2] + sWr * T[5] - sWi * T[6];  // Eq. 3
        reinterpret_cast<float2*>(p.Y)[lane * p.ldy + row] = make_float2(yre, yim);
    }
    __syncwarp();
}

// Shared-memory carve-up (bytes), identical on host (plan) and device.
struct SmemLayout {
    int64_t x_bytes, scratch_off, bar_off, total;
};
__host__ __device__ inline SmemLayout smem_layout(int B, int TC, int warps, int ntiles) {
    const int64_t nv = next_pow2(8 * B);
    SmemLayout L;
    L.x_bytes = (int64_t)B * TC * 128;
    L.scratch_off = L.x_bytes;
    L.bar_off = L.scratch_off + (int64_t)warps * nv * 4;
    const int64_t nbars = ntiles == 1 ? (TC + 31) / 32 : 0;
    L.total = L.bar_off + 8 * nbars;
    return L;
}

// register cap: B == 1 keeps <= 64 registers so two CTAs fit an SM and a PDL-launched next
// layer can start on every SM while this one drains
template <int B>
__host__ __device__ constexpr int min_blocks() { return B == 1 ? 2 : 1; }

template <int B>
__global__ void __launch_bounds__(warps_for<B>() * 32, min_blocks<B>())
wl_gemv_kernel(const Params p) {
    constexpr int NV = next_pow2(8 * B);
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t xs = (uint32_t)__cvta_generic_to_shared(smem);
    const int TC = p.tile_chunks;
    const int nwarps = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int J = (TC + 31) / 32;  // lane sweeps per tile
    const SmemLayout SL = smem_layout(B, TC, nwarps, p.ntiles);
    float* sc = reinterpret_cast<float*>(smem + SL.scratch_off) + warp * NV;
    const uint32_t bars = xs + (uint32_t)SL.bar_off;

    // balanced contiguous row range of this CTA (A12 row-parallel decomposition);
    // the host sizes the CTA so its rows split into equal waves over its warps
    const int64_t r0 = (int64_t)blockIdx.x * p.n / gridDim.x;
    const int64_t r1 = (int64_t)(blockIdx.x + 1) * p.n / gridDim.x;
    const bool single = p.ntiles == 1;
    if (single && threadIdx.x == 0)
        for (int j = 0; j < J; ++j) mbar_init(bars + 8 * j, blockDim.x);

    // PDL: let the next kernel launch now and warm L2 with this CTA's weights (never written
    // by other kernels) before waiting for the producer of x / consumer of y.
    pdl_launch_dependents();
    if (threadIdx.x == 0) {
        const char* wb = reinterpret_cast<const char*>(p.packed + r0 * p.W);
        const int64_t bytes = (r1 - r0) * p.W * 16;
        for (int64_t off = 0; off < bytes; off += 65536)
            prefetch_l2(wb + off, (uint32_t)(bytes - off < 65536 ? bytes - off : 65536));
    }
    Acc<B> acc;
    acc.zero();

    uint32_t off[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) off[kk] = (uint32_t)((kk ^ (lane & 7)) << 4);
    const uint32_t bstride = (uint32_t)TC * 128u;

    if (single) {
        // This warp's rows r0 + warp + k*nwarps, each swept in J steps of 32 chunks (lane =
        // chunk within the step; the last step has `lastw` active lanes).  The weights stream
        // two steps ahead in registers across row boundaries; all loop state is incremental.
        const int lastw = TC - 32 * (J - 1);
        const int64_t myrows = r0 + warp < r1 ? (r1 - r0 - warp + nwarps - 1) / nwarps : 0;
        const uint4* pf = p.packed + (r0 + warp) * p.W + lane;  // prefetch pointer
        const int64_t row_jump = (int64_t)nwarps * p.W - 32 * J;
        int64_t pf_rows = myrows;
        int pf_j = 0;
        auto load_next = [&]() -> uint4 {
            uint4 w = make_uint4(0, 0, 0, 0);
            if (pf_rows > 0 && (pf_j < J - 1 || lane < lastw)) w = ldg_stream(pf);
            pf += 32;
            if (++pf_j == J) {
                pf_j = 0;
                pf += row_jump;
                --pf_rows;
            }
            return w;
        };
        uint4 qa = load_next(), qb = load_next();
        __syncthreads();  // mbarrier inits visible
        pdl_wait();
        for (int j = 0; j < J; ++j) {  // x in 32-chunk slices, each completing its mbarrier
            stage_x<B>(p, xs, 0, 32 * j, 32 * j + 32 < TC ? 32 * j + 32 : TC);
            cp_async_arrive(bars + 8 * j);
        }
        const uint32_t xlane = xs + (uint32_t)lane * 128u;
        int64_t row = r0 + warp;
        for (int64_t k = 0; k < myrows; ++k, row += nwarps) {
            uint32_t xc = xlane;
            for (int j = 0; j < J; ++j, xc += 4096u) {
                const uint4 cur = qa;
                qa = qb;
                qb = load_next();
                if (k == 0) mbar_wait0(bars + 8 * j);
                if (j < J - 1 || lane < lastw) chunk<B>(acc, cur, xc, bstride, off);
            }
            reduce_to<B>(acc, sc);
            epilogue<B>(p, sc, row);
            acc.zero();
        }
        return;
    }

    // x does not fit one tile: row waves, each streaming the tiles with CTA-wide syncs
    pdl_wait();
    for (int64_t wr = r0; wr < r1; wr += nwarps) {  // uniform across the CTA
        const int64_t row = wr + warp;
        const bool active = row < r1;
        for (int t = 0; t < p.ntiles; ++t) {
            const int64_t c0 = (int64_t)t * TC;
            const int tc_n = (int)(p.W - c0 < TC ? p.W - c0 : TC);
            __syncthreads();  // previous tile fully consumed
            stage_x<B>(p, xs, c0, 0, tc_n);
            cp_async_wait_all();
            __syncthreads();
            if (active) {
                const uint4* wrow = p.packed + row * p.W + c0;
                int tc = lane;
                uint4 cur = tc < tc_n ? ldg_stream(wrow + tc) : make_uint4(0, 0, 0, 0);
                for (; tc < tc_n; tc += 32) {
                    const uint4 nxt =
                        tc + 32 < tc_n ? ldg_stream(wrow + tc + 32) : make_uint4(0, 0, 0, 0);
                    chunk<B>(acc, cur, xs + (uint32_t)tc * 128u, bstride, off);
                    cur = nxt;
                }
            }
        }
        if (active) {
            reduce_to<B>(acc, sc);
            epilogue<B>(p, sc, row);
            acc.zero();
        }
    }
}

// ------------------------------------------------------------------ device packer
// One thread per output word: columns 16c + 4q .. +3 of row i, all four planes.
__global__ void pack_col4_kernel(const int8_t* __restrict__ planes, int64_t n, int64_t m,
                                 int64_t ld, int64_t W, uint32_t* __restrict__ out,
                                 int32_t* bad) {
    const int64_t total = n * W * 4;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / (W * 4);
        const int64_t rem = e - i * W * 4;
        const int64_t c = rem >> 2;
        const int q = (int)(rem & 3);
        uint32_t word = 0;
        bool badv = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t j = 16 * c + 4 * q + k;
            if (j >= m) continue;
            uint32_t byte = 0;
#pragma unroll
            for (int pl = 0; pl < 4; ++pl) {
                const int8_t t = planes[(int64_t)pl * n * ld + i * ld + j];
                if (t == 1) byte |= 2u << (2 * pl);
                else if (t == -1) byte |= 1u << (2 * pl);
                else if (t != 0) badv = true;
            }
            if (!badv) word |= byte << (8 * k);
        }
        out[e] = word;
        if (badv && bad) atomicOr(bad, 1);
    }
}

// ------------------------------------------------------------------ launch configuration
int num_sms() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            cached <= 0)
            cached = 148;  // B200
    }
    return cached;
}

ww_status plan(const ww_layer* L, int32_t B, int sms, ww_launch_info* li) {
    const int64_t W = ww::words_per_row(L->m);
    const int64_t per_chunk = (int64_t)B * 128;  // x bytes per chunk for B vectors
    int64_t tc = kXBudgetBytes / per_chunk;
    if (tc >= W) {
        tc = W;
    } else {
        tc = std::max<int64_t>(32, tc / 32 * 32);  // whole lane sweeps per tile
    }
    const int64_t ntiles = (W + tc - 1) / tc;
    // one CTA per SM (persistent); a CTA's rows split into equal waves over its warps
    const int64_t grid = std::min<int64_t>(sms, L->n);
    const int max_warps = B <= 4 ? 16 : 8;
    const int64_t rows_cta = (L->n + grid - 1) / grid;
    const int64_t waves = (rows_cta + max_warps - 1) / max_warps;
    const int warps = (int)((rows_cta + waves - 1) / waves);
    const SmemLayout SL = smem_layout(B, (int)tc, warps, (int)ntiles);
    li->grid = (int32_t)grid;
    li->block = 32 * warps;
    li->tile_chunks = (int32_t)tc;
    li->tiles = (int32_t)ntiles;
    li->smem_bytes = (int32_t)SL.total;
    li->num_sms = sms;
    return WW_OK;
}

template <int B>
cudaError_t launch_b(const Params& p, const ww_launch_info& li, cudaStream_t s, bool pdl) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(wl_gemv_kernel<B>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)li.grid);
    cfg.blockDim = dim3((unsigned)li.block);
    cfg.dynamicSmemBytes = (size_t)li.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, wl_gemv_kernel<B>, p);
}

cudaError_t launch(const Params& p, const ww_launch_info& li, int B, cudaStream_t s, bool pdl) {
    switch (B) {
#define WW_CASE(b) \
    case b: return launch_b<b>(p, li, s, pdl);
        WW_CASE(1) WW_CASE(2) WW_CASE(3) WW_CASE(4) WW_CASE(5) WW_CASE(6) WW_CASE(7) WW_CASE(8)
        WW_CASE(9) WW_CASE(10) WW_CASE(11) WW_CASE(12) WW_CASE(13) WW_CASE(14) WW_CASE(15)
        WW_CASE(16)
#undef WW_CASE
    }
    return cudaErrorInvalidValue;
}

ww_status check_layer(const ww_layer* L, const char* fn) {
    if (!L) return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: null layer", fn);
    if (L->n < 1 || L->m < 1)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: n=%lld m=%lld", fn, (long long)L->n,
                        (long long)L->m);
    if (L->layout != WW_LAYOUT_COL4)
        return ww::fail(WW_ERR_UNSUPPORTED, "%s: GPU kernels take WW_LAYOUT_COL4 (got %d)", fn,
                        L->layout);
    if (L->scale_mode != WW_SCALES_PER_ROW && L->scale_mode != WW_SCALES_PER_TENSOR)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: scale_mode %d", fn, L->scale_mode);
    if (L->conv != WW_CONV_EQ1 && L->conv != WW_CONV_ALG1)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: conv %d", fn, L->conv);
    if (L->n > (int64_t)1 << 40 || L->m > (int64_t)1 << 36)
        return ww::fail(WW_ERR_UNSUPPORTED, "%s: shape too large", fn);
    return WW_OK;
}

}  // namespace

extern "C" ww_status ww_query_launch(const ww_layer* L, int32_t B, ww_launch_info* out) {
    ww_status st = check_layer(L, "ww_query_launch");
    if (st != WW_OK) return st;
    if (!out) return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_query_launch: null out");
    if (B < 1 || B > WW_MAX_BATCH)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_query_launch: B=%d", B);
    plan(L, B, num_sms(), out);
    return ww::ok();
}

extern "C" ww_status ww_wl_gemv_batched(const ww_layer* L, const void* packed_d,
                                        const float* scales_d, const float* X_d, int64_t ldx,
                                        float* Y_d, int64_t ldy, int32_t B, void* stream) {
    ww_status st = check_layer(L, "ww_wl_gemv");
    if (st != WW_OK) return st;
    if (!packed_d || !scales_d || !X_d || !Y_d)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_gemv: null pointer");
    if (B < 1) return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_gemv: B=%d", B);
    if (B > WW_MAX_BATCH)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_wl_gemv: B=%d > %d", B, WW_MAX_BATCH);
    if (ldx < L->m || ldy < L->n)
        return ww::fail(WW_ERR_DIMENSION_MISMATCH, "ww_wl_gemv: ldx=%lld (m=%lld) ldy=%lld (n=%lld)",
                        (long long)ldx, (long long)L->m, (long long)ldy, (long long)L->n);
    if (((uintptr_t)packed_d & 15) || ((uintptr_t)X_d & 7) || ((uintptr_t)Y_d & 7) ||
        ((uintptr_t)scales_d & 3))
        return ww::fail(WW_ERR_MISALIGNED, "ww_wl_gemv: packed must be 16-B, x/y 8-B aligned");
    const char* xb = reinterpret_cast<const char*>(X_d);
    const char* yb = reinterpret_cast<const char*>(Y_d);
    if (xb < yb + 8 * (ldy * (B - 1) + L->n) && yb < xb + 8 * (ldx * (B - 1) + L->m))
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_gemv: x and y overlap");
    ww_launch_info li;
    plan(L, B, num_sms(), &li);
    Params p;
    p.packed = reinterpret_cast<const uint4*>(packed_d);
    p.scales = scales_d;
    p.X = X_d;
    p.Y = Y_d;
    p.n = L->n;
    p.m = L->m;
    p.W = ww::words_per_row(L->m);
    p.ldx = ldx;
    p.ldy = ldy;
    p.per_row_scales = L->scale_mode == WW_SCALES_PER_ROW;
    p.conv = L->conv;
    p.tile_chunks = li.tile_chunks;
    p.ntiles = li.tiles;

    p.aligned16 = (((uintptr_t)X_d & 15) == 0) && (ldx % 2 == 0);
    cudaError_t e = launch(p, li, B, (cudaStream_t)stream, (L->flags & WW_FLAG_PDL) != 0);
    if (e != cudaSuccess)
        return ww::fail(WW_ERR_CUDA, "ww_wl_gemv: launch failed: %s", cudaGetErrorString(e));
    return ww::ok();
}

extern "C" ww_status ww_wl_gemv(const ww_layer* L, const void* packed_d, const float* scales_d,
                                const float* x_d, float* y_d, void* stream) {
    if (!L) return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_gemv: null layer");
    return ww_wl_gemv_batched(L, packed_d, scales_d, x_d, L->m, y_d, L->n, 1, stream);
}

extern "C" ww_status ww_pack_ternary_device(const int8_t* planes_d, int64_t n, int64_t m,
                                            int64_t ld, uint32_t* out_d, int32_t* bad_d,
                                            void* stream) {
    if (!planes_d || !out_d)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_pack_ternary_device: null pointer");
    if (n < 1 || m < 1 || ld < m)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_pack_ternary_device: n=%lld m=%lld ld=%lld",
                        (long long)n, (long long)m, (long long)ld);
    if ((uintptr_t)out_d & 15)
        return ww::fail(WW_ERR_MISALIGNED, "ww_pack_ternary_device: out must be 16-B aligned");
    const int64_t W = ww::words_per_row(m);
    pack_col4_kernel<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(planes_d, n, m, ld, W,
                                                                      out_d, bad_d);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return ww::fail(WW_ERR_CUDA, "ww_pack_ternary_device: %s", cudaGetErrorString(e));
    return ww::ok();
}
