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
#include <cuda.h>  // CUtensorMap (types only; the encoder comes from the runtime entry point)
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

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

#ifdef WW_TRACE
// per-warp event timestamps (globaltimer ns) for tools/trace_kernel.py; not in the product build
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ void trace(int ev) {
    if (g_trace && (threadIdx.x & 31) == 0 && ev < 32) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[((size_t)blockIdx.x * 32 + (threadIdx.x >> 5)) * 32 + ev] = t;
    }
}
#else
__device__ __forceinline__ void trace(int) {}
#endif

struct alignas(64) Params {
    CUtensorMap tmap;     // x as a [B][W][32 floats] tensor, 128B-swizzled boxes (use_tma)
    const uint4* packed;  // COL4 chunks, row-major n x W
    const float* scales;  // n x 4 or 4
    const float* X;       // B x ldx complex64
    float* Y;             // B x ldy complex64
    int64_t n, m, W, ldx, ldy;
    int32_t per_row_scales, conv, tile_chunks, ntiles, aligned16;
    int32_t x_stride;     // chunks per vector in the shared x tile (multiple of 32)
    int32_t use_tma;      // stage x with cp.async.bulk.tensor (else per-thread cp.async)
};

__host__ __device__ constexpr int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// TMA (cp.async.bulk.tensor) load of one 32-chunk x box into shared memory, completing
// `bytes` of transaction on mbarrier `bar`
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
    const int XS = p.x_stride;
    const int span8 = (tc_hi - tc_lo) * 8;
#pragma unroll 1
    for (int b = 0; b < B; ++b) {
        const float* xb = p.X + 2 * (b * p.ldx + (c0 + tc_lo) * 16);
        const int64_t left0 = p.m - (c0 + tc_lo) * 16;  // valid columns from the slice start
        const uint32_t base = xs + (uint32_t)((b * XS + tc_lo) * 128);
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

// Single-tile staging of all of x, sliced for early start: granules (16 B = 2 columns) are
// numbered g = (b*TC + tc)*8 + gg; slice j = 32-chunk sweep j of every vector completes
// mbarrier j.  Each thread issues its granules in slice order and arrives on barrier j once
// all of its slice-<=j copies are issued (cp.async.mbarrier.arrive fires when they land).
template <int B>
__device__ __forceinline__ void stage_x_sliced(const Params& p, uint32_t xs, uint32_t bars,
                                               int J) {
    const int TC = p.tile_chunks, XS = p.x_stride;
    const int per_b = TC * 8;  // granules per vector
    int next = 0;              // next slice barrier to arrive on
    // iterate slice-major so a thread's copies are issued in slice order
    for (int j = 0; j < J; ++j) {
        const int g_lo = 256 * j, g_hi = (256 * j + 256 < per_b ? 256 * j + 256 : per_b);
        const int span = g_hi - g_lo;
        for (int t = threadIdx.x; t < B * span; t += blockDim.x) {
            const int b = B == 1 ? 0 : t / span;
            const int g = g_lo + (B == 1 ? t : t - b * span);
            const int tc = g >> 3, gg = g & 7;
            const int64_t col = (int64_t)tc * 16 + 2 * gg;
            const int64_t valid = p.m - col;
            const float* src = p.X + 2 * (b * p.ldx + col);
            const uint32_t dst = xs + (uint32_t)(((b * XS + tc) * 8 + (gg ^ (tc & 7))) * 16);
            if (p.aligned16) {
                const int bytes = valid >= 2 ? 16 : (valid == 1 ? 8 : 0);
                cp_async16(dst, bytes ? (const void*)src : (const void*)p.X, bytes);
            } else {
                cp_async8(dst, valid >= 1 ? (const void*)src : (const void*)p.X, valid >= 1 ? 8 : 0);
                cp_async8(dst + 8, valid >= 2 ? (const void*)(src + 2) : (const void*)p.X,
                          valid >= 2 ? 8 : 0);
            }
        }
        cp_async_arrive(bars + 8 * next);
        ++next;
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
    const float2 nx = make_float2(-x.x, -x.y);
    // bits in ascending order (bit 2q = -1 of plane q, bit 2q+1 = +1) so the compiler can
    // turn a column's 8 predicates into one R2P of bits 0..6 plus one bit test
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int q = k >> 1;
        if (bits & (1u << k)) {
            if (k & 1) pos[q] = fadd2(pos[q], x);
            else if (N == 2) neg[q] = fadd2(neg[q], x);
            else pos[q] = fadd2(pos[q], nx);
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
// x tile first (1024-B aligned for the 128B-swizzled TMA boxes), then the per-warp reduction
// scratch, then one mbarrier per 32-chunk x slice (single-tile launches)
__host__ __device__ inline SmemLayout smem_layout(int B, int XS, int warps, int ntiles) {
    const int64_t nv = next_pow2(8 * B);
    SmemLayout L;
    L.x_bytes = (int64_t)B * XS * 128;
    L.scratch_off = L.x_bytes;
    L.bar_off = L.scratch_off + (int64_t)warps * nv * 4;
    const int64_t nbars = ntiles == 1 ? XS / 32 : 0;
    L.total = L.bar_off + 8 * nbars + 1024;  // + alignment slack of the dynamic smem base
    return L;
}

// register cap: B == 1 keeps <= 64 registers so two CTAs fit an SM and a PDL-launched next
// layer can start on every SM while this one drains
template <int B>
__host__ __device__ constexpr int min_blocks() { return B == 1 ? 2 : 1; }

template <int B>
__global__ void __launch_bounds__(warps_for<B>() * 32, min_blocks<B>())
wl_gemv_kernel(const __grid_constant__ Params p) {
    constexpr int NV = next_pow2(8 * B);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t xs = (raw + 1023u) & ~1023u;  // 1024-B aligned x tile
    unsigned char* smem = smem_raw + (xs - raw);
    const int TC = p.tile_chunks;
    const int nwarps = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int J = (TC + 31) / 32;  // lane sweeps per tile
    const SmemLayout SL = smem_layout(B, p.x_stride, nwarps, p.ntiles);
    float* sc = reinterpret_cast<float*>(smem + SL.scratch_off) + warp * NV;
    const uint32_t bars = xs + (uint32_t)SL.bar_off;

    // balanced contiguous row range of this CTA (A12 row-parallel decomposition);
    // the host sizes the CTA so its rows split into equal waves over its warps
    const int64_t r0 = (int64_t)blockIdx.x * p.n / gridDim.x;
    const int64_t r1 = (int64_t)(blockIdx.x + 1) * p.n / gridDim.x;
    const bool single = p.ntiles == 1;
    if (single && threadIdx.x == 0) {
        for (int j = 0; j < J; ++j) mbar_init(bars + 8 * j, p.use_tma ? 1u : blockDim.x);
        fence_barrier_init();
    }

    // PDL: let the next kernel launch now and warm L2 with this CTA's weights (never written
    // by other kernels) before waiting for the producer of x / consumer of y.
    trace(0);
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
    const uint32_t bstride = (uint32_t)p.x_stride * 128u;

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
        trace(1);
        pdl_wait();
        trace(2);
        if (p.use_tma) {  // one thread: a 4 KB 128B-swizzled box per slice and vector
            if (threadIdx.x == 0) {
                for (int j = 0; j < J; ++j) {
                    mbar_expect_tx(bars + 8 * j, (uint32_t)(B * 4096));
#pragma unroll 1
                    for (int b = 0; b < B; ++b)
                        tma_load_3d(xs + (uint32_t)((b * p.x_stride + 32 * j) * 128), &p.tmap, 0,
                                    32 * j, b, bars + 8 * j);
                }
            }
        } else {
            stage_x_sliced<B>(p, xs, bars, J);
        }
        trace(3);
        int tr_sweep = 4;
        const uint32_t xlane = xs + (uint32_t)lane * 128u;
        const int64_t total = myrows * J;  // sweeps of this warp
        int64_t row = r0 + warp;
        int j = 0;
        uint32_t xc = xlane;
        bool first = true;  // x slices still to be waited for (first row only)
        auto consume = [&](const uint4& w) {
            if (first) mbar_wait0(bars + 8 * j);
            trace(tr_sweep++);
            if (j < J - 1 || lane < lastw) chunk<B>(acc, w, xc, bstride, off);
            xc += 4096u;
            if (++j == J) {
                reduce_to<B>(acc, sc);
                epilogue<B>(p, sc, row);
                trace(tr_sweep++);
                acc.zero();
                j = 0;
                xc = xlane;
                row += nwarps;
                first = false;
            }
        };
        // unrolled by two with fixed registers: q0 holds even sweeps, q1 odd sweeps
        for (int64_t s = 0; s < total; s += 2) {
            consume(qa);
            qa = load_next();
            if (s + 1 < total) {
                consume(qb);
                qb = load_next();
            }
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
    const int64_t xstride = (tc + 31) / 32 * 32;  // whole 32-chunk sweeps per vector
    const SmemLayout SL = smem_layout(B, (int)xstride, warps, (int)ntiles);
    li->grid = (int32_t)grid;
    li->block = 32 * warps;
    li->tile_chunks = (int32_t)tc;
    li->tiles = (int32_t)ntiles;
    li->smem_bytes = (int32_t)SL.total;
    li->num_sms = sms;
    return WW_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// x viewed as a [B][W][32 floats] tensor (one 128-byte row per 16-column chunk); boxes of
// 32 chunks x 128 B land 128B-swizzled, i.e. granule g of chunk tc at g ^ (tc & 7) -- the
// layout chunk() reads.  Needs 16 | m, a 16-B aligned x and an even ldx (else cp.async).
bool encode_x_map(Params& p, int B) {
    if (p.m % 16 != 0 || ((uintptr_t)p.X & 15) || (B > 1 && (p.ldx % 2) != 0)) return false;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {32, (cuuint64_t)p.W, (cuuint64_t)B};
    const cuuint64_t strides[2] = {128, (cuuint64_t)p.ldx * 8};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p.X), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
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

bool g_force_cp_async = false;  // tests: exercise the per-thread cp.async staging path

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

// Not part of the ABI (no declaration in ww.h): lets the tests force the cp.async staging path.
extern "C" void ww_debug_force_cp_async(int on) { g_force_cp_async = on != 0; }

extern "C" ww_status ww_query_launch(const ww_layer* L, int32_t B, ww_launch_info* out) {
    ww_status st = check_layer(L, "ww_query_launch");
    if (st != WW_OK) return st;
    if (!out) return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_query_launch: null out");
    if (B < 1 || B > WW_MAX_BATCH)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_query_launch: B=%d", B);
    plan(L, B, num_sms(), out);
    return ww::ok();
}

#ifdef WW_TRACE
extern "C" int ww_debug_set_trace(void* dev_ptr) {
    return (int)cudaMemcpyToSymbol(g_trace, &dev_ptr, sizeof(void*));
}
#endif

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
    memset(&p, 0, sizeof p);
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
    p.x_stride = (li.tile_chunks + 31) / 32 * 32;
    p.use_tma = li.tiles == 1 && !g_force_cp_async ? (encode_x_map(p, B) ? 1 : 0) : 0;
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
