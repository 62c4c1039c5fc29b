// wl_lut_kernel: B = 1 WL-GEMV by ternary subset-sum lookup (ww_wl_gemv_lut, WW_LAYOUT_LUT81).
//
// The eight real sub-GEMVs of Eq. 1 (Eqs. 6-7) are still sums of
// +x, -x and nothing; here the sum over each group of 4 columns is read from a
// table instead of being accumulated code by code.  For every 4 columns the CTA builds, with
// adds and subtracts only, the 81 values sum_k c_k (x_re, x_im)_k, c in {-1,0,+1}^4, in
// shared memory; a weight byte is the index of its 4 codes of one plane (a bijection of the
// App. H bit pairs, ww.h "WW_LAYOUT_LUT81"), so 4 codes cost one PRMT, one LDS.64 and one
// FADD2 instead of 8 predicated FADD2 -- the predicated datapath's 32 codes/clk/SM ceiling
// becomes the shared-memory ceiling of 64 codes/clk/SM.
//
// Table layout: a block = 128 columns = 32 groups, one per lane; entry e of lane l's group
// at block + e * 256 + l * 8, so a warp's LDS.64 is conflict-free whatever the 32 indices
// are (each half-warp covers the 32 banks once).  81 * 256 B = 20,736 B per block; a CTA
// holds 8 blocks (1024 columns), so a row's columns are split over the S = ceil(T / 2) CTAs
// of a thread-block cluster (T = ceil(m / 512) steps of 512 columns) and the per-row partial
// totals meet through distributed shared memory, summed in rank order (deterministic).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "ww_internal.h"

namespace cg = cooperative_groups;

namespace {

#ifdef WW_LUT_WARPS32  // experiment: 32 warps of 64 registers, ring of 4
constexpr int kWarps = 32;
#else
constexpr int kWarps = 16;
#endif
constexpr int kThreads = kWarps * 32;
constexpr int kBlockBytes = 81 * 256;   // one 128-column table block
constexpr int kStepBytes = 4 * kBlockBytes;
constexpr int kMaxStepsPerCta = 2;      // 8 blocks = 165,888 B of tables
constexpr int kMaxRowsPerCluster = 1536;  // 48 KB of partial totals
constexpr int kMaxCluster = 8;
// tables start at a 64 KB boundary: with the window's first 1 KB reserved, 63 KB in front of them
constexpr int kDynSmem = 0x10000 + kMaxStepsPerCta * kStepBytes;  // 231,424 B: any window offset >= 0

struct LutParams {
    const uint4* Wp;      // [n][T][32] uint4
    const float* scales;  // n x 4 or 4
    const float2* X;      // m complex64
    float2* Y;            // n complex64
    int64_t n, m;
    int T, S;             // steps per row, cluster size
    int per_row, conv, pdl;
};

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void sts64(uint32_t a, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

// the 9 values (d0 - 1) a + (d1 - 1) b, index d0 + 3 d1 (adds and subtracts only)
__device__ __forceinline__ void pair9(float2 a, float2 b, float2 (&t)[9]) {
    const float2 s = add2(a, b), d = add2(a, neg2(b));
    t[0] = neg2(s); t[1] = neg2(b); t[2] = d;
    t[3] = neg2(a); t[4] = make_float2(0.f, 0.f); t[5] = a;
    t[6] = neg2(d); t[7] = b; t[8] = s;
}

// one plane word = 4 bytes = the lane's group in 4 consecutive blocks
// base = table address (a multiple of 64 KB) + lane * 8: byte 1 of the address is the index
template <int OFF>
__device__ __forceinline__ void lookup(float2& acc, uint32_t w, uint32_t base, int k) {
    const uint32_t a = __byte_perm(w, base, 0x7604 | (k << 4));  // byte k of w -> bits 8..15
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0,%1}, [%2+%3];" : "=f"(v.x), "=f"(v.y) : "r"(a), "n"(OFF));
    acc = add2(acc, v);
}
// one plane word = 4 bytes = the lane's group in 4 consecutive blocks of step STEP of the CTA
template <int STEP>
__device__ __forceinline__ void plane4(float2& acc, uint32_t w, uint32_t base) {
    lookup<STEP * kStepBytes + 0 * kBlockBytes>(acc, w, base, 0);
    lookup<STEP * kStepBytes + 1 * kBlockBytes>(acc, w, base, 1);
    lookup<STEP * kStepBytes + 2 * kBlockBytes>(acc, w, base, 2);
    lookup<STEP * kStepBytes + 3 * kBlockBytes>(acc, w, base, 3);
}

// totals over the 32 lanes of the 8 values in a[4] (x = re, y = im of plane p): value v ends
// up on lanes with (lane >> 2) & 7 == v ... reduced by halving the value set 8 -> 4 -> 2 -> 1
// (9 shuffles); returns the total of value index ((lane >> 2) & 7), the same on 4 lanes.
__device__ __forceinline__ float reduce8(const float2 (&a)[4], int lane) {
    float v[8] = {a[0].x, a[0].y, a[1].x, a[1].y, a[2].x, a[2].y, a[3].x, a[3].y};
    float u[4];
    const bool h4 = lane & 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // keep values 4*h4 .. 4*h4+3
        const float send = h4 ? v[i] : v[i + 4];
        const float keep = h4 ? v[i + 4] : v[i];
        u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float t[2];
    const bool h3 = lane & 8;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = h3 ? u[i] : u[i + 2];
        const float keep = h3 ? u[i + 2] : u[i];
        t[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const bool h2 = lane & 4;
    const float send = h2 ? t[0] : t[1];
    const float keep = h2 ? t[1] : t[0];
    float r = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;  // value index 4*h4 + 2*h3 + h2 = (lane >> 2) & 7 with bits reversed: see caller
}

constexpr int kRing = kWarps == 32 ? 4 : 8;  // 128-bit weight loads in flight per lane

// item q of a warp = (row q / nsteps, step q % nsteps) of its rows
__device__ __forceinline__ uint4 load_item(const uint4* wp, int64_t stride, int q, int nsteps) {
    const int row = nsteps == 2 ? q >> 1 : q, s = nsteps == 2 ? q & 1 : 0;
    return ldg_stream(wp + (int64_t)row * stride + s * 32);
}

// predicated 128-bit streaming load: v keeps its value when !pred
__device__ __forceinline__ void ldg_stream_if(uint4& v, const uint4* p, bool pred) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
        : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
        : "l"(p), "r"((uint32_t)pred));
}

// slot J of the ring holds item q + J = (row (q + J) / NSTEPS, step (q + J) % NSTEPS); its
// lookups, the refill with item q + J + kRing from `next` (when LOAD), and the row's end
template <int NSTEPS, int J, bool LOAD>
__device__ __forceinline__ void ring_item(const uint4* next, int64_t stride, int q, int Q, uint32_t base,
                                          float* part, int lane, int vi, uint4 (&buf)[kRing],
                                          float2 (&acc)[4]) {
    const uint4 w = buf[J];
    if (LOAD)
        ldg_stream_if(buf[J], next + (int64_t)(J / NSTEPS) * stride + (J % NSTEPS) * 32,
                      q + J + kRing < Q);
    constexpr int kStep = NSTEPS == 2 ? (J & 1) : 0;
    plane4<kStep>(acc[0], w.x, base);
    plane4<kStep>(acc[1], w.y, base);
    plane4<kStep>(acc[2], w.z, base);
    plane4<kStep>(acc[3], w.w, base);
    if (NSTEPS == 1 || (J & 1)) {  // the row's last step
        const float r = reduce8(acc, lane);
        if ((lane & 3) == 0) part[(q + J) / NSTEPS * 8 + vi] = r;
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
    }
}

#define WW_RING_ITEM(J, LOAD, GUARD) \
    if (J < kRing && (!(GUARD) || q + J < Q)) \
        ring_item<NSTEPS, (J < kRing ? J : 0), LOAD>(wq, stride, q, Q, base, part, lane, vi, buf, acc);
#define WW_RING_ITEMS(LOAD, GUARD)                                                       \
    WW_RING_ITEM(0, LOAD, GUARD) WW_RING_ITEM(1, LOAD, GUARD) WW_RING_ITEM(2, LOAD, GUARD) \
    WW_RING_ITEM(3, LOAD, GUARD) WW_RING_ITEM(4, LOAD, GUARD) WW_RING_ITEM(5, LOAD, GUARD) \
    WW_RING_ITEM(6, LOAD, GUARD) WW_RING_ITEM(7, LOAD, GUARD)

template <int NSTEPS>
__device__ __forceinline__ void sweep_rows(const uint4* wp, int64_t stride, int nrows, uint32_t tab,
                                           float* part, int lane, uint4 (&buf)[kRing]) {
    static_assert(kRing <= 8 && kRing % 2 == 0, "WW_RING_ITEMS");
    const int Q = nrows * NSTEPS;
    float2 acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
    const uint32_t base = tab + lane * 8;
    // value index held by this lane after reduce8
    const int vi = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    const int64_t adv = (int64_t)(kRing / NSTEPS) * stride;  // one ring of items further
    const uint4* wq = wp;
    int q = 0;
    for (; q + kRing <= Q; q += kRing) {  // full rings: no guards around the lookups
        wq += adv;
        WW_RING_ITEMS(true, false)
    }
    WW_RING_ITEMS(false, true)  // the tail: items already in the ring
}
#undef WW_RING_ITEMS
#undef WW_RING_ITEM

__global__ void __launch_bounds__(kThreads, 1) wl_lut_kernel(const LutParams p) {
    extern __shared__ __align__(1024) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int S = p.S;
    const int rank = (int)cluster.block_rank();
    const int cid = blockIdx.x / S, C = gridDim.x / S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // rows of this cluster (balanced contiguous ranges), then of this warp
    const int64_t rb = p.n / C, rr = p.n % C;
    const int64_t r0 = cid * rb + min((int64_t)cid, rr);
    const int NR = (int)(rb + (cid < rr ? 1 : 0));
    const int wb = NR / kWarps, wr = NR % kWarps;
    const int w0 = warp * wb + min(warp, wr);
    const int nrows = wb + (warp < wr ? 1 : 0);

    // this CTA's steps [t0, t0 + nsteps)
    const int Tc = (p.T + S - 1) / S;
    const int t0 = rank * Tc;
    const int nsteps = max(0, min(Tc, p.T - t0));

    float* part = reinterpret_cast<float*>(smem);  // [NR][8] partial totals of this CTA
    // tables at the first 64 KB boundary of the shared window past the partial totals (bits
    // 8..15 of a lookup address are then the index alone); in a cluster the CTA's window
    // does not start near 0, only its offset within 64 KB matters
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t tab = (sbase + kMaxRowsPerCluster * 32 + 0xFFFFu) & ~0xFFFFu;
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (tab + kMaxStepsPerCta * kStepBytes > sbase + dyn) __trap();

    // the weights never depend on the previous kernel: the first loads go out before the wait
    const uint4* wp = p.Wp + ((r0 + w0) * p.T + t0) * 32 + lane;
    const int64_t stride = (int64_t)p.T * 32;
    uint4 buf[kRing];
#pragma unroll
    for (int j = 0; j < kRing; ++j)
        if (j < nrows * nsteps) buf[j] = load_item(wp, stride, j, nsteps);
    if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- build the tables: warp -> (block, share of the 9 second-pair values), lane = group
    const int nb = nsteps * 4;
    if (nb > 0) {
        const int parts = kWarps / nb;  // 2 (8 blocks) or 4 (4 blocks)
        const int b = warp % nb, part_i = warp / nb;
        if (part_i < parts) {
            const int64_t col = (int64_t)(t0 + b / 4) * 512 + (b & 3) * 128 + lane * 4;
            float2 x[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                x[k] = col + k < p.m ? __ldg(p.X + col + k) : make_float2(0.f, 0.f);
            float2 lo[9], hi[9];
            pair9(x[0], x[1], lo);
            pair9(x[2], x[3], hi);
            const int j0 = part_i * 9 / parts, j1 = (part_i + 1) * 9 / parts;
            const uint32_t dst = tab + b * kBlockBytes + lane * 8;
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                if (j >= j0 && j < j1) {
#pragma unroll
                    for (int i = 0; i < 9; ++i)
                        sts64(dst + (uint32_t)(9 * j + i) * 256, add2(lo[i], hi[j]));
                }
            }
        }
    }
    __syncthreads();

    // ---- sweep this warp's rows over this CTA's columns
    if (nsteps == 2)
        sweep_rows<2>(wp, stride, nrows, tab, part + w0 * 8, lane, buf);
    else if (nsteps == 1)
        sweep_rows<1>(wp, stride, nrows, tab, part + w0 * 8, lane, buf);
    else
        for (int i = lane; i < nrows * 8; i += 32) part[w0 * 8 + i] = 0.f;

    cluster.sync();

    // ---- rows r with r % S == rank: partial totals of all ranks in rank order, epilogue
    for (int r = rank + S * (int)threadIdx.x; r < NR; r += S * kThreads) {
        float T8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) T8[i] = 0.f;
        for (int c = 0; c < S; ++c) {
            const float4* src =
                reinterpret_cast<const float4*>(cluster.map_shared_rank(part, c) + r * 8);
            const float4 a = src[0], bq = src[1];
            T8[0] += a.x; T8[1] += a.y; T8[2] += a.z; T8[3] += a.w;
            T8[4] += bq.x; T8[5] += bq.y; T8[6] += bq.z; T8[7] += bq.w;
        }
        const int64_t row = r0 + r;
        const float* s = p.scales + (p.per_row ? 4 * row : 0);
        // the row's 8 scale multiplies, once after accumulation
        const float sUr = s[0], sUi = s[1], sWr = s[2], sWi = s[3];
        const float yre = sUr * T8[0] - sUi * T8[3] + sWr * T8[4] + sWi * T8[7];  // Eq. 2
        const float yim = p.conv == WW_CONV_EQ1
                              ? sUr * T8[1] + sUi * T8[2] - sWr * T8[5] + sWi * T8[6]   // Eq. 1
                              : sUr * T8[1] + sUi * T8[2] + sWr * T8[5] - sWi * T8[6];  // Eq. 3
        p.Y[row] = make_float2(yre, yim);
    }
    cluster.sync();  // partial totals stay mapped until every rank has read them
}

inline int lut_steps(int64_t m) { return (int)((m + 511) / 512); }

// device packer: one thread per output word = (row i, step t, lane l, plane p), 4 blocks k.
// A value outside {-1,0,+1} packs as the zero code and sets *bad (as the COL4 packer, ww.h).
__global__ void pack_lut81_kernel(const int8_t* __restrict__ planes, int64_t n, int64_t m, int64_t ld,
                                  int T, int64_t total, uint32_t* __restrict__ out, int32_t* bad) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)(w & 3), l = (int)((w >> 2) & 31);
        const int64_t it = w >> 7, i = it / T, t = it % T;
        const int8_t* row = planes + ((int64_t)p * n + i) * ld;
        uint32_t word = 0;
        bool any_bad = false;
        for (int k = 0; k < 4; ++k) {
            const int64_t col = t * 512 + k * 128 + l * 4;
            int idx = 0, pw = 1;
            for (int c = 0; c < 4; ++c, pw *= 3) {
                int v = col + c < m ? (int)row[col + c] : 0;
                if (v < -1 || v > 1) {
                    any_bad = true;
                    v = 0;
                }
                idx += pw * (v + 1);
            }
            word |= (uint32_t)idx << (8 * k);
        }
        out[w] = word;
        if (any_bad && bad) atomicOr(bad, 1);
    }
}

std::mutex g_lut_mu;
int g_resident[64][kMaxCluster + 1] = {};  // resident clusters per (device, cluster size); 0 = not queried

}  // namespace

extern "C" size_t ww_lut81_packed_bytes(int64_t n, int64_t m) {
    if (n < 0 || m < 0) return 0;
    return (size_t)n * (size_t)lut_steps(m) * 512u;
}

// byte of (row i, plane p, column group g = j / 4): step t = j / 512, block k = (j % 512) / 128,
// lane l = (j % 128) / 4  ->  byte 16 * ((i T + t) 32 + l) + 4 p + k
static inline size_t lut_byte(int64_t i, int T, int p, int64_t j) {
    const int64_t t = j / 512, k = (j % 512) / 128, l = (j % 128) / 4;
    return (size_t)(((i * T + t) * 32 + l) * 16 + 4 * p + k);
}

extern "C" ww_status ww_lut81_from_planar(int64_t n, int64_t m, const void* planar, void* out) {
    if (!planar || !out || n < 1 || m < 1)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_lut81_from_planar: bad argument");
    const int64_t W = ww::words_per_row(m);
    const int T = lut_steps(m);
    const uint32_t* src = static_cast<const uint32_t*>(planar);
    uint8_t* dst = static_cast<uint8_t*>(out);
    for (int p = 0; p < 4; ++p)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t g = 0; g < (int64_t)T * 128; ++g) {
                int idx = 0, pw = 1;
                for (int k = 0; k < 4; ++k, pw *= 3) {
                    const int64_t j = 4 * g + k;
                    uint32_t c = 0;
                    if (j < 16 * W) c = (src[(p * n + i) * W + j / 16] >> (2 * (j % 16))) & 3u;
                    if (c == 3u)
                        return ww::fail(WW_ERR_INVALID_ENCODING,
                                        "ww_lut81_from_planar: (1,1) at plane %d row %lld col %lld", p,
                                        (long long)i, (long long)j);
                    idx += pw * (c == 2u ? 2 : c == 1u ? 0 : 1);  // digit = code + 1
                }
                dst[lut_byte(i, T, p, 4 * g)] = (uint8_t)idx;
            }
    return ww::ok();
}

extern "C" ww_status ww_lut81_to_planar(int64_t n, int64_t m, const void* lut, void* planar_out) {
    if (!lut || !planar_out || n < 1 || m < 1)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_lut81_to_planar: bad argument");
    const int64_t W = ww::words_per_row(m);
    const int T = lut_steps(m);
    const uint8_t* src = static_cast<const uint8_t*>(lut);
    uint32_t* dst = static_cast<uint32_t*>(planar_out);
    std::memset(dst, 0, (size_t)4 * n * W * 4);
    for (int p = 0; p < 4; ++p)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t g = 0; g < (int64_t)T * 128; ++g) {
                int idx = src[lut_byte(i, T, p, 4 * g)];
                if (idx > 80)
                    return ww::fail(WW_ERR_INVALID_ENCODING,
                                    "ww_lut81_to_planar: byte %d > 80 at plane %d row %lld group %lld",
                                    idx, p, (long long)i, (long long)g);
                for (int k = 0; k < 4; ++k, idx /= 3) {
                    const int64_t j = 4 * g + k;
                    const int d = idx % 3;  // code + 1
                    if (j >= 16 * W) {
                        if (d != 1)
                            return ww::fail(WW_ERR_INVALID_ENCODING,
                                            "ww_lut81_to_planar: nonzero padding code");
                        continue;
                    }
                    const uint32_t c = d == 2 ? 2u : d == 0 ? 1u : 0u;
                    dst[(p * n + i) * W + j / 16] |= c << (2 * (j % 16));
                }
            }
    return ww::ok();
}

extern "C" ww_status ww_wl_gemv_lut(const ww_layer* L, const void* packed_d, const float* scales_d,
                                    const float* x_d, float* y_d, void* stream) {
    if (!L || !packed_d || !scales_d || !x_d || !y_d)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_gemv_lut: null pointer");
    if (L->n < 1 || L->m < 1 || L->n > ((int64_t)1 << 30))
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_gemv_lut: n=%lld m=%lld", (long long)L->n,
                        (long long)L->m);
    if ((L->conv != WW_CONV_EQ1 && L->conv != WW_CONV_ALG1) ||
        (L->scale_mode != WW_SCALES_PER_ROW && L->scale_mode != WW_SCALES_PER_TENSOR))
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_gemv_lut: conv=%d scale_mode=%d", (int)L->conv,
                        (int)L->scale_mode);
    if (L->layout != WW_LAYOUT_LUT81)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_wl_gemv_lut: layout %d is not WW_LAYOUT_LUT81",
                        (int)L->layout);
    if (((uintptr_t)packed_d & 15) || ((uintptr_t)x_d & 7) || ((uintptr_t)y_d & 7) ||
        ((uintptr_t)scales_d & 3))
        return ww::fail(WW_ERR_MISALIGNED, "ww_wl_gemv_lut: misaligned pointer");
    const int T = lut_steps(L->m);
    const int S = (T + kMaxStepsPerCta - 1) / kMaxStepsPerCta;
    if (S > kMaxCluster)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_wl_gemv_lut: m=%lld needs a cluster of %d CTAs (max %d)",
                        (long long)L->m, S, kMaxCluster);
    const int sms = ww::device_sms();
    const size_t smem = kDynSmem;
    const int e = ww::prepare_kernel(reinterpret_cast<const void*>(wl_lut_kernel), kDynSmem);
    if (e)
        return ww::fail(WW_ERR_CUDA, "ww_wl_gemv_lut: %s", cudaGetErrorString((cudaError_t)e));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms / S * S);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // one wave: no more clusters than can be resident at once (GPC boundaries)
    int resident;
    {
        const int dev = ww::current_device();
        std::lock_guard<std::mutex> lk(g_lut_mu);
        int& slot = g_resident[dev >= 0 && dev < 64 ? dev : 0][S];
        if (slot == 0) {
            int r = 0;
            if (cudaOccupancyMaxActiveClusters(&r, wl_lut_kernel, &cfg) != cudaSuccess || r < 1) {
                cudaGetLastError();
                r = std::max(1, sms / S);
            }
            slot = r;
        }
        resident = slot;
    }
    const int C = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(sms / S, resident), L->n));
    if ((L->n + C - 1) / C > kMaxRowsPerCluster)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_wl_gemv_lut: n=%lld exceeds %d rows per cluster",
                        (long long)L->n, kMaxRowsPerCluster);
    LutParams p;
    p.Wp = static_cast<const uint4*>(packed_d);
    p.scales = scales_d;
    p.X = reinterpret_cast<const float2*>(x_d);
    p.Y = reinterpret_cast<float2*>(y_d);
    p.n = L->n;
    p.m = L->m;
    p.T = T;
    p.S = S;
    p.per_row = L->scale_mode == WW_SCALES_PER_ROW;
    p.conv = L->conv;
    p.pdl = (L->flags & WW_FLAG_PDL) != 0;
    cfg.gridDim = dim3(C * S);
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
    cfg.numAttrs = 2;
    const cudaError_t le = cudaLaunchKernelEx(&cfg, wl_lut_kernel, p);
    if (le != cudaSuccess)
        return ww::fail(WW_ERR_CUDA, "ww_wl_gemv_lut: %s", cudaGetErrorString(le));
    return ww::ok();
}

// WW_LAYOUT_LUT81 arm of ww_pack_ternary_device_layout (arguments already checked there)
namespace ww {
int pack_lut81_device(const int8_t* planes_d, int64_t n, int64_t m, int64_t ld, uint32_t* out_d,
                      int32_t* bad_d, void* stream) {
    const int T = lut_steps(m);
    const int64_t total = n * (int64_t)T * 128;
    pack_lut81_kernel<<<ww::device_sms() * 8, 256, 0, (cudaStream_t)stream>>>(planes_d, n, m, ld, T, total,
                                                                           out_d, bad_d);
    return (int)cudaGetLastError();
}
}  // namespace ww
