// sm_100a kernels of the fused ternary widely-linear GEMV (FairyFuse, arXiv 2604.20913)
// and the device packer, plus their C-ABI launchers (include/ww.h).
//
// Hot path per output row i (Alg. 1, re-designed for B200):
//   * weights: one 16-byte COL4 chunk (16 columns x 4 planes, 2 bits per code) per lane per
//     step, 128-bit coalesced non-allocating loads straight from HBM (a4);
//   * activations: x staged once per CTA in shared memory by TMA (cp.async.bulk.tensor, else
//     cp.async) (a3; O2), 16-byte granules XOR-swizzled (128B swizzle) so the 32
//     lanes (32 different chunks) read conflict-free;
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
#include <atomic>
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "ww.h"
#include "ww_internal.h"
#include "ww_sweep.cuh"

#ifndef WW_X_LDG
#define WW_X_LDG 0  // experiment switch: x staged by plain 16-B loads of every thread
#endif
#ifndef WW_SWEEP_UNROLL2
#define WW_SWEEP_UNROLL2 0  // experiment switch (tools/build.py --variant)
#endif
#ifndef WW_DEBUG_FLAGS
#define WW_DEBUG_FLAGS 0  // 1: honour Params::dbg (tools/chain_time.py builds build/libww_dbg.so)
#endif

namespace {

// warps per CTA, a multiple of 4 so the four SM sub-partitions get equal warps: 16 while
// the B accumulators leave room, 8 (255-register cap) above
template <int B>
__host__ __device__ constexpr int warps_for() { return B <= 4 ? 16 : 8; }
inline int warps_for_b(int B) { return B <= 4 ? 16 : 8; }
constexpr int kXBudgetBytes = 184 * 1024;  // x tile per CTA (multi-tile path)
constexpr int kGroup = 4;                  // batches above this run as groups of 4 vectors
constexpr int64_t kSmemBudget = 226 * 1024; // single-tile path: all shared memory of a CTA
constexpr int kPrefetch = 2;                 // L2 prefetch distance beyond the weight loads
// bytes of one lane's accumulator state handed between warps (split rows, B = 1 only)
constexpr int kHandLaneBytes = (int)sizeof(Acc<1>);  // 2 column-parity sets x 4 planes x float2

#if WW_DEBUG_FLAGS
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
#endif

#ifdef WW_TRACE
// per-warp event timestamps (globaltimer ns) for tools/trace_kernel.py; not in the product build
__device__ unsigned long long* g_trace = nullptr;
// slot = Params::dbg >> 8: tools/trace_kernel.py --chain gives every launch of a captured
// chain its own 148*32*32 region of the trace buffer
__device__ __forceinline__ void trace(int slot, int ev) {  // 0..28 events, 29 sweeps done,
                                                           // 30 = SM id, 31 = exit
    if (g_trace && (threadIdx.x & 31) == 0 && ev < 32) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (ev == 30) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            t = sm;
        }
        g_trace[(size_t)slot * 148 * 32 * 32 + ((size_t)blockIdx.x * 32 + (threadIdx.x >> 5)) * 32 +
                ev] = t;
    }
}
#else
__device__ __forceinline__ void trace(int, int) {}
#endif

struct alignas(64) Params {
    CUtensorMap tmap;     // x as a [B][W][32 floats] tensor, 128B-swizzled boxes (use_tma)
    const uint4* packed;  // COL4 chunks, row-major n x W
    const float* scales;  // n x 4 or 4
    const float* X;       // B x ldx complex64
    float* Y;             // B x ldy complex64
    int64_t n, m, W, ldx, ldy;
    int32_t per_row_scales, conv, tile_chunks, ntiles, aligned16;
    int32_t x_stride;     // multi-tile path: chunks per vector in the shared x tile
    int32_t use_tma;      // stage x with cp.async.bulk.tensor (else per-thread cp.async)
    int32_t single;       // 1: single x tile path (ww_launch_info.path == 0)
    int32_t J;            // single-tile path: 32-chunk sweeps (= x slices) per row
    int32_t rows_cap;     // single-tile path: rows per CTA the shared totals / scales hold
    int32_t split;        // single tile, B = 1: rows cut in two halves handed between warps
                          // (ww_launch_info.parts == 2)
    int32_t dbg;          // tools only (ww_debug_set_flags): 1 = skip griddepcontrol.wait,
                          // bits 8..: trace slot (WW_TRACE builds),
                          // 2 = skip the accumulation, 8 = bulk L2 prefetch of the CTA's
                          // weights at kernel start (overhead measurement); 0 in the product
    // fused decode-block ops (ww_wl_gemv_fused; B = 1, single tile, TMA staging only)
    int32_t pro, epi;     // WW_PRO_*, WW_EPI_*
    float eps;
    const float* gamma;   // WW_PRO_RMSNORM: 2m fp32
    const float* residual;  // WW_EPI_RESIDUAL: complex64 by global row
    int64_t silu_rows, row0;  // WW_EPI_SILU bound; global index of local row 0
    CUtensorMap tmap2;    // WW_PRO_MUL: second operand, staged after x
};

// cp.async of one 16-byte x granule (columns col, col+1 of vector row `src`), zero-filling
// columns >= m (R6)
__device__ __forceinline__ void stage_granule(const Params& p, uint32_t dst, const float* src,
                                              int64_t valid) {
    if (p.aligned16) {
        const int bytes = valid >= 2 ? 16 : (valid == 1 ? 8 : 0);
        cp_async16(dst, bytes ? (const void*)src : (const void*)p.X, bytes);
    } else {
        cp_async8(dst, valid >= 1 ? (const void*)src : (const void*)p.X, valid >= 1 ? 8 : 0);
        cp_async8(dst + 8, valid >= 2 ? (const void*)(src + 2) : (const void*)p.X,
                  valid >= 2 ? 8 : 0);
    }
}

// Multi-tile path: cp.async copies of x columns of chunks [c0, c0 + tc_n) for all B vectors
// into the swizzled tile: granule g (columns 2g, 2g+1) of tile chunk tc lives at
// ((b*XS + tc)*8 + (g ^ (tc&7)))*16, so 32 lanes reading 32 consecutive chunks hit 32 banks.
template <int B>
__device__ __forceinline__ void stage_x(const Params& p, uint32_t xs, int64_t c0, int tc_n) {
    const int XS = p.x_stride;
    const int span8 = tc_n * 8;
#pragma unroll 1
    for (int b = 0; b < B; ++b) {
        const float* xb = p.X + 2 * (b * p.ldx + c0 * 16);
        const uint32_t base = xs + (uint32_t)(b * XS * 128);
        for (int g = threadIdx.x; g < span8; g += blockDim.x) {
            const int tc = g >> 3, gg = g & 7;
            const uint32_t dst = base + (uint32_t)((tc * 8 + (gg ^ (tc & 7))) * 16);
            stage_granule(p, dst, xb + 4 * g, p.m - (c0 * 16 + 2 * g));
        }
    }
}

// Single-tile x staging: vector b's 32*J chunks at xs + b*J*4096, chunk c at + c*128,
// granules swizzled by (c & 7) -- the 128B-swizzle TMA layout, since the region is 1024-B
// aligned.  Slice j = chunks [32j, 32j+32) of every vector, completing mbarrier j.

template <int B>
__device__ __forceinline__ void stage_x_regions_cp_async(const Params& p, uint32_t xs,
                                                         uint32_t bars) {
    const int J = p.J;
    for (int j = 0; j < J; ++j) {
        const int span = 32 * 8;  // granules per vector in one slice
        for (int t = threadIdx.x; t < B * span; t += blockDim.x) {
            const int b = B == 1 ? 0 : t / span;
            const int g = 32 * 8 * j + (B == 1 ? t : t - b * span);
            const int tc = g >> 3, gg = g & 7;
            const int64_t col = (int64_t)tc * 16 + 2 * gg;
            const uint32_t dst = xs + (uint32_t)(((b * J * 32 + tc) * 8 + (gg ^ (tc & 7))) * 16);
            // columns past m (padding of the last slice) are zero-filled
            stage_granule(p, dst, p.X + 2 * (b * p.ldx + col), p.m - col);
        }
        cp_async_arrive(bars + 8 * j);
    }
}

// one thread per slice issues its TMA boxes (B of them), so all slices are in flight at once
template <int B>
__device__ __forceinline__ void stage_x_regions_tma(const Params& p, uint32_t xs, uint32_t bars) {
    const int J = p.J;
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
        const uint32_t bar = bars + 8 * j;
        const bool two = B == 1 && p.pro == WW_PRO_MUL;  // + the second operand's slice
        mbar_expect_tx(bar, (uint32_t)(B * 4096 * (two ? 2 : 1)));
#pragma unroll 1
        for (int b = 0; b < B; ++b)
            tma_load_3d(xs + (uint32_t)((b * J + j) * 4096), &p.tmap, 0, 32 * j, b, bar);
        if (two) tma_load_3d(xs + (uint32_t)((J + j) * 4096), &p.tmap2, 0, 32 * j, 0, bar);
    }
}

// Epilogue arithmetic (a8): the row's 8 scales applied once to its totals T of vector b
// (s = [sUr, sUi, sWr, sWi]), EQ1 or ALG1 signs, one complex64 store.
__device__ __forceinline__ void store_y(const Params& p, const float (&T)[8], const float* s,
                                        int b, int64_t row) {
    const float sUr = s[0], sUi = s[1], sWr = s[2], sWi = s[3];
    const float yre = sUr * T[0] - sUi * T[3] + sWr * T[4] + sWi * T[7];          // Eq. 2
    const float yim = p.conv == WW_CONV_EQ1
                          ? sUr * T[1] + sUi * T[2] - sWr * T[5] + sWi * T[6]   // Eq. 1
                          : sUr * T[1] + sUi * T[2] + sWr * T[5] - sWi * T[6];  // Eq. 3
    reinterpret_cast<float2*>(p.Y)[b * p.ldy + row] = make_float2(yre, yim);
}

// B = 1 epilogue with a fused op (NEXT-3): residual add, or SiLU of the rows below silu_rows
// (global row index), after the scales -- the same arithmetic as the program kernel.
__device__ __forceinline__ void store_y_ops(const Params& p, const float (&T)[8], const float* s,
                                            int64_t row, float2 res, float rnorm) {
    const float sUr = s[0], sUi = s[1], sWr = s[2], sWi = s[3];
    float yre = sUr * T[0] - sUi * T[3] + sWr * T[4] + sWi * T[7];               // Eq. 2
    float yim = p.conv == WW_CONV_EQ1 ? sUr * T[1] + sUi * T[2] - sWr * T[5] + sWi * T[6]
                                      : sUr * T[1] + sUi * T[2] + sWr * T[5] - sWi * T[6];
    if (p.pro == WW_PRO_RMSNORM) {  // the RMSNorm scalar of the prologue (linear map)
        yre = yre * rnorm;
        yim = yim * rnorm;
    }
    if (p.epi == WW_EPI_RESIDUAL) {
        yre = yre + res.x;
        yim = yim + res.y;
    } else if (p.epi == WW_EPI_SILU && p.row0 + row < p.silu_rows) {
        yre = silu_f(yre);
        yim = silu_f(yim);
    }
    reinterpret_cast<float2*>(p.Y)[row] = make_float2(yre, yim);
}

// Multi-tile epilogue: lane b < B takes vector b's totals from the warp scratch T0.
template <int B>
__device__ __forceinline__ void epilogue(const Params& p, const float* T0, int64_t row) {
    const int lane = threadIdx.x & 31;
    if (lane < B) {
        float T[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) T[i] = T0[8 * lane + i];
        store_y(p, T, p.scales + (p.per_row_scales ? 4 * row : 0), lane, row);
    }
    __syncwarp();
}

// Split-row hand-off of one lane's accumulator state (B = 1): float4 i of the lane at
// addr + 512 i (32 lanes x 16 B per step: conflict-free), published by the 32 lanes'
// mbarrier arrivals (release) and read after the receiver's wait (acquire).
template <int B>
__device__ __forceinline__ void hand_store(const Acc<B>& acc, uint32_t addr) {
    const float2* a = &acc.a[0][0][0][0];
#pragma unroll
    for (int i = 0; i < (int)sizeof(Acc<B>) / 16; ++i)
        sts128_f4(addr + 512u * i, make_float4(a[2 * i].x, a[2 * i].y, a[2 * i + 1].x, a[2 * i + 1].y));
}
template <int B>
__device__ __forceinline__ void hand_load(Acc<B>& acc, uint32_t addr) {
    float2* a = &acc.a[0][0][0][0];
#pragma unroll
    for (int i = 0; i < (int)sizeof(Acc<B>) / 16; ++i) {
        const float4 v = lds128(addr + 512u * i);
        a[2 * i] = make_float2(v.x, v.y);
        a[2 * i + 1] = make_float2(v.z, v.w);
    }
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Shared-memory carve-up (bytes), identical on host (plan) and device.
struct SmemLayout {
    int64_t x_bytes, scratch_off, tot_off, scale_off, bar_off, hand_off, hbar_off, desc_off, total;
};

// x first (1024-B aligned for the 128B-swizzled TMA boxes), then per-warp reduction scratch
// (multi-tile path), then -- single tile only -- the reduced totals of every CTA row
// ([rows][NV] floats), the CTA's row scales and one mbarrier per x slice.
// Single tile: x_chunks = 32*J per vector; multi-tile: the tile width.
// Split rows (single tile, B = 1): one hand-off slot of 32 lane states per warp, then one
// mbarrier per warp.
__host__ __device__ inline SmemLayout smem_layout(int B, int x_chunks, int warps, bool single,
                                                  int nbars, int rows, bool x2 = false,
                                                  bool split = false) {
    const int64_t nv = next_pow2(8 * B);
    SmemLayout L;
    L.x_bytes = (int64_t)B * x_chunks * 128;
    // WW_PRO_MUL: the second operand right after x; then 32 floats of RMSNorm partials
    L.scratch_off = L.x_bytes * (x2 ? 2 : 1) + 128;
    L.tot_off = L.scratch_off + (single ? 0 : (int64_t)warps * nv * 4);
    L.scale_off = L.tot_off + (single ? (int64_t)rows * nv * 4 : 0);
    // scales: one 16-B slot per CTA row (per-row mode) or per warp (per-tensor mode)
    L.bar_off = L.scale_off + (single ? 16 * (int64_t)(rows > warps ? rows : warps) : 0);
    L.hand_off = (L.bar_off + (single ? 8 * (int64_t)nbars : 0) + 15) / 16 * 16;
    L.hbar_off = L.hand_off + (split ? (int64_t)warps * 32 * kHandLaneBytes : 0);
    L.desc_off = L.hbar_off + (split ? 8 * (int64_t)warps : 0);  // 16-B per-warp descriptors
    L.total = L.desc_off + (split ? 16 * (int64_t)warps : 0) + 1024;  // + base alignment slack
    return L;
}

// register cap: B == 1 keeps <= 64 registers so two CTAs fit an SM and a PDL-launched next
// layer can start on every SM while this one drains
template <int B>
__host__ __device__ constexpr int min_blocks() { return B == 1 ? 2 : 1; }

// kStream: single x tile with W a multiple of 32 -- the warp's rows are one contiguous stream
// of whole sweeps (launch_b picks the instantiation; each has only one sweep loop)
template <int B, bool kStream>
__global__ void __launch_bounds__(warps_for<B>() * 32, min_blocks<B>())
wl_gemv_kernel(const __grid_constant__ Params p) {
    constexpr int NV = next_pow2(8 * B);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t xs = (raw + 1023u) & ~1023u;  // 1024-B aligned x tile
    unsigned char* smem = smem_raw + (xs - raw);
    const int nwarps = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool single = p.single != 0;
    const int nbars = single ? p.J : 0;
    const SmemLayout SL = smem_layout(B, single ? 32 * p.J : p.x_stride, nwarps, single, nbars,
                                      p.rows_cap, p.pro == WW_PRO_MUL, B == 1 && p.split);
    float* part = reinterpret_cast<float*>(smem + SL.scratch_off - 128);  // [32]
    float* sc = reinterpret_cast<float*>(smem + SL.scratch_off) + warp * NV;
    const uint32_t bars = xs + (uint32_t)SL.bar_off;

    // balanced contiguous row range of this CTA (A12 row-parallel decomposition)
    const int64_t r0 = (int64_t)blockIdx.x * p.n / gridDim.x;
    const int64_t r1 = (int64_t)(blockIdx.x + 1) * p.n / gridDim.x;
    if (single) {
        // one mbarrier per thread (an init is a shared-memory atomic; a serial loop by one
        // thread is measurably slow)
        for (int j = threadIdx.x; j < nbars; j += blockDim.x)
            mbar_init(bars + 8 * j, p.use_tma ? 1u : blockDim.x);
        if (B == 1 && p.split && threadIdx.x < nwarps)  // hand-off barriers: 32 lane arrivals
            mbar_init(xs + (uint32_t)SL.hbar_off + 8u * threadIdx.x, 32u);
        fence_barrier_init();
    }

    // PDL: let the next kernel launch now.  (A bulk L2 prefetch of the CTA's weights here
    // measured slower -- it competes with the running layer's stream; tools only: dbg & 8.)
    const int tslot = p.dbg >> 8;
    trace(tslot, 0);
    trace(tslot, 30);
    pdl_launch_dependents();
    // the x tensor maps' descriptors into the TMA unit's cache before the wait (they do not
    // depend on the previous kernel), so the first box after the wait does not fetch them
    if (single && p.use_tma && threadIdx.x == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
        if (p.pro == WW_PRO_MUL)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap2)) : "memory");
    }
#if WW_DEBUG_FLAGS
    if (threadIdx.x == 0 && (p.dbg & 8)) {
        const char* wb = reinterpret_cast<const char*>(p.packed + r0 * p.W);
        const int64_t bytes = (r1 - r0) * p.W * 16;
        for (int64_t off = 0; off < bytes; off += 65536)
            prefetch_l2(wb + off, (uint32_t)(bytes - off < 65536 ? bytes - off : 65536));
    }
#endif
    Acc<B> acc;
    acc.zero();

    if (single) {
        // Rows: the CTA's rows are cut into contiguous per-warp ranges
        // [w0, w1) whose sizes differ by at most one, the longer ones on warps 0..e-1, so the
        // four SM sub-partitions (warp % 4) get equal work (+-1 row).  A row is J sweeps of 32
        // chunks, lane = chunk within the sweep; its arithmetic depends on (m, B) only --
        // never on n, the shard, the grid or the warp split.  Row indices are relative to
        // the CTA (int32: n <= 2^30, check_layer).
        const int NRc = (int)(r1 - r0);
        const int ub = NRc / nwarps, ue = NRc - ub * nwarps;
        const int w0 = warp * ub + (warp < ue ? warp : ue);
        const int w1 = w0 + ub + (warp < ue ? 1 : 0);
        const int J = p.J;
        const bool lastok = lane < (int)p.W - 32 * (J - 1);  // lane active in the last sweep

        // Weight stream (a4): the warp's rows in order; each lane reads its 16-byte chunk of
        // a sweep with a streaming 128-bit load, two sweeps ahead, the first two issued
        // before griddepcontrol.wait (weights never depend on the previous kernel).  Lanes
        // past the row's end load zeros, so no predicate fires for them.  Sweep pk of the
        // producer's row pr is loaded iff pk < kv: kv = J on lanes active in the last sweep,
        // J - 1 on the others, 0 past the warp's last row (one compare per sweep).
        const int kvl = lastok ? J : J - 1;
        int pr = w0, pk = 0, kv = w0 < w1 ? kvl : 0;
        const uint4* pptr = p.packed + (r0 + w0) * p.W + lane;
        const int64_t jrow = p.W - 32 * (int64_t)J;  // from the chunk after a row to the next
        auto load_rows = [&]() -> uint4 {
            const uint4 w = ldg_stream_lt(pptr, pk, kv);
            pptr += 32;
            if (++pk == J) {  // next row
                pk = 0;
                pptr += jrow;
                kv = ++pr < w1 ? kvl : 0;
            }
            return w;
        };
        // kStream: the producer only counts sweeps (no row transitions), and prefetches into
        // L2 the chunk kPrefetch sweeps beyond each load
        const int nsweeps = (w1 - w0) * J;
        auto load_stream = [&]() -> uint4 {
            prefetch_chunk_lt(pptr + 32 * kPrefetch, pk + kPrefetch, nsweeps);
            const uint4 w = ldg_stream_lt(pptr, pk, nsweeps);
            pptr += 32;
            ++pk;
            return w;
        };
        // Split rows (p.split, B = 1): the CTA's rows are cut into 2 NRc half
        // units (row u >> 1, sweeps [0, h) or [h, J), h = ceil(J/2)) and the units are dealt
        // out like rows, so the four sub-partitions get equal work to +-1 half row.  A warp
        // whose range ends with a first half (giver) sweeps it first and hands its lane state
        // to the next warp through shared memory; a warp whose range starts with a second half
        // (receiver) sweeps it last, continuing from that state -- no warp waits on a later
        // one, and a row's accumulation order is the whole-row order.
        const int hJ = (J + 1) / 2;
        // the warp's split geometry {mr0, mr1, giver | receiver << 1, nseg} lives in shared
        // memory and is re-read at each (rare) segment change, so it holds no registers
        // across the sweep loop
        const uint32_t desc = xs + (uint32_t)SL.desc_off + 16u * warp;
        int er0 = w0, er1 = w1;  // rows whose epilogue this warp runs (scales copied)
        bool has_work = w0 < w1;
        if (B == 1 && p.split) {
            const int NU = 2 * NRc;
            const int uub = NU / nwarps, uue = NU - uub * nwarps;
            const int u0 = warp * uub + (warp < uue ? warp : uue);
            const int u1 = u0 + uub + (warp < uue ? 1 : 0);
            const bool giv = u1 > u0 && ((u1 - 1) & 1) == 0;
            const bool rcv = u1 > u0 && (u0 & 1) == 1;
            const int mr0 = (u0 + (rcv ? 1 : 0)) >> 1, mr1 = (u1 - (giv ? 1 : 0)) >> 1;
            const int nseg = (giv ? 1 : 0) + (mr1 - mr0) + (rcv ? 1 : 0);
            if (lane == 0)
                asm volatile("st.shared.v4.s32 [%0], {%1,%2,%3,%4};" ::"r"(desc), "r"(mr0), "r"(mr1),
                             "r"((giv ? 1 : 0) | (rcv ? 2 : 0)), "r"(nseg)
                             : "memory");
            __syncwarp();
            er0 = rcv ? mr0 - 1 : mr0;
            er1 = mr1;
            has_work = nseg > 0;
        }
        struct Seg {
            int row, kb, ke, kind;  // kind: 0 giver half, 1 whole row, 2 receiver half
        };
        auto seg_of = [&](int i, int& nseg) -> Seg {
            int mr0, mr1, fl;
            asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(mr0), "=r"(mr1), "=r"(fl), "=r"(nseg)
                         : "r"(desc)
                         : "memory");
            const int g = fl & 1;
            if (g && i == 0) return Seg{mr1, 0, hJ, 0};
            if (i - g < mr1 - mr0) return Seg{mr0 + i - g, 0, J, 1};
            return Seg{mr0 - 1, hJ, J, 2};
        };
        // segmented producer (split rows): sweeps of the segments in processing order, the
        // L2 prefetch kPrefetch sweeps ahead inside a segment as in the stream producer
        int spi = 0, spk = 0, spke = 0, skv = 0;
        const uint4* sptr = p.packed;
        if (B == 1 && p.split && has_work) {
            int ns;
            const Seg sg = seg_of(0, ns);
            spk = sg.kb;
            spke = sg.ke;
            skv = spke < kvl ? spke : kvl;
            sptr = p.packed + (r0 + sg.row) * p.W + lane + 32 * spk;
        }
        auto load_seg = [&]() -> uint4 {
            prefetch_chunk_lt(sptr + 32 * kPrefetch, spk + kPrefetch, skv);
            const uint4 w = ldg_stream_lt(sptr, spk, skv);
            sptr += 32;
            if (++spk == spke) {
                int ns;
                const Seg sg = seg_of(++spi, ns);
                if (spi < ns) {
                    const int kv = (threadIdx.x & 31) < (int)p.W - 32 * (p.J - 1) ? p.J : p.J - 1;
                    spk = sg.kb;
                    spke = sg.ke;
                    skv = spke < kv ? spke : kv;
                    sptr = p.packed + (r0 + sg.row) * p.W + (threadIdx.x & 31) + 32 * spk;
                } else {
                    skv = 0;
                }
            }
            return w;
        };
        float* tot = reinterpret_cast<float*>(smem + SL.tot_off);  // [rows][NV]
        float4 gam[kGammaRegs];  // WW_PRO_RMSNORM: this thread's gamma (a weight), pre-wait
        if (B == 1 && p.pro == WW_PRO_RMSNORM)
            gamma_prefetch(gam, p.gamma, p.m, J, threadIdx.x, blockDim.x);
        float rnorm = 1.0f;  // RMSNorm factor, applied in the epilogue
        auto run = [&](auto&& load_next, auto split_tag) {
            uint4 qa = load_next(), qb = load_next();
            __syncthreads();  // mbarrier inits visible
            trace(tslot, 1);
#if WW_DEBUG_FLAGS
            if (!(p.dbg & 1))
#endif
                pdl_wait();
            trace(tslot, 2);
            if (WW_X_LDG && B == 1 && p.use_tma && p.pro == WW_PRO_NONE) {
                // experiment: every thread loads its x granules (16 B) and stores them swizzled
                const int ng = 8 * 32 * J;
                const float4* xg = reinterpret_cast<const float4*>(p.X);
                for (int gi = threadIdx.x; gi < ng; gi += blockDim.x) {
                    const int c = gi >> 3, g = gi & 7;
                    const int64_t col = 16 * (int64_t)c + 2 * g;
                    const float4 v = col < p.m ? __ldcg(xg + (col >> 1)) : make_float4(0.f, 0.f, 0.f, 0.f);
                    sts128_f4(xs + 16u * (uint32_t)(c * 8 + (g ^ (c & 7))), v);
                }
                __syncthreads();
            } else if (p.use_tma) {
                stage_x_regions_tma<B>(p, xs, bars);
            } else {
                stage_x_regions_cp_async<B>(p, xs, bars);
            }
            // (x first: the scales are needed only at the end of the warp's first row)
            // the warp's row scales -> shared memory (cp.async), after griddepcontrol.wait so
            // a preceding kernel may write them (ww.h WW_FLAG_PDL); per-row mode: rows
            // [w0, w1) at slot r, per-tensor mode: the 4 scales at the warp's own slot.  The
            // warp waits for its copies before its first epilogue (no CTA barrier).
            {
                const uint32_t sdst = xs + (uint32_t)SL.scale_off;
                if (p.per_row_scales) {
                    const float* src = p.scales + 4 * (r0 + er0);
                    const int ns = 4 * (er1 - er0);
                    for (int i = lane; i < ns; i += 32) cp_async4(sdst + 16u * er0 + 4u * i, src + i);
                } else if (lane < 4) {
                    cp_async4(sdst + 16u * warp + 4u * lane, p.scales + lane);
                }
            }

            trace(tslot, 3);
            int tr_sweep = 4;

            const uint32_t l7 = (uint32_t)(lane & 7) << 4;  // swizzle key of the lane's chunks
            const uint32_t xb = (xs + (uint32_t)lane * 128u) | l7;
            const uint32_t bstride = (uint32_t)J * 4096u;
            if (B == 1 && p.pro != WW_PRO_NONE) {
                // fused prologue op (ww_sweep.cuh, NEXT-3): the whole CTA waits for x, rewrites
                // it in place, and only then sweeps
                for (int j = 0; j < J; ++j) mbar_wait0(bars + 8 * j);
                const int ng = 8 * 32 * J;
                if (p.pro == WW_PRO_MUL) {
                    x_mul(xs, xs + (uint32_t)J * 4096u, ng, threadIdx.x, blockDim.x);
                } else {
                    const float ss =
                        x_gamma_sumsq_warp(xs, ng, threadIdx.x, blockDim.x, gam, p.gamma, p.m);
                    if (lane == 0) part[warp] = ss;
                }
                __syncthreads();
                if (p.pro == WW_PRO_RMSNORM) rnorm = rms_factor(part, nwarps, p.m, p.eps);
            } else if (has_work && !(WW_X_LDG && B == 1 && p.use_tma)) {  // x slices in before
                for (int j = 0; j < J; ++j) mbar_wait0(bars + 8 * j);     // the warp's first sweep
            }
            if constexpr (decltype(split_tag)::value) {
                // split rows: segments in processing order (giver half, whole rows, receiver
                // half); the lane state of a row's first half continues in the next warp, so
                // every row is accumulated sweep 0..J-1 in order, exactly as a whole row
                const uint32_t hand = xs + (uint32_t)SL.hand_off;
                const uint32_t hbar = xs + (uint32_t)SL.hbar_off;
                bool scales_ready = false;
                int nseg = has_work ? 1 : 0;
#pragma unroll 1
                for (int i = 0; i < nseg; ++i) {
                    const Seg sg = seg_of(i, nseg);
                    const int row = sg.row, kb = sg.kb, ke = sg.ke;
                    const bool is_giv = sg.kind == 0, is_rcv = sg.kind == 2;
                    float2 res = make_float2(0.f, 0.f);
                    if (B == 1 && p.epi == WW_EPI_RESIDUAL && lane == 0 && !is_giv)
                        res = __ldcg(reinterpret_cast<const float2*>(p.residual) + p.row0 + r0 + row);
                    if (is_rcv) {  // the previous warp's state after sweeps [0, h) of this row
                        mbar_wait0(hbar + 8u * (warp - 1));
                        const uint32_t src = hand + (uint32_t)(warp - 1) * 32u * kHandLaneBytes;
                        hand_load(acc, src + 16u * lane);
                    }
                    uint32_t xc = xb + 4096u * (uint32_t)kb;
#pragma unroll 1
                    for (int k = kb; k < ke; ++k) {
                        const uint4 cur = qa;
                        qa = qb;
                        qb = load_next();
                        chunk<B>(acc, cur, xc, bstride);
                        xc += 4096u;
                    }
                    if (is_giv) {  // hand the lane state to the next warp
                        hand_store(acc, hand + (uint32_t)warp * 32u * kHandLaneBytes + 16u * lane);
                        mbar_arrive(hbar + 8u * warp);
                        acc.zero();
                        continue;
                    }
                    reduce_to<B>(acc, tot + row * NV);
                    if (!scales_ready) {
                        cp_async_wait_all();
                        __syncwarp();
                        scales_ready = true;
                    }
                    if (lane < B) {
                        float T[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) T[q] = tot[row * NV + 8 * lane + q];
                        const float* sr = reinterpret_cast<const float*>(smem + SL.scale_off) +
                                          4 * (p.per_row_scales ? row : warp);
                        if (B == 1 && (p.epi != WW_EPI_NONE || p.pro == WW_PRO_RMSNORM))
                            store_y_ops(p, T, sr, r0 + row, res, rnorm);
                        else
                            store_y(p, T, sr, lane, r0 + row);
                    }
                    acc.zero();
                }
            } else {
#pragma unroll 1
            for (int r = w0; r < w1; ++r) {
                uint32_t xc = xb;
                float2 res = make_float2(0.f, 0.f);  // WW_EPI_RESIDUAL operand, a row ahead
                if (B == 1 && p.epi == WW_EPI_RESIDUAL && lane == 0)
                    res = __ldcg(reinterpret_cast<const float2*>(p.residual) + p.row0 + r0 + r);
#if WW_SWEEP_UNROLL2
                // two sweeps per iteration: the second sweep's x sits 4096 B above the
                // first's with the same swizzle key, so its LDS use immediate offsets
#pragma unroll 1
                for (int k = 0; k + 1 < J; k += 2) {
                    uint4 cur = qa;
                    qa = qb;
                    qb = load_next();
                    chunk<B>(acc, cur, xc, bstride, 0u);
                    cur = qa;
                    qa = qb;
                    qb = load_next();
                    chunk<B>(acc, cur, xc, bstride, 4096u);
                    xc += 8192u;
                }
                if (J & 1) {
                    const uint4 cur = qa;
                    qa = qb;
                    qb = load_next();
                    chunk<B>(acc, cur, xc, bstride);
                    xc += 4096u;
                }
#else
#pragma unroll 1
                for (int k = 0; k < J; ++k) {
                    const uint4 cur = qa;
                    qa = qb;
                    qb = load_next();
                    if (tr_sweep < 29) trace(tslot, tr_sweep++);
#if WW_DEBUG_FLAGS
                    if (!(p.dbg & 2))
#endif
                        chunk<B>(acc, cur, xc, bstride);
                    xc += 4096u;
                }
#endif
                // reduce the row over the lanes (a7) into the CTA's totals
                reduce_to<B>(acc, tot + r * NV);
                if (r == w0) {  // before the warp's first epilogue: its scale copies have landed
                    cp_async_wait_all();
                    __syncwarp();
                }
                // epilogue (a8) of the row by its own warp (no CTA barrier): lane b < B
                // applies the row's 8 scale multiplies to vector b's totals, one complex64
                // store
                if (lane < B) {
                    float T[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) T[i] = tot[r * NV + 8 * lane + i];
                    const float* sr = reinterpret_cast<const float*>(smem + SL.scale_off) +
                                      4 * (p.per_row_scales ? r : warp);
                    if (B == 1 && (p.epi != WW_EPI_NONE || p.pro == WW_PRO_RMSNORM))
                        store_y_ops(p, T, sr, r0 + r, res, rnorm);
                    else
                        store_y(p, T, sr, lane, r0 + r);
                }
                if (tr_sweep < 29) trace(tslot, tr_sweep++);
                acc.zero();
            }
            }
        };
        bool ran = false;
        if constexpr (B == 1) {
            if (p.split) {
                run(load_seg, std::true_type{});
                ran = true;
            }
        }
        if (!ran) {
            if constexpr (kStream)
                run(load_stream, std::false_type{});
            else
                run(load_rows, std::false_type{});
        }
        trace(tslot, 29);  // sweeps done
        trace(tslot, 31);
        return;
    }

    // x does not fit one tile: row waves, each streaming the tiles with CTA-wide syncs
    const int TC = p.tile_chunks;
    const uint32_t bstride = (uint32_t)p.x_stride * 128u;
    pdl_wait();
    for (int64_t wr = r0; wr < r1; wr += nwarps) {  // uniform across the CTA
        const int64_t row = wr + warp;
        const bool active = row < r1;
        for (int t = 0; t < p.ntiles; ++t) {
            const int64_t c0 = (int64_t)t * TC;
            const int tc_n = (int)(p.W - c0 < TC ? p.W - c0 : TC);
            __syncthreads();  // previous tile fully consumed
            stage_x<B>(p, xs, c0, tc_n);
            cp_async_wait_all();
            __syncthreads();
            if (active) {
                const uint4* wrow = p.packed + row * p.W + c0;
                int tc = lane;
                uint4 cur = tc < tc_n ? ldg_stream(wrow + tc) : make_uint4(0, 0, 0, 0);
                for (; tc < tc_n; tc += 32) {
                    const uint4 nxt =
                        tc + 32 < tc_n ? ldg_stream(wrow + tc + 32) : make_uint4(0, 0, 0, 0);
                    chunk<B>(acc, cur, (xs + (uint32_t)tc * 128u) | ((uint32_t)(lane & 7) << 4),
                             bstride);
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
        bool bad_word = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t j = 16 * c + 4 * q + k;
            if (j >= m) continue;
            uint32_t byte = 0;
            bool bad_col = false;  // only this column packs as zero (ww.h)
#pragma unroll
            for (int pl = 0; pl < 4; ++pl) {
                const int8_t t = planes[(int64_t)pl * n * ld + i * ld + j];
                if (t == 1) byte |= 2u << (2 * pl);
                else if (t == -1) byte |= 1u << (2 * pl);
                else if (t != 0) bad_col = true;
            }
            if (!bad_col) word |= byte << (8 * k);
            bad_word |= bad_col;
        }
        out[e] = word;
        if (bad_word && bad) atomicOr(bad, 1);
    }
}

// ------------------------------------------------------------------ launch configuration
int num_sms() { return ww::device_sms(); }

// tests: -1 = planner decides, 0 / 1 = force whole / split rows (B = 1, single tile, J >= 2)
std::atomic<int> g_force_split{-1};

ww_status plan(const ww_layer* L, int32_t B, int sms, ww_launch_info* li) {
    const int64_t W = ww::words_per_row(L->m);
    const int warps = warps_for_b(B);
    // one CTA per SM (persistent), each owning a contiguous, balanced row range
#ifndef WW_CTAS_PER_SM
#define WW_CTAS_PER_SM 1  // experiment switch: B = 1 launches with 2 CTAs per SM (tools only)
#endif
    const int64_t grid = std::min<int64_t>((B == 1 ? WW_CTAS_PER_SM : 1) * (int64_t)sms, L->n);
    const int64_t rows = (L->n + grid - 1) / grid;  // rows per CTA (at most)
    // Single x tile: the whole row is one work unit of T = ceil(W/32) sweeps (x must fit
    // kXBudgetBytes); else column tiles.  (Splitting rows into column parts handed between
    // warps measured slower once the per-sweep load logic was one compare: DESIGN.md §6.)
    const int64_t T = (W + 31) / 32;
    const int64_t single_bytes =  // + the CTA's row totals and scales
        smem_layout(B, (int)(32 * T), warps, true, (int)T, (int)std::min<int64_t>(rows, 1 << 20))
            .total;
    li->grid = (int32_t)grid;
    li->block = 32 * warps;
    li->num_sms = sms;
    if ((int64_t)B * 32 * T * 128 <= kXBudgetBytes && single_bytes <= kSmemBudget) {
        li->tile_chunks = (int32_t)W;
        li->tiles = 1;
        li->parts = 1;
        li->split_chunks = (int32_t)W;
        li->smem_bytes = (int32_t)single_bytes;
        li->path = 0;
        // B = 1: cut rows into two halves handed between warps when that shortens the
        // busiest SM sub-partition's share by >= 4 % (n = 2048 shapes: 14 rows per CTA on 16
        // warps leave sub-partitions with 4 + 4 + 3 + 3 rows; halves give 7 + 7 + 7 + 7).
        // Results are bitwise the same either way (the hand-off keeps the row's order).
        // Only for rows of a ragged last sweep (W % 32 != 0, the row-by-row producer): where
        // W = 32 J the whole-row stream producer (no row transitions) measured faster than
        // halves on every config-4 shape.
        if (B == 1 && T >= 2 && (W % 32 != 0 || g_force_split.load() == 1)) {
            const int sp = warps / 4;  // warps per sub-partition
            const double whole = (double)((rows + 4 - 1) / 4) * T;
            const double halves = (double)((2 * rows + 4 - 1) / 4) * 0.5 * T;
            const int force = g_force_split.load();
            const bool split = force >= 0 ? force != 0 : (sp >= 1 && halves <= 0.96 * whole);
            const int64_t split_bytes =
                smem_layout(B, (int)(32 * T), warps, true, (int)T,
                            (int)std::min<int64_t>(rows, 1 << 20), false, true).total;
            if (split && split_bytes <= kSmemBudget) {
                li->parts = 2;
                li->split_chunks = (int32_t)((T + 1) / 2 * 32);
                li->smem_bytes = (int32_t)split_bytes;
            }
        }
        return WW_OK;
    }
    // x (or the CTA's row totals) does not fit one tile: column tiles of whole 32-chunk
    // sweeps, one part per row, row waves
    int64_t tc = kXBudgetBytes / ((int64_t)B * 128);
    tc = std::min<int64_t>(std::max<int64_t>(32, tc / 32 * 32), (W + 31) / 32 * 32);
    li->tile_chunks = (int32_t)tc;
    li->tiles = (int32_t)((W + tc - 1) / tc);
    li->parts = 1;
    li->split_chunks = (int32_t)W;
    li->path = 1;
    li->smem_bytes = (int32_t)smem_layout(B, (int)tc, warps, false, 0, 0).total;
    return WW_OK;
}

bool encode_x_map(Params& p, int B) {
    if (p.m % 16 != 0 || ((uintptr_t)p.X & 15) || (B > 1 && (p.ldx % 2) != 0)) return false;
    return ww::encode_x_map(&p.tmap, p.X, p.W, B, p.ldx) == 0;
}

std::atomic<bool> g_force_rows{false};  // tests: run the row-by-row instantiation where kStream applies
std::atomic<int> g_last_stream{-1};     // tests: 1 if the last launch ran the kStream instantiation

template <int B>
cudaError_t launch_b(const Params& p, const ww_launch_info& li, cudaStream_t s, bool pdl) {
    void (*const kernels[2])(Params) = {wl_gemv_kernel<B, false>, wl_gemv_kernel<B, true>};
    for (auto k : kernels) {  // once per (device, kernel): ww_device.cu
        const int e = ww::prepare_kernel(reinterpret_cast<const void*>(k), 227 * 1024);
        if (e) return (cudaError_t)e;
    }
    const bool stream_rows = p.single && (p.W & 31) == 0 && !g_force_rows;
    g_last_stream = stream_rows ? 1 : 0;
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
    return cudaLaunchKernelEx(&cfg, kernels[stream_rows ? 1 : 0], p);
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

std::atomic<bool> g_force_cp_async{false};  // tests: exercise the per-thread cp.async staging path
std::atomic<int> g_debug_flags{0};           // tools/chain_time.py: Params::dbg
std::atomic<int> g_last_use_tma{-1};         // tests: whether the last launch staged x with TMA

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
    if (L->n > (int64_t)1 << 30 || L->m > (int64_t)1 << 30)
        return ww::fail(WW_ERR_UNSUPPORTED, "%s: shape too large", fn);
    return WW_OK;
}

}  // namespace

// Debug hooks: not part of the ABI (no declaration in ww.h), inert unless a test or tool
// calls them (process-wide atomics).  Lets the tests force the cp.async staging path.
extern "C" void ww_debug_force_cp_async(int on) { g_force_cp_async = on != 0; }
// Not part of the ABI: tests compare the two producer instantiations (kStream / row by row).
extern "C" void ww_debug_force_rows(int on) { g_force_rows = on != 0; }
extern "C" int ww_debug_last_stream(void) { return g_last_stream; }
// Not part of the ABI: tests compare split and whole rows (-1 = the planner's choice).
extern "C" void ww_debug_force_split(int mode) { g_force_split = mode < 0 ? -1 : (mode != 0); }
// Not part of the ABI: overhead-measurement switches for tools/chain_time.py (Params::dbg).
extern "C" void ww_debug_set_flags(int flags) { g_debug_flags = flags; }
// Not part of the ABI: 1 if the last WL-GEMV launch staged x with TMA, 0 cp.async, -1 none yet.
extern "C" int ww_debug_last_use_tma(void) { return g_last_use_tma; }

extern "C" ww_status ww_query_launch(const ww_layer* L, int32_t B, ww_launch_info* out) {
    ww_status st = check_layer(L, "ww_query_launch");
    if (st != WW_OK) return st;
    if (!out) return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_query_launch: null out");
    if (B < 1 || B > WW_MAX_BATCH)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_query_launch: B=%d", B);
    plan(L, B > kGroup ? kGroup : B, num_sms(), out);  // B > 4: one launch per group of 4
    return ww::ok();
}

#ifdef WW_TRACE
extern "C" int ww_debug_set_trace(void* dev_ptr) {
    return (int)cudaMemcpyToSymbol(g_trace, &dev_ptr, sizeof(void*));
}
#endif

namespace {
// one launch of wl_gemv_kernel<B> (arguments already validated)
ww_status launch_batch(const ww_layer* L, const void* packed_d, const float* scales_d,
                       const float* X_d, int64_t ldx, float* Y_d, int64_t ldy, int32_t B,
                       void* stream, const ww_ops* ops = nullptr) {
    ww_launch_info li;
    plan(L, B, num_sms(), &li);
    Params p;
    memset(&p, 0, sizeof p);
    if (ops) {  // ww_wl_gemv_fused (validated by the caller): B = 1, single tile, TMA
        p.pro = ops->prologue;
        p.epi = ops->epilogue;
        p.eps = ops->eps;
        p.gamma = ops->gamma;
        p.residual = ops->residual;
        p.silu_rows = ops->silu_rows;
        p.row0 = ops->row0;
        if (li.path != 0)
            return ww::fail(WW_ERR_UNSUPPORTED, "ww_wl_gemv_fused: x of m=%lld does not fit one tile",
                            (long long)L->m);
        if (p.pro == WW_PRO_MUL) {
            const int64_t T = (ww::words_per_row(L->m) + 31) / 32;
            const int64_t rows = (L->n + li.grid - 1) / li.grid;
            const int64_t bytes =
                smem_layout(1, (int)(32 * T), li.block / 32, true, (int)T, (int)rows, true,
                            li.parts == 2)
                    .total;
            if (bytes > kSmemBudget)
                return ww::fail(WW_ERR_UNSUPPORTED, "ww_wl_gemv_fused: x and x2 of m=%lld do not fit",
                                (long long)L->m);
            li.smem_bytes = (int32_t)bytes;
            if (ww::encode_x_map(&p.tmap2, ops->x2, ww::words_per_row(L->m), 1, L->m) != 0)
                return ww::fail(WW_ERR_CUDA, "ww_wl_gemv_fused: tensor map of x2");
        }
    }
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
    p.J = (int32_t)((p.W + 31) / 32);
    p.rows_cap = (int32_t)((L->n + li.grid - 1) / li.grid);
    p.aligned16 = (((uintptr_t)X_d & 15) == 0) && (ldx % 2 == 0);
    p.x_stride = (li.tile_chunks + 31) / 32 * 32;
    p.single = li.path == 0;
    p.split = li.parts == 2 ? 1 : 0;
    p.use_tma = p.single && (ops || !g_force_cp_async) ? (encode_x_map(p, B) ? 1 : 0) : 0;
    if (ops && !p.use_tma)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_wl_gemv_fused: needs TMA staging (16 | m, 16-B x)");
    p.dbg = g_debug_flags;
    g_last_use_tma = p.use_tma;
    cudaError_t e = launch(p, li, B, (cudaStream_t)stream, (L->flags & WW_FLAG_PDL) != 0);
    if (e != cudaSuccess)
        return ww::fail(WW_ERR_CUDA, "ww_wl_gemv: launch failed: %s", cudaGetErrorString(e));
    return ww::ok();
}
}  // namespace

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
    if (B > kGroup) {
        // groups of kGroup vectors, one launch each (the last group may overlap the previous
        // one and rewrite identical values): a vector's accumulation order is the same in
        // every group of the B >= 3 family, and the weights are streamed once per group --
        // cheaper than one launch over all B (x beyond one tile, 255 registers, 8 warps)
        for (int32_t g0 = 0; g0 < B; g0 += kGroup) {
            const int32_t s0 = g0 + kGroup <= B ? g0 : B - kGroup;
            const ww_status gs = launch_batch(L, packed_d, scales_d, X_d + 2 * s0 * ldx, ldx,
                                              Y_d + 2 * s0 * ldy, ldy, kGroup, stream);
            if (gs != WW_OK) return gs;
            if (s0 + kGroup >= B) break;
        }
        return ww::ok();
    }
    return launch_batch(L, packed_d, scales_d, X_d, ldx, Y_d, ldy, B, stream);
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

extern "C" ww_status ww_wl_gemv_fused(const ww_layer* L, const void* packed_d, const float* scales_d,
                                      const float* x_d, float* y_d, const ww_ops* ops,
                                      void* stream) {
    const char* fn = "ww_wl_gemv_fused";
    ww_status st = check_layer(L, fn);
    if (st != WW_OK) return st;
    if (!ops) return ww_wl_gemv(L, packed_d, scales_d, x_d, y_d, stream);
    if (!packed_d || !scales_d || !x_d || !y_d)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: null pointer", fn);
    if (ops->prologue < WW_PRO_NONE || ops->prologue > WW_PRO_MUL || ops->epilogue < WW_EPI_NONE ||
        ops->epilogue > WW_EPI_SILU || (ops->prologue == WW_PRO_MUL && !ops->x2) ||
        (ops->prologue == WW_PRO_RMSNORM && (!ops->gamma || !(ops->eps >= 0.f))) ||
        (ops->epilogue == WW_EPI_RESIDUAL && !ops->residual) || ops->row0 < 0)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: ops", fn);
    if (L->m % 16 || ((uintptr_t)x_d & 15) || ((uintptr_t)ops->x2 & 15) ||
        ((uintptr_t)ops->gamma & 15) || ((uintptr_t)ops->residual & 7) || ((uintptr_t)packed_d & 15) ||
        ((uintptr_t)y_d & 7) || ((uintptr_t)scales_d & 3))
        return ww::fail(WW_ERR_MISALIGNED, "%s: needs 16 | m and 16-B aligned x / x2 / gamma", fn);
    const char* xb = reinterpret_cast<const char*>(x_d);
    const char* yb = reinterpret_cast<const char*>(y_d);
    if (xb < yb + 8 * L->n && yb < xb + 8 * L->m)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: x and y overlap", fn);
    return launch_batch(L, packed_d, scales_d, x_d, L->m, y_d, L->n, 1, stream, ops);
}
