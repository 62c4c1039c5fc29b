// WL-GEMV for one vector (and batches up to 4) on the 5th-generation tensor cores, with the
// ternary operand decoded into TENSOR MEMORY.
//
// Why: the predicated-add datapath (wl_gemv_kernel) issues two FADD2 per code plus the
// decode and is bound by the FP32 pipe at ~32 codes/clk/SM -- 35 % of B200's HBM rate
// (DESIGN.md §6).  Streaming the paper's 2-bit codes at HBM speed needs ~63 codes/clk/SM.
// Here the eight real sub-GEMVs of Eq. 1 (Eqs. 6-7) become one exact
// integer contraction per 32-row tile:
//   D[(row, plane), (vector, component, limb)] = sum_j T_plane[row, j] * limb[j]
// with T in {-1, 0, +1} (int8) and x split into three unsigned 8-bit limbs of an offset
// 22-bit fixed-point value, so every "product" is still a sign-selected add (the tensor core
// does the adds) and the scales are applied once per row after accumulation.
//
// Data path per CTA (one persistent CTA per SM, a balanced contiguous range of
// (tile, slab) units, slab = 64 columns x 128 M-rows = 2 KB of WW_LAYOUT_TILE32 words):
//   * producer warp: cp.async.bulk of 8 KB weight stages into a shared-memory ring, issued
//     before griddepcontrol.wait (weights never depend on the previous kernel);
//   * decoder warps (4 per group, warp % 4 = TMEM lane quarter): one LDS.128 = 4 App. H words
//     of one M-row = 64 codes; each word -> 16 int8 by 4 PRMTs through the byte table
//     {0, -1, +1, 0} (codes 00, 01, 10, 11: bit 2k = -1, bit 2k+1 = +1, App. H P:597-604;
//     the unused (1,1) maps to 0, DESIGN R3); tcgen05.st of 16 columns into an A slot of
//     tensor memory (no shared-memory round trip for the expanded operand);
//   * x warps (4): after griddepcontrol.wait, max |x| per vector and component over all of
//     x, E = 20 - ilogb(max), u = bits(x 2^E + 1.5 2^23) & 0x7FFFFF = 2^22 + rint(x 2^E)
//     (the magic-number rounding of one fp32 add), its three bytes as the limbs of B in
//     shared memory (canonical K-major layout) plus a row of ones (sum_j T_ij, to remove the
//     2^22 offset exactly), for the slabs this CTA touches;
//   * MMA warp: tcgen05.mma.kind::i8 (A signed from TMEM, B unsigned from shared memory,
//     M = 128, N = 16 or 32, K = 32), int32 accumulation in TMEM (exact), double-buffered
//     accumulators per tile segment;
//   * epilogue (the x warps): tcgen05.ld, and per tile either the final epilogue (the CTA
//     owns the whole tile) or red.add of the int32 partial sums into a workspace slot; the
//     last CTA to arrive (counter) finishes the tile and leaves the workspace zeroed.
// Final epilogue per row: V = D2 2^16 + D1 2^8 + D0 - 2^22 D1s (exact in fp64), times 2^-E and
// the plane's scale, EQ1 / ALG1 signs, planes summed over four lanes, complex64 store.
// Integer sums are exact, so results do not depend on the grid, the split of a tile or the
// shard: the only rounding is x's grid (2^-E, about max|x| 2^-21) and fp64 -> fp32.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

#include "ww.h"
#include "ww_internal.h"

namespace {

constexpr int kSlabBytes = 2048;   // one (tile, slab) unit: 128 M-rows x 4 words
constexpr int kUnitsPerStage = 4;  // units per weight-ring stage (one 8 KB bulk copy)
constexpr int kStageBytes = kUnitsPerStage * kSlabBytes;
constexpr int kRing = 4;           // weight-ring stages (32 KB in flight per SM)
constexpr int kAStages = 6;        // A stages in tensor memory (4 units = 64 columns each)
constexpr int kXWarps = 4;         // x preparation, then the epilogue (TMEM lane quarters 0-3)
constexpr int kDecGroups = 2;      // decoder groups of 4 warps (one per TMEM lane quarter)
constexpr int kUnitsPerGroup = 2;  // consecutive units of a stage per group (one 32-column store)
constexpr int kDecWarps = 4 * kDecGroups;
constexpr int kProdWarp = kXWarps + kDecWarps;
constexpr int kMmaWarp = kProdWarp + 1;
constexpr int kThreads = 32 * (kMmaWarp + 1);
constexpr int kTmemCols = 512;     // one CTA per SM (the register file holds one anyway)
constexpr int kXThreads = 32 * kXWarps;
constexpr int kPWarps = kXWarps + kDecWarps;  // warps 0 .. kPWarps-1 prepare x together
constexpr int kPThreads = 32 * kPWarps;
constexpr int kMaxB = 4;

static_assert(kDecGroups * kUnitsPerGroup == kUnitsPerStage, "the groups cover a stage");

// --------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
// a converged warp waits with one polling lane (32 polling lanes per warp flood the shared
// memory pipe the working warps need); __syncwarp orders the other lanes after the acquire
__device__ __forceinline__ void mbar_wait_warp(uint32_t bar, uint32_t parity) {
    if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
    __syncwarp();
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* a, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
// one lane of a converged warp (elect.sync): the compiler then knows the lane is unique and the
// operands of the tcgen05 instructions it issues stay in uniform registers
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, 0xffffffff;\n\tselp.b32 %0, 1, 0, px;\n\t}"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void pbar() {  // named barrier of the x preparation (x + decoder warps)
    asm volatile("bar.sync 1, %0;" ::"n"(kPThreads) : "memory");
}

// UMMA shared-memory descriptor of the B operand: K-major, no swizzle, core matrices of
// 8 rows x 16 bytes, the two 16-byte K halves of a K = 32 step LBO = 128 B apart,
// consecutive 8-row groups SBO = 256 B apart; version 1 (sm_100)
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((256u >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
// instruction descriptor: kind::i8, D s32, A signed 8-bit, B unsigned 8-bit, K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int N) {
    return (2u << 4) | (1u << 7) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// D[tmem_d] (+)= A[tmem_a] . B[desc]^T: A (128 x 32 int8) read from tensor memory
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
template <int NB>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, int32_t (&v)[NB]);
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, int32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
template <>
__device__ __forceinline__ void tmem_ld<32>(uint32_t taddr, int32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// One App. H word (16 codes of one plane and row, bit 2k = -1, bit 2k+1 = +1) -> 16 int8 in
// the K order [0,2,4,6, 8,10,12,14, 1,3,5,7, 9,11,13,15] (the B operand uses the same order):
// the nibbles of w & 0x3333_3333 are the even codes, of (w >> 2) & 0x3333_3333 the odd ones,
// and PRMT with a nibble selector picks byte `code` of the table {0x00, 0xFF, 0x01, 0x00}.
__device__ __forceinline__ void decode_word(uint32_t w, uint32_t* o) {
    constexpr uint32_t kTable = 0x0001FF00u;
    const uint32_t e = w & 0x33333333u;
    const uint32_t d = (w >> 2) & 0x33333333u;
    o[0] = prmt(kTable, 0u, e);
    o[1] = prmt(kTable, 0u, e >> 16);
    o[2] = prmt(kTable, 0u, d);
    o[3] = prmt(kTable, 0u, d >> 16);
}

struct TcvParams {
    const uint8_t* packed;  // WW_LAYOUT_TILE32
    const float* scales;
    const float* X;         // B rows of m complex64, stride ldx
    float* Y;               // B rows of n complex64, stride ldy
    unsigned long long* ws; // [T][maxc][128][NB] flagged partial sums (zero between launches)
    int64_t n, m, ldx, ldy, U;
    int64_t maxc;           // workspace slots per tile (most contributing CTAs of a split tile)
    int32_t S, B, per_row, conv, nsl;
    unsigned long long* trace;  // tools only: globaltimer stamps of CTAs 0 and grid/2
    int32_t dbg;                // tools only (ww_debug_tcv_flags): 1 = skip the limb arithmetic,
                                // 2 = split tiles not reduced (wrong results), 4 = skip the x max
};

// wait-time accounting of CTA 0 (tools builds with -DWW_TCV_WAITSTATS only: the counters
// cost registers in the decoder loop)
#ifdef WW_TCV_WAITSTATS
#define WSTAT_DECL(v) long long v = 0
#define WSTAT_BEGIN() const long long wstat_t0 = clock64()
#define WSTAT_END(v) v += clock64() - wstat_t0
#define WSTAT_STORE(cond, slot, v) \
    if ((cond) && p.trace && blockIdx.x == 0) p.trace[slot] = (unsigned long long)(v)
#else
#define WSTAT_DECL(v)
#define WSTAT_BEGIN()
#define WSTAT_END(v)
#define WSTAT_STORE(cond, slot, v)
#endif

// event stamps (ns) of two CTAs for tools/tcv_trace.py (null in the product)
__device__ __forceinline__ void tstamp(const TcvParams& p, int ev) {
    if (!p.trace) return;
    const unsigned slot = blockIdx.x == 0 ? 0u : (blockIdx.x == gridDim.x / 2 ? 1u : 2u);
    if (slot > 1) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
    p.trace[slot * 32 + ev] = t;
}

// index of the CTA whose unit range [c U / G, (c+1) U / G) holds unit u
__device__ __forceinline__ int64_t owner(int64_t u, int64_t U, int64_t G) { return ((u + 1) * G - 1) / U; }

// the four x warps: this lane's M-row (row 8 warp + lane / 4 of the tile, plane lane % 4)
template <int NB>
__device__ __forceinline__ void finalize(const TcvParams& p, int64_t tile, const int32_t (&D)[NB],
                                         const int (&E)[2 * kMaxB], float sc, int warp, int lane) {
    const int pl = lane & 3;
    const int64_t row = tile * 32 + 8 * warp + (lane >> 2);
    const bool ok = row < p.n;
    const double s = (double)sc;
    const bool eq1 = p.conv == WW_CONV_EQ1;
    // the ones row: sum_j T_ij (compile-time register indices)
    const int32_t d1s = p.B == 1 ? D[6] : (p.B == 2 || NB == 16) ? D[12 % NB] : p.B == 3 ? D[18 % NB] : D[24 % NB];
    const double ones = (double)d1s;
#pragma unroll
    for (int b = 0; b < kMaxB; ++b) {
        if (b >= p.B) break;
        double S[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int k = 6 * b + 3 * c;
            // exact: |D| < 2^8 m, the recombined value < 2^53
            const double v = (double)D[k + 2] * 65536.0 + (double)D[k + 1] * 256.0 + (double)D[k] -
                             4194304.0 * ones;
            S[c] = v * __longlong_as_double((long long)(1023 - E[2 * b + c]) << 52) * s;  // 2^-E
        }
        // this plane's share of y (Eq. 1 / Eqs. 2-3 signs):
        // U_re: (re, im); U_im: (-im, re); W_re: (re, -+im); W_im: (im, +-re)
        double yre, yim;
        if (pl == 0) { yre = S[0]; yim = S[1]; }
        else if (pl == 1) { yre = -S[1]; yim = S[0]; }
        else if (pl == 2) { yre = S[0]; yim = eq1 ? -S[1] : S[1]; }
        else { yre = S[1]; yim = eq1 ? S[0] : -S[0]; }
        yre += __shfl_xor_sync(0xffffffffu, yre, 1);  // planes (0+1) + (2+3), fixed order
        yim += __shfl_xor_sync(0xffffffffu, yim, 1);
        yre += __shfl_xor_sync(0xffffffffu, yre, 2);
        yim += __shfl_xor_sync(0xffffffffu, yim, 2);
        if (pl == (b & 3) && ok)
            reinterpret_cast<float2*>(p.Y)[(int64_t)b * p.ldy + row] = make_float2((float)yre, (float)yim);
    }
}

template <int NB>
__global__ void __launch_bounds__(kThreads, 1) wl_tcv_kernel(const __grid_constant__ TcvParams p) {
    constexpr uint32_t kBSlab = (uint32_t)NB * 64;  // B operand bytes per slab (2 K-steps)
    constexpr uint32_t kA0 = 2 * NB;                // first TMEM column of the A stages
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* smem = smem_raw + (base - raw);
    const uint32_t ring = base;
    const uint32_t bop = ring + kRing * kStageBytes;
    const uint32_t xs = bop + (uint32_t)p.nsl * kBSlab;            // one x vector (8 m bytes)
    const uint32_t bars = xs + (uint32_t)((8 * p.m + 127) / 128 * 128);
    const uint32_t full = bars, empty = full + 8 * kRing, afull = empty + 8 * kRing;
    const uint32_t aempty = afull + 8 * kAStages, dfull = aempty + 8 * kAStages, dempty = dfull + 16;
    const uint32_t bready = dempty + 16, xfull = bready + 8;
    unsigned char* misc = smem + (xfull + 8 - base);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(misc);
    float* red = reinterpret_cast<float*>(misc + 16);           // [kPWarps][2]
    const float* xsp = reinterpret_cast<const float*>(smem + (xs - base));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t G = gridDim.x, U = p.U;
    const int64_t u0 = (int64_t)blockIdx.x * U / G, u1 = ((int64_t)blockIdx.x + 1) * U / G;
    const int nu = (int)(u1 - u0);
    const int S = p.S;
    const int s_first = (int)(u0 % S);
    const int nst = (nu + kUnitsPerStage - 1) / kUnitsPerStage;
    if (tid == 0) tstamp(p, 0);
    pdl_launch();

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    auto stage_bytes = [&](int st) -> uint32_t {
        const int c = nu - st * kUnitsPerStage;
        return (uint32_t)(c < kUnitsPerStage ? c : kUnitsPerStage) * kSlabBytes;
    };
    if (warp == kProdWarp && lane == 0) {
        for (int i = 0; i < kRing; ++i) {
            mbar_init(full + 8 * i, 1);
            mbar_init(empty + 8 * i, kDecWarps);
        }
        for (int i = 0; i < kAStages; ++i) {
            mbar_init(afull + 8 * i, kDecWarps);
            mbar_init(aempty + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(dfull + 8 * i, 1);
            mbar_init(dempty + 8 * i, kXWarps);
        }
        mbar_init(bready, 1);
        mbar_init(xfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the first stages stream in while the previous kernel finishes (PDL)
        for (int st = 0; st < kRing && st < nst; ++st) {
            mbar_expect_tx(full + 8 * st, stage_bytes(st));
            bulk_g2s(ring + st * kStageBytes, p.packed + (u0 + (int64_t)st * kUnitsPerStage) * kSlabBytes,
                     stage_bytes(st), full + 8 * st);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
    if (tid == 0) tstamp(p, 1);

    if (warp == kProdWarp) {
        // ---- producer: refill a ring stage once all decoder warps have read it
        if (lane == 0)
            for (int st = kRing; st < nst; ++st) {
                const int r = st % kRing;
                mbar_wait(empty + 8 * r, ((st / kRing) - 1) & 1);
                mbar_expect_tx(full + 8 * r, stage_bytes(st));
                bulk_g2s(ring + r * kStageBytes, p.packed + (u0 + (int64_t)st * kUnitsPerStage) * kSlabBytes,
                         stage_bytes(st), full + 8 * r);
            }
    } else if (warp == kMmaWarp) {
        // ---- MMA issuer: per A stage (4 units = 8 MMAs of K = 32) one wait and one commit;
        // accumulators double-buffered per tile segment (this CTA's units of one tile).  The
        // whole warp runs the loop (its state stays warp-uniform, in uniform registers) and one
        // elected lane issues the tcgen05 instructions.
        {
            mbar_wait_warp(bready, 0);
            tc_fence_after();
            if (lane == 0) tstamp(p, 5);
            constexpr uint32_t idesc = idesc_i8(NB);
            const bool leader = elect_one();
#define MMA(d, a, b, acc)                      \
    do {                                       \
        if (leader) mma_ts(d, a, b, idesc, acc); \
    } while (0)
            int seg = 0, s = s_first, sl = 0;
            bool first = true;
            WSTAT_DECL(mma_wait);
            const int nas = (nu + kUnitsPerStage - 1) / kUnitsPerStage;
            for (int k = 0; k < nas; ++k) {
                const int as = k % kAStages;
                WSTAT_BEGIN();
                mbar_wait_warp(afull + 8 * as, (uint32_t)(k / kAStages) & 1);
                WSTAT_END(mma_wait);
                tc_fence_after();
                const uint32_t ta0 = tmem + kA0 + (uint32_t)(as * 64);
                // fast path (no segment ends, four units): straight-line MMAs and one commit --
                // UTC instructions under runtime branches make ptxas serialise their issue
                const int i0 = k * kUnitsPerStage;
#ifdef WW_TCV_NOFAST
                const bool fast = false;
#else
                const bool fast = i0 + kUnitsPerStage < nu && s + kUnitsPerStage < S && sl + kUnitsPerStage <= S &&
                                  !(first && seg >= 2);
#endif
                if (fast) {
                    const uint32_t td = tmem + (uint32_t)(NB * (seg & 1));
                    const uint64_t bd = bdesc(bop + (uint32_t)sl * kBSlab);
#pragma unroll
                    for (int j = 0; j < kUnitsPerStage; ++j) {
                        const uint64_t bj = bd + (uint64_t)(j * (kBSlab / 16));
                        MMA(td, ta0 + 16u * j, bj, (j == 0 && first) ? 0u : 1u);
                        MMA(td, ta0 + 16u * j + 8u, bj + (uint64_t)(NB * 32 / 16), 1u);
                    }
                    if (leader) mma_commit(aempty + 8 * as);
                    first = false;
                    s += kUnitsPerStage;  // s + 4 < S: no wrap
                    sl += kUnitsPerStage;
                    if (sl == S) sl = 0;
                } else {
#pragma unroll 1
                    for (int j = 0; j < kUnitsPerStage; ++j) {
                        const int i = i0 + j;
                        if (i >= nu) break;
                        const bool last = i == nu - 1 || s == S - 1;
                        const int db = seg & 1;
                        if (first && seg >= 2) {
                            mbar_wait_warp(dempty + 8 * db, (uint32_t)((seg >> 1) - 1) & 1);
                            tc_fence_after();
                        }
                        const uint64_t bd = bdesc(bop + (uint32_t)sl * kBSlab);
                        const uint32_t ta = ta0 + 16u * j;
                        MMA(tmem + (uint32_t)(NB * db), ta, bd, first ? 0u : 1u);
                        MMA(tmem + (uint32_t)(NB * db), ta + 8u, bd + (uint64_t)(NB * 32 / 16), 1u);
                        if (last) {
                            if (leader) mma_commit(dfull + 8 * db);
                            ++seg;
                        }
                        first = last;
                        s = s == S - 1 ? 0 : s + 1;
                        sl = sl == S - 1 ? 0 : sl + 1;
                    }
                    if (leader) mma_commit(aempty + 8 * as);
                }
                __syncwarp();
                if (k == 0 && leader) tstamp(p, 6);
            }
            if (leader) tstamp(p, 7);
            WSTAT_STORE(leader, 24, mma_wait);
        }
    } else {
        // ---- x preparation, shared by the x warps and (after they have filled the A stages)
        // the decoder warps: x_b staged in shared memory, max |x| per component, E, and the
        // fixed-point limbs of the slabs this CTA touches (B operand rows 6 b + 3 comp + limb,
        // row 6B = ones, rows above = 0)
        const int B = p.B;
        const int nslc = nu < S ? nu : S;
        int E[2 * kMaxB];
        auto x_prepare = [&]() {
            const uint32_t xbytes = (uint32_t)(8 * p.m) & ~15u;
            const bool bulk = (((uintptr_t)p.X | (uintptr_t)(p.ldx * 8)) & 15) == 0;
#pragma unroll 1
            for (int b = 0; b < B; ++b) {
                const float* xg = p.X + 2 * (int64_t)b * p.ldx;
                if (b > 0) pbar();  // every thread is done with x_{b-1}
                if (bulk) {
                    if (tid == 0) {  // an x warp, after griddepcontrol.wait
                        mbar_expect_tx(xfull, xbytes);
                        if (xbytes) bulk_g2s(xs, xg, xbytes, xfull);
                    }
                    mbar_wait_warp(xfull, (uint32_t)b & 1);
                    if (tid == 0 && b == 0) tstamp(p, 21);
                    if (tid == kXThreads && b == 0) tstamp(p, 23);  // first decoder thread
                    if (p.m & 1) {  // the odd tail element
                        if (tid == 1)
                            *reinterpret_cast<float2*>(smem + (xs - base) + 8 * (p.m - 1)) =
                                reinterpret_cast<const float2*>(xg)[p.m - 1];
                        pbar();
                    }
                } else {
                    if (tid < kXThreads)  // griddepcontrol.wait was executed by these threads
                        for (int64_t j = tid; j < p.m; j += kXThreads)
                            *reinterpret_cast<float2*>(smem + (xs - base) + 8 * j) =
                                reinterpret_cast<const float2*>(xg)[j];
                    pbar();
                }
                float mr = 0.f, mi = 0.f;
                for (int64_t j = tid; j < ((p.dbg & 4) ? 0 : (p.m + 1) / 2); j += kPThreads) {
                    const float4 v = reinterpret_cast<const float4*>(xsp)[j];
                    const bool two = 2 * j + 1 < p.m;
                    mr = fmaxf(mr, fmaxf(fabsf(v.x), two ? fabsf(v.z) : 0.f));
                    mi = fmaxf(mi, fmaxf(fabsf(v.y), two ? fabsf(v.w) : 0.f));
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
                    mi = fmaxf(mi, __shfl_xor_sync(0xffffffffu, mi, o));
                }
                if (lane == 0) {
                    red[2 * warp] = mr;
                    red[2 * warp + 1] = mi;
                }
                pbar();
                if (tid == 0 && b == 0) tstamp(p, 22);
                const long long ck0 = clock64();
                float f1[2], f2[2];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float v = 0.f;
                    for (int w = 0; w < kPWarps; ++w) v = fmaxf(v, red[2 * w + c]);
                    // |rint(x 2^E)| <= 2^21: u = 2^22 + q stays in [0, 2^23) (one fp32 binade)
                    const int e = v > 0.f ? 20 - ilogbf(v) : 0;
#pragma unroll
                    for (int bb = 0; bb < kMaxB; ++bb)
                        if (bb == b) E[2 * bb + c] = e;
                    f1[c] = ldexpf(1.0f, e / 2);  // 2^E as two exact power-of-two factors
                    f2[c] = ldexpf(1.0f, e - e / 2);
                }
                if (tid == 0 && b == 0 && p.trace) p.trace[17] = (unsigned long long)(clock64() - ck0);
                for (int it = tid; it < ((p.dbg & 1) ? 0 : nslc * 4); it += kPThreads) {
                    const int sl = it >> 2, g16 = it & 3;
                    int s = s_first + sl;
                    if (s >= S) s -= S;
                    const int64_t col0 = (int64_t)s * 64 + g16 * 16;
                    const uint32_t dst = bop + (uint32_t)sl * kBSlab + (uint32_t)(g16 >> 1) * (NB * 32) +
                                         (uint32_t)(g16 & 1) * 128u;
                    float2 v[16];
                    if (tid == 0) tstamp(p, 19);
                    if (col0 + 16 <= p.m) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const float4 t = reinterpret_cast<const float4*>(xsp + 2 * col0)[k];
                            v[2 * k] = make_float2(t.x, t.y);
                            v[2 * k + 1] = make_float2(t.z, t.w);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            v[k] = col0 + k < p.m ? reinterpret_cast<const float2*>(xsp)[col0 + k]
                                                  : make_float2(0.f, 0.f);
                    }
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t u[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const float xv = c ? v[k].y : v[k].x;
                            u[k] = __float_as_uint(__fadd_rn(__fmul_rn(__fmul_rn(xv, f1[c]), f2[c]), 12582912.0f));
                        }
#pragma unroll
                        for (int l = 0; l < 3; ++l) {
                            const uint32_t sel = (uint32_t)l | ((uint32_t)(4 + l) << 4);
                            // K order [0,2,4,6 | 8,10,12,14 | 1,3,5,7 | 9,11,13,15] (decode_word)
                            const uint32_t w0 = prmt(prmt(u[0], u[2], sel), prmt(u[4], u[6], sel), 0x5410u);
                            const uint32_t w1 = prmt(prmt(u[8], u[10], sel), prmt(u[12], u[14], sel), 0x5410u);
                            const uint32_t w2 = prmt(prmt(u[1], u[3], sel), prmt(u[5], u[7], sel), 0x5410u);
                            const uint32_t w3 = prmt(prmt(u[9], u[11], sel), prmt(u[13], u[15], sel), 0x5410u);
                            const int nrow = 6 * b + 3 * c + l;
                            sts128(dst + (uint32_t)(nrow >> 3) * 256u + (uint32_t)(nrow & 7) * 16u, w0, w1, w2, w3);
                        }
                        if (tid == 0) tstamp(p, 30 + c);
                    }
                    if (b == B - 1)  // the ones row (sum_j T_ij) and the unused rows
                        for (int nrow = 6 * B; nrow < NB; ++nrow) {
                            const uint32_t f = nrow == 6 * B ? 0x01010101u : 0u;
                            sts128(dst + (uint32_t)(nrow >> 3) * 256u + (uint32_t)(nrow & 7) * 16u, f, f, f, f);
                        }
                }
            }
            if (tid == 0) tstamp(p, 28);
            // generic -> async proxy, by the threads that wrote B-operand rows only (the fence
            // is expensive when hundreds of threads issue it at once)
            if (tid < nslc * 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (tid == 0) tstamp(p, 29);
            pbar();
            if (tid == 0) {
                tstamp(p, 3);
                mbar_arrive(bready);
            }
        };

        if (warp >= kXWarps) {
            // ---- decoders: unit i of this CTA goes to group i % 4 (A stage i / 4, slot i % 4);
            // a warp's lanes are the 32 M-rows of its TMEM lane quarter.  Groups arrive for
            // the missing units of a partial last stage too (the A-stage barrier counts 16).
            const int dw = warp - kXWarps, g = dw >> 2, q = warp & 3;
            const int nas = (nu + kUnitsPerStage - 1) / kUnitsPerStage;
            WSTAT_DECL(wfull);
            WSTAT_DECL(wempty);
            // the TMEM store of stage k completes (tcgen05.wait::st) while stage k+1 decodes;
            // its A-stage arrival follows the wait
            int pend = -1;  // A stage whose arrival is pending
            auto flush = [&]() {
                if (pend >= 0) {
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(afull + 8 * pend);
                    pend = -1;
                }
            };
            uint32_t o[2][32];
            auto decode_stage = [&](int k, uint32_t (&ob)[32]) {
                const int i = k * kUnitsPerStage + kUnitsPerGroup * g;  // units i, i+1
                const int as = k % kAStages;
                const bool have = i < nu;
                if (have) {
                    const int r = k % kRing;  // ring stage k holds units 4k .. 4k+3 (= A stage k)
                    WSTAT_BEGIN();
                    mbar_wait_warp(full + 8 * r, (uint32_t)(k / kRing) & 1);
                    WSTAT_END(wfull);
                    const uint32_t src = ring + r * kStageBytes + (uint32_t)(kUnitsPerGroup * g) * kSlabBytes +
                                         (uint32_t)(32 * q + lane) * 16u;
                    const uint4 w0 = lds128(src);
                    const uint4 w1 = i + 1 < nu ? lds128(src + kSlabBytes) : make_uint4(0, 0, 0, 0);
                    decode_word(w0.x, ob);
                    decode_word(w0.y, ob + 4);
                    decode_word(w0.z, ob + 8);
                    decode_word(w0.w, ob + 12);
                    decode_word(w1.x, ob + 16);
                    decode_word(w1.y, ob + 20);
                    decode_word(w1.z, ob + 24);
                    decode_word(w1.w, ob + 28);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + 8 * r);
                }
                flush();  // the previous stage's store has had this decode to complete
                if (k >= kAStages) {
                    WSTAT_BEGIN();
                    mbar_wait_warp(aempty + 8 * as, (uint32_t)((k / kAStages) - 1) & 1);
                    WSTAT_END(wempty);
                    tc_fence_after();
                }
                if (have)
                    tmem_st32(tmem + ((uint32_t)(32 * q) << 16) + kA0 + (uint32_t)(as * 64 + 16 * kUnitsPerGroup * g), ob);
                pend = as;
                if (warp == kXWarps && lane == 0 && k == 0) tstamp(p, 8);
                if (warp == kXWarps && lane == 0 && k == nas - 1) tstamp(p, 9);
            };
            auto x_landed = [&]() {  // non-blocking test of the first x copy
                uint32_t done;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                    "selp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(done)
                    : "r"(xfull)
                    : "memory");
                return __shfl_sync(0xffffffffu, done, 0) != 0;
            };
            const int pre = nas < kAStages ? nas : kAStages;
            int k = 0;
            for (; k < pre; ++k) {
                if (k > 0 && x_landed()) break;  // join the x preparation as soon as x is there
                decode_stage(k, o[k & 1]);
            }
            flush();
            x_prepare();
            for (; k + 1 < nas; k += 2) {
                decode_stage(k, o[0]);
                decode_stage(k + 1, o[1]);
            }
            if (k < nas) decode_stage(k, o[0]);
            flush();
            WSTAT_STORE(warp == kXWarps && lane == 0, 25, wfull);
            WSTAT_STORE(warp == kXWarps && lane == 0, 26, wempty);
            WSTAT_STORE(warp == kXWarps && lane == 0, 27, nas);
        } else {
            pdl_wait();  // x, scales, y and the workspace may belong to the previous kernel
            if (tid == 0) tstamp(p, 2);
            x_prepare();
            if (tid == 0) tstamp(p, 4);

            // ---- epilogue, one tile segment at a time.  A tile split across CTAs c0 < ... < c1
            // is finished by c0 (for which it is the LAST segment): c0+1 .. c1 publish their
            // exact int32 partial sums as flagged 64-bit words (value | 1 << 32) in their own
            // workspace slot, normally early (their FIRST segment); c0 polls the words (one
            // round trip once they are there), adds them to its own sums, finishes the tile
            // and zeroes the words for the next launch.
            int seg = 0;
            const int cols = 6 * B + 1;
            for (int64_t u = u0; u < u1; ++seg) {
                const int64_t t = u / S;
                const int64_t e = u1 < (t + 1) * S ? u1 : (t + 1) * S;
                const int db = seg & 1;
                const int64_t c0 = owner(t * S, U, G), c1 = owner((t + 1) * S - 1, U, G);
                // the scale of this lane's row, loaded before the accumulators are ready
                const int pl = lane & 3;
                const int64_t row = t * 32 + 8 * warp + (lane >> 2);
                const float sc = row < p.n ? p.scales[p.per_row ? 4 * row + pl : pl] : 0.f;
                mbar_wait_warp(dfull + 8 * db, (uint32_t)(seg >> 1) & 1);
                tc_fence_after();
                if (tid == 0 && seg < 4) tstamp(p, 10 + 2 * seg);
                int32_t D[NB];
                tmem_ld<NB>(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(NB * db), D);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(dempty + 8 * db);
                const int mr = 32 * warp + lane;
                if (c0 == c1 || (p.dbg & 2)) {
                    finalize<NB>(p, t, D, E, sc, warp, lane);
                } else if ((int64_t)blockIdx.x != c0) {
                    unsigned long long* w =
                        p.ws + ((t * p.maxc + ((int64_t)blockIdx.x - c0 - 1)) * 128 + mr) * NB;
#pragma unroll
                    for (int k = 0; k < NB; ++k)
                        if (k < cols) st_relaxed64(w + k, (1ull << 32) | (uint32_t)D[k]);
                } else {
                    // 8 columns x every contributor slot (at most 4 in flight per column) polled
                    // together: every not-yet-flagged word re-polled in the same pass (one round
                    // trip per pass); bounded: a workspace that was not zeroed fails loudly
                    const int nj = (int)(c1 - c0);
#pragma unroll
                    for (int k0 = 0; k0 < NB; k0 += 8) {
                        if (k0 < cols) {
                            for (int j0 = 0; j0 < nj; j0 += 4) {
                                unsigned long long v[4][8];
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                                    for (int k = 0; k < 8; ++k)
                                        v[jj][k] = (j0 + jj < nj && k0 + k < cols)
                                                       ? ld_relaxed64(p.ws + ((t * p.maxc + j0 + jj) * 128 + mr) * NB + k0 + k)
                                                       : (1ull << 32);
                                for (long long pass = 0;; ++pass) {
                                    bool all = true;
#pragma unroll
                                    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                                        for (int k = 0; k < 8; ++k) all = all && (v[jj][k] >> 32) != 0;
                                    if (all) break;
                                    if (pass > (1ll << 24)) __trap();
#pragma unroll
                                    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                                        for (int k = 0; k < 8; ++k)
                                            if ((v[jj][k] >> 32) == 0)
                                                v[jj][k] = ld_relaxed64(p.ws + ((t * p.maxc + j0 + jj) * 128 + mr) * NB + k0 + k);
                                }
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                                    for (int k = 0; k < 8; ++k)
                                        if (j0 + jj < nj && k0 + k < cols) {
                                            D[k0 + k] += (int32_t)(uint32_t)v[jj][k];
                                            p.ws[((t * p.maxc + j0 + jj) * 128 + mr) * NB + k0 + k] = 0ull;
                                        }
                            }
                        }
                    }
                    finalize<NB>(p, t, D, E, sc, warp, lane);
                }
                if (tid == 0 && seg < 4) tstamp(p, 11 + 2 * seg);
                u = e;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) tstamp(p, 20);
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols)
                     : "memory");
}

// ------------------------------------------------------------------ device packer (TILE32)
// one output word per thread: App. H word wi of plane p, row i, from the dense int8 planes
__global__ void pack_tile32_kernel(const int8_t* __restrict__ planes, int64_t n, int64_t m, int64_t ld,
                                   int64_t S, int64_t total, uint32_t* __restrict__ out,
                                   int32_t* __restrict__ bad) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t wi4 = x & 3, mr = (x >> 2) & 127, ts = x >> 9;
        const int64_t t = ts / S, s = ts % S;
        const int64_t i = t * 32 + (mr >> 2);
        const int p = (int)(mr & 3);
        const int64_t j0 = (s * 4 + wi4) * 16;
        uint32_t word = 0;
        bool badw = false;
        if (i < n)
            for (int k = 0; k < 16; ++k) {
                const int64_t j = j0 + k;
                if (j >= m) break;
                const int v = planes[((int64_t)p * n + i) * ld + j];
                if (v == 1) word |= 2u << (2 * k);
                else if (v == -1) word |= 1u << (2 * k);
                else if (v != 0) badw = true;
            }
        if (badw) {
            word = 0;
            if (bad) atomicOr(bad, 1);
        }
        out[x] = word;
    }
}

template <int NB>
size_t tcv_smem(int nsl, int64_t m) {
    return (size_t)kRing * kStageBytes + (size_t)nsl * NB * 64 + (size_t)((8 * m + 127) / 128 * 128) +
           8 * (2 * kRing + 2 * kAStages + 6) + 16 + 4 * kPWarps * 2 + 16 + 1024;
}

template <int NB>
cudaError_t launch_tcv(const TcvParams& p, int grid, cudaStream_t s, bool pdl) {
    const size_t smem = tcv_smem<NB>(p.nsl, p.m);
    const int pe = ww::prepare_kernel(reinterpret_cast<const void*>(wl_tcv_kernel<NB>), 227 * 1024);
    if (pe) return (cudaError_t)pe;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, wl_tcv_kernel<NB>, p);
}

inline int tcv_nb(int B) { return B <= 2 ? 16 : 32; }

// work decomposition of a launch: T tiles x S slabs = U units over G CTAs (balanced
// contiguous ranges); maxc = the most CTAs contributing to one split tile besides its first
struct TcvGeom {
    int64_t T, S, U, G, maxc;
};
TcvGeom tcv_geom(int64_t n, int64_t m) {
    TcvGeom g;
    g.T = ww::tile32_tiles(n);
    g.S = ww::tile32_slabs(m);
    g.U = g.T * g.S;
    const int64_t sms = ww::device_sms();
    g.G = g.U < sms ? g.U : sms;
    auto own = [&](int64_t u) { return ((u + 1) * g.G - 1) / g.U; };
    int64_t mx = 1;
    if (g.T <= (1 << 20)) {
        for (int64_t t = 0; t < g.T; ++t) {
            const int64_t c = own((t + 1) * g.S - 1) - own(t * g.S);
            if (c > mx) mx = c;
        }
    } else {
        mx = (g.S + g.U / g.G - 1) / (g.U / g.G) + 1;
    }
    g.maxc = mx;
    return g;
}

unsigned long long* g_tcv_trace = nullptr;
int g_tcv_dbg = 0;

}  // namespace

// Not part of the ABI: tools point CTAs 0 and grid/2 of wl_tcv_kernel at a trace buffer.
extern "C" void ww_debug_tcv_trace(void* buf) { g_tcv_trace = reinterpret_cast<unsigned long long*>(buf); }
// Not part of the ABI: ablation switches of wl_tcv_kernel for tools (see TcvParams::dbg).
extern "C" void ww_debug_tcv_flags(int f) { g_tcv_dbg = f; }

extern "C" size_t ww_tcv_workspace_bytes(int64_t n, int64_t m, int32_t B) {
    if (n < 1 || m < 1 || B < 1 || B > kMaxB) return 0;
    const TcvGeom g = tcv_geom(n, m);
    return (size_t)g.T * (size_t)g.maxc * 128u * (size_t)tcv_nb(B) * 8u;
}

extern "C" ww_status ww_pack_ternary_device_layout(const int8_t* planes_d, int64_t n, int64_t m, int64_t ld,
                                                   int32_t layout, uint32_t* out_d, int32_t* bad_d,
                                                   void* stream) {
    const char* fn = "ww_pack_ternary_device_layout";
    if (layout == WW_LAYOUT_COL4) return ww_pack_ternary_device(planes_d, n, m, ld, out_d, bad_d, stream);
    if (layout != WW_LAYOUT_TILE32 && layout != WW_LAYOUT_LUT81)
        return ww::fail(WW_ERR_UNSUPPORTED, "%s: layout %d", fn, layout);
    if (!planes_d || !out_d) return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: null pointer", fn);
    if (n < 1 || m < 1 || ld < m)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: n=%lld m=%lld ld=%lld", fn, (long long)n, (long long)m,
                        (long long)ld);
    if ((uintptr_t)out_d & 15) return ww::fail(WW_ERR_MISALIGNED, "%s: out must be 16-B aligned", fn);
    if (layout == WW_LAYOUT_LUT81) {
        const int el = ww::pack_lut81_device(planes_d, n, m, ld, out_d, bad_d, stream);
        if (el) return ww::fail(WW_ERR_CUDA, "%s: %s", fn, cudaGetErrorString((cudaError_t)el));
        return ww::ok();
    }
    const int64_t S = ww::tile32_slabs(m);
    const int64_t total = ww::tile32_tiles(n) * S * 512;
    pack_tile32_kernel<<<ww::device_sms() * 8, 256, 0, (cudaStream_t)stream>>>(planes_d, n, m, ld, S, total,
                                                                            out_d, bad_d);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return ww::fail(WW_ERR_CUDA, "%s: %s", fn, cudaGetErrorString(e));
    return ww::ok();
}

extern "C" ww_status ww_wl_gemv_tc(const ww_layer* L, const void* packed_d, const float* scales_d,
                                   const float* X_d, int64_t ldx, float* Y_d, int64_t ldy, int32_t B,
                                   void* workspace_d, void* stream) {
    const char* fn = "ww_wl_gemv_tc";
    if (!L || !packed_d || !scales_d || !X_d || !Y_d || !workspace_d)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: null pointer", fn);
    if (L->n < 1 || L->m < 1 || L->n > ((int64_t)1 << 31) || L->m > ((int64_t)1 << 24))
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: n=%lld m=%lld", fn, (long long)L->n, (long long)L->m);
    if (L->layout != WW_LAYOUT_TILE32) return ww::fail(WW_ERR_UNSUPPORTED, "%s: needs WW_LAYOUT_TILE32", fn);
    if (L->conv != WW_CONV_EQ1 && L->conv != WW_CONV_ALG1)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: conv %d", fn, L->conv);
    if (L->scale_mode != WW_SCALES_PER_ROW && L->scale_mode != WW_SCALES_PER_TENSOR)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: scale mode %d", fn, L->scale_mode);
    if (B < 1) return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: B=%d", fn, B);
    if (B > kMaxB) return ww::fail(WW_ERR_UNSUPPORTED, "%s: B=%d (1..%d)", fn, B, kMaxB);
    if (ldx < L->m || ldy < L->n)
        return ww::fail(WW_ERR_DIMENSION_MISMATCH, "%s: ldx=%lld ldy=%lld", fn, (long long)ldx, (long long)ldy);
    if (((uintptr_t)packed_d & 15) || ((uintptr_t)X_d & 7) || ((uintptr_t)Y_d & 7) ||
        ((uintptr_t)scales_d & 3) || ((uintptr_t)workspace_d & 15))
        return ww::fail(WW_ERR_MISALIGNED, "%s: packed / workspace 16-B, x / y 8-B aligned", fn);
    const char* xb = reinterpret_cast<const char*>(X_d);
    const char* yb = reinterpret_cast<const char*>(Y_d);
    if (xb < yb + 8 * (ldy * (B - 1) + L->n) && yb < xb + 8 * (ldx * (B - 1) + L->m))
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: x and y overlap", fn);
    TcvParams p;
    memset(&p, 0, sizeof p);
    const TcvGeom geo = tcv_geom(L->n, L->m);
    p.packed = reinterpret_cast<const uint8_t*>(packed_d);
    p.scales = scales_d;
    p.X = X_d;
    p.Y = Y_d;
    p.n = L->n;
    p.m = L->m;
    p.ldx = ldx;
    p.ldy = ldy;
    p.S = (int32_t)geo.S;
    p.U = geo.U;
    p.maxc = geo.maxc;
    p.B = B;
    p.per_row = L->scale_mode == WW_SCALES_PER_ROW;
    p.conv = L->conv;
    p.trace = g_tcv_trace;
    p.dbg = g_tcv_dbg;
    const int NB = tcv_nb(B);
    p.ws = reinterpret_cast<unsigned long long*>(workspace_d);
    const int grid = (int)geo.G;
    const int64_t per = (p.U + grid - 1) / grid;  // most units a CTA owns
    p.nsl = (int32_t)(per < p.S ? per : p.S);
    const size_t smem = NB == 16 ? tcv_smem<16>(p.nsl, p.m) : tcv_smem<32>(p.nsl, p.m);
    if (smem > 227 * 1024)
        return ww::fail(WW_ERR_UNSUPPORTED, "%s: m=%lld needs %zu B of shared memory", fn, (long long)L->m, smem);
    const bool pdl = (L->flags & WW_FLAG_PDL) != 0;
    cudaError_t e = NB == 16 ? launch_tcv<16>(p, grid, (cudaStream_t)stream, pdl)
                             : launch_tcv<32>(p, grid, (cudaStream_t)stream, pdl);
    if (e != cudaSuccess) return ww::fail(WW_ERR_CUDA, "%s: %s", fn, cudaGetErrorString(e));
    return ww::ok();
}
