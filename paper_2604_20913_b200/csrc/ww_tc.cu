// Batched WL-GEMV on the 5th-generation tensor cores (tcgen05, kind::i8) for the small-batch
// variant (a9, BASELINE config 5): with B vectors the layer IS a dense contraction
// Y[n x 2B] <- T[4n x m] . X[m x 2B] (T: the four ternary planes stacked per row), so for
// B >= 8 the sign-selected adds of the per-vector path are replaced by exact integer MMAs:
//   * T is decoded in-kernel from the packed COL4 codes (2 bits per code, read once from HBM)
//     into signed int8 {-1, 0, +1} tiles in shared memory (K-major, no swizzle, the UMMA
//     canonical layout) -- the only expansion of the codes, never written to HBM;
//   * each x component is split once per launch into three signed 8-bit limbs of a 22-bit
//     fixed-point value (x = 2^-E (l2 2^16 + l1 2^8 + l0), E per vector and component,
//     ww_tc_limbs_kernel) laid out in the same canonical layout;
//   * tcgen05.mma kind::i8 accumulates D[(row, plane), (vector, component, limb)] in int32 in
//     tensor memory -- every product is t * limb with t in {-1, 0, +1} and the sums are exact;
//   * the epilogue (tcgen05.ld) recombines the limbs exactly in fp64, applies the scales once
//     per row with the EQ1 / ALG1 signs, reduces the four planes of a
//     row across four lanes and stores complex64.
// The only rounding is x's 22-bit fixed-point grid (relative to max |x| of that vector and
// component) and the final fp64 -> fp32 conversion, well inside the north-star bar.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "ww.h"
#include "ww_internal.h"

namespace {

constexpr int kTM = 128;      // MMA M: 32 output rows x 4 planes
constexpr int kRows = 32;     // output rows per CTA tile
constexpr int kKB = 256;      // K columns per pipeline block (8 MMAs of K = 32)
constexpr int kDecodeWarps = 16;  // decode warps: one 16-column chunk of one row per thread
                                  // and block (warps 0-3 also run the epilogue)
constexpr int kThreads = (kDecodeWarps + 1) * 32;  // + one MMA / limb-producer warp
constexpr int kLimbs = 3;
constexpr int kSlab32 = 2048;  // WW_LAYOUT_TILE32: one (32-row tile, 64-column slab) unit
constexpr int kMaxB = 16;      // 2B (vector, component) columns per limb group of 32
constexpr int kStages = 3;     // A decode slots (and packed words in flight per thread)
constexpr int kBStages = 4;    // limb slots
constexpr int kLag = 2;        // a limb slot is refilled kLag iterations after its MMAs were issued

// accumulator columns: limb-major, n = k * LW + (2 b + comp), LW = 16 or 32 columns per limb
// (2B <= 32: B <= 16), so the epilogue finds each limb of every (vector, component) in one
// 32-column TMEM load at a compile-time register index
__host__ __device__ inline int tc_lw(int B) { return 2 * B <= 16 ? 16 : 32; }
__host__ __device__ inline int tc_n(int B) { return kLimbs * tc_lw(B); }
__host__ __device__ inline int64_t tc_kpad(int64_t m) { return (m + kKB - 1) / kKB * kKB; }

// --------------------------------------------------------------------------- PTX helpers
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
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
// cluster helpers (split tiles): all threads of every CTA of the cluster
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, int32_t a, int32_t b, int32_t c, int32_t d) {
    asm volatile("st.shared::cluster.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle (canonical ((8,n),2):((16 B, SBO), LBO)):
// 8-row core matrices of 16 bytes, the two 16-byte K halves of a K = 32 step LBO = 128 B
// apart, consecutive 8-row groups SBO = 256 B apart; version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((256u >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
// instruction descriptor: kind::i8, D = s32, A and B signed 8-bit, both K-major, M = 128
__host__ __device__ inline uint32_t umma_idesc_i8(int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 32 lanes x 32 columns of 32-bit: thread i of the warp gets lane (base + i), columns c..c+31
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t (&v)[32]) {
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

// canonical byte offset of element (row n, column k) of an operand with N rows, K-major
__host__ __device__ inline int64_t canon_off(int N, int64_t n, int64_t k) {
    const int64_t s = k >> 5, h = (k >> 4) & 1, c = k & 15;
    return s * (int64_t)N * 32 + (n >> 3) * 256 + h * 128 + (n & 7) * 16 + c;
}

// ------------------------------------------------------------------ x -> fixed-point limbs
// block (b, comp) < 2B: E = 21 - floor(log2 max |x|), q = rint(x 2^E) (|q| < 2^22, an exact
// power-of-two scaling), balanced signed 8-bit limbs q = l2 2^16 + l1 2^8 + l0 written to
// rows (2b + comp) * 3 + k of the canonical B operand; the last block zero-fills the pad rows
// one block per (vector b, component): x component staged in shared memory by all threads
// (coalesced, one round of loads), E = 21 - floor(log2 max |x|), q = rint(x 2^E) (|q| < 2^22,
// exact power-of-two scaling), balanced signed 8-bit limbs q = l2 2^16 + l1 2^8 + l0 written
// as 16-byte core-matrix rows to rows k * LW + (2b + comp) of the canonical B operand; the
// last block zero-fills the unused rows (2B .. LW-1 of every limb group)
constexpr int kLimbThreads = 1024;
constexpr int kLimbMaxM = 11264;  // x component in shared memory (44 KB)
__global__ void __launch_bounds__(kLimbThreads) tc_limbs_kernel(const float* __restrict__ X, int64_t ldx,
                                                                int B, int64_t m, int64_t kpad, int N,
                                                                int8_t* __restrict__ limbs,
                                                                int* __restrict__ expo) {
    __shared__ float xs[kLimbMaxM];
    __shared__ float red[kLimbThreads / 32];
    // the MMA kernel (launched as a programmatic dependent) starts decoding weights now; it
    // waits (griddepcontrol.wait) before it reads the limbs or the exponents
    asm volatile("griddepcontrol.launch_dependents;" :::);
    const int bc = blockIdx.x, LW = N / kLimbs;
    const int64_t ng = kpad / 16;  // 16-column groups: one 16-byte core-matrix row each
    if (bc == 2 * B) {
        const int pad = LW - 2 * B;
        for (int64_t e = threadIdx.x; e < (int64_t)kLimbs * pad * ng; e += blockDim.x) {
            const int64_t rowi = e / ng, g = e % ng;
            const int64_t n = (rowi / pad) * LW + 2 * B + rowi % pad;
            *reinterpret_cast<uint4*>(limbs + canon_off(N, n, 16 * g)) = make_uint4(0, 0, 0, 0);
        }
        return;
    }
    const int b = bc >> 1, comp = bc & 1;
    const float* xb = X + 2 * (int64_t)b * ldx + comp;
    float mx = 0.f;
    for (int64_t j = threadIdx.x; j < kpad; j += blockDim.x) {
        const float v = j < m ? xb[2 * j] : 0.f;
        xs[j] = v;
        mx = fmaxf(mx, fabsf(v));
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
    const int E = mx > 0.f ? 21 - ilogbf(mx) : 0;
    if (threadIdx.x == 0) expo[bc] = E;
    // 2^E as two exact power-of-two factors (E in about [-100, 150] for finite nonzero x)
    const float f1 = ldexpf(1.0f, E / 2), f2 = ldexpf(1.0f, E - E / 2);
    for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) {
        uint32_t L[kLimbs][4] = {};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int32_t q = __float2int_rn((xs[16 * g + i] * f1) * f2);
            const int32_t l0 = (int32_t)(int8_t)(q & 0xff);
            const int32_t q1 = (q - l0) >> 8;
            const int32_t l1 = (int32_t)(int8_t)(q1 & 0xff);
            const int32_t l2 = (q1 - l1) >> 8;
            // column i of the group sits at K position kp of the decoded A rows (decode_word)
            const int kp = (i & 1) ? 8 + (i >> 1) : (i >> 1);
            L[0][kp >> 2] |= ((uint32_t)l0 & 0xffu) << (8 * (kp & 3));
            L[1][kp >> 2] |= ((uint32_t)l1 & 0xffu) << (8 * (kp & 3));
            L[2][kp >> 2] |= ((uint32_t)l2 & 0xffu) << (8 * (kp & 3));
        }
#pragma unroll
        for (int k = 0; k < kLimbs; ++k)
            *reinterpret_cast<uint4*>(limbs + canon_off(N, (int64_t)k * LW + bc, 16 * g)) =
                make_uint4(L[k][0], L[k][1], L[k][2], L[k][3]);
    }
}

struct TcParams {
    const uint8_t* packed;  // WW_LAYOUT_TILE32 (App. H words re-tiled)
    const float* scales;
    const int8_t* limbs;  // canonical B operand, kpad/32 K-steps of N x 32 bytes
    const int* expo;      // 2B exponents
    float* Y;
    int64_t n, S, kpad, ldy;  // S: 64-column slabs per row (TILE32)
    int32_t B, N, per_row, conv;
    int32_t splits;                // CTAs per 32-row tile (one cluster), each a contiguous share
                                   // of the K blocks
    unsigned long long* trace;  // tools only: CTA 0's per-block globaltimer stamps
};

__device__ __forceinline__ void tc_trace(const TcParams& p, int kb, int ev) {
    if (p.trace && blockIdx.x < 2) p.trace[blockIdx.x * 512 + kb * 8 + ev] = clock64();  // SM cycles (CTAs 0, 1)
}

// One App. H word (16 codes of one plane and row, bit 2k = -1, bit 2k+1 = +1) -> 16 int8 in
// the K order [0,2,4,6, 8,10,12,14, 1,3,5,7, 9,11,13,15] (the limbs use the same order): the
// nibbles of w & 0x3333_3333 are the even codes, of (w >> 2) & 0x3333_3333 the odd ones, and
// PRMT with a nibble selector picks byte `code` of the table {0x00, 0xFF, 0x01, 0x00} (the
// unused code (1,1) gives 0, DESIGN R3)
__device__ __forceinline__ void decode_word(uint32_t w, uint32_t* o) {
    constexpr uint32_t kTable = 0x0001FF00u;
    const uint32_t e = w & 0x33333333u;
    const uint32_t d = (w >> 2) & 0x33333333u;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(o[0]) : "r"(kTable), "r"(e));
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(o[1]) : "r"(kTable), "r"(e >> 16));
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(o[2]) : "r"(kTable), "r"(d));
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(o[3]) : "r"(kTable), "r"(d >> 16));
}

__global__ void __launch_bounds__(kThreads, 1) wl_tc_kernel(const __grid_constant__ TcParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* smem = smem_raw + (base - raw);
    const int N = p.N;
    const uint32_t a_bytes = (uint32_t)kTM * kKB;           // one A block (4 K-steps)
    const uint32_t b_bytes = (uint32_t)N * kKB;             // one B block
    const uint32_t sa = base, sb = base + kStages * a_bytes;  // A ring, then the limb ring
    // barriers: bfull[kBStages] (limbs landed), done[kBStages] (MMAs of a block completed, by
    // block % kBStages), afull[kStages] (A tile decoded)
    const uint32_t bars = sb + kBStages * b_bytes;
    const uint32_t bfull = bars, bdone = bars + 8u * kBStages, afull = bars + 16u * kBStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + (bars - base) + 16 * kBStages + 8 * kStages);
    int* expo_s = reinterpret_cast<int*>(tmem_slot) + 4;  // the 2B exponents, staged once
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // tile and K share of this CTA: the K blocks of a tile are split into p.splits contiguous
    // ranges, so a layer with fewer tiles than SMs still fills the GPU; share 0 finishes the
    // tile from the others' flagged partial sums (exact int32)
    const int tile = blockIdx.x / p.splits, share = blockIdx.x % p.splits;
    const int64_t row0 = (int64_t)tile * kRows;
    if (tid == 0) tc_trace(p, 60, 0);  // kernel entry
    const int nkb_all = (int)(p.kpad / kKB);
    const int kb0 = (int)((int64_t)share * nkb_all / p.splits);
    const int nkb = (int)((int64_t)(share + 1) * nkb_all / p.splits) - kb0;  // this CTA's blocks

    if (warp == 0) {  // tensor-memory accumulator: N (>= 32, power of 2) columns x 128 lanes
        uint32_t cols = 32;
        while ((int)cols < N) cols <<= 1;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(tmem_slot)),
                     "r"(cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid >= 64 && tid < 64 + 2 * p.B) {  // read in the epilogue; written by the limb kernel
        asm volatile("griddepcontrol.wait;" ::: "memory");
        expo_s[tid - 64] = p.expo[tid - 64];
    }
    if (tid == 32) {
        for (int i = 0; i < 2 * kBStages; ++i) mbar_init(bars + 8u * i, 1);
        for (int i = 0; i < kStages; ++i) mbar_init(afull + 8u * i, kDecodeWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
    const uint32_t idesc = umma_idesc_i8(N);
    // the limbs of the first kStages - 1 blocks in flight (block kb + kStages - 1 is requested
    // once the MMAs of block kb - 1 have released its slot)
    // the limbs come from tc_limbs_kernel, the preceding (PDL primary) launch: the MMA warp waits
    // for it; the decode warps start on the weights at once
    if (warp == kDecodeWarps) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == kDecodeWarps * 32)
        for (int kb = 0; kb < kBStages - kLag && kb < nkb; ++kb) {
            mbar_expect_tx(bfull + 8u * kb, b_bytes);
            bulk_g2s(sb + (uint32_t)kb * b_bytes, p.limbs + (int64_t)(kb0 + kb) * b_bytes, b_bytes, bfull + 8u * kb);
        }

    if (warp == kDecodeWarps) {
        // ---- MMA warp: lane 0 issues the 4 MMAs of a block once its A tile is decoded (afull,
        // 8 warp arrivals) and its limbs have landed (bfull), commits to mdone, and keeps the
        // limb ring kStages - kLag blocks ahead
        if (lane == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % kStages, bs = kb % kBStages;
                tc_trace(p, kb, 6);
                mbar_wait(afull + 8u * st, (kb / kStages) & 1);   // A decoded
                tc_trace(p, kb, 5);
                mbar_wait(bfull + 8u * bs, (kb / kBStages) & 1);  // limbs landed
                tc_trace(p, kb, 3);
                tc_fence_after();
                // descriptors of the block's first K step; each next step advances the start
                // address field (16-byte units) by one K-step tile
                const uint64_t ad = umma_desc(sa + (uint32_t)st * a_bytes);
                const uint64_t bd = umma_desc(sb + (uint32_t)bs * b_bytes);
#pragma unroll
                for (int s4 = 0; s4 < kKB / 32; ++s4)
                    umma_i8(tmem, ad + (uint64_t)(s4 * (kTM * 32 / 16)),
                            bd + (uint64_t)(s4 * (N * 32 / 16)), idesc, (kb > 0 || s4 > 0) ? 1u : 0u);
                umma_commit(bdone + 8u * bs);  // block kb's MMAs: frees A slot st and limb slot bs
                tc_trace(p, kb, 4);
                // the limbs of block kb + kBStages - kLag into its slot, whose previous block
                // kb - kLag had its MMAs issued kLag iterations ago (MMA completion latency
                // stays off the critical path); the first kLag such slots start empty
                const int nb = kb + kBStages - kLag;
                if (nb < nkb) {
                    const int ps = nb % kBStages;
                    if (kb >= kLag) mbar_wait(bdone + 8u * ps, ((kb - kLag) / kBStages) & 1);
                    mbar_expect_tx(bfull + 8u * ps, b_bytes);
                    bulk_g2s(sb + (uint32_t)ps * b_bytes, p.limbs + (int64_t)(kb0 + nb) * b_bytes, b_bytes,
                             bfull + 8u * ps);
                }
            }
        }
    } else {
        // ---- decode warps.  Task of this thread: M-row mr (= 4 (row % 32) + plane, the
        // WW_LAYOUT_TILE32 order) and slab j (64 columns) of the K block: its 4 App. H words
        // (16 bytes, one coalesced 512-byte request per warp) become 64 int8 by 16 PRMTs
        // (decode_word) and 4 conflict-free STS.128 into the canonical K-major A tile.  The
        // words stream kStages blocks ahead in registers.
        const int mr = tid & 127, j = tid >> 7;
        const uint32_t a_off = (uint32_t)(2 * j) * (kTM * 32) + (uint32_t)(mr >> 3) * 256u + (uint32_t)(mr & 7) * 16u;
        const uint8_t* tsrc = p.packed + (int64_t)tile * p.S * kSlab32 + (int64_t)mr * 16;
        auto load_w = [&](int kb) -> uint4 {
            const int64_t slab = (int64_t)(kb0 + kb) * (kKB / 64) + j;
            return (kb < nkb && slab < p.S) ? ldg_stream(reinterpret_cast<const uint4*>(tsrc + slab * kSlab32))
                                            : make_uint4(0, 0, 0, 0);
        };
        uint4 wq[kStages];
#pragma unroll
        for (int i = 0; i < kStages; ++i) wq[i] = load_w(i);
        for (int kb = 0; kb < nkb; ++kb) {
            const int st = kb % kStages;
            if (tid == 0) tc_trace(p, kb, 0);
            if (kb >= kStages) {  // the MMAs of block kb - kStages released this A slot
                const int ob = kb - kStages;
                mbar_wait(bdone + 8u * (ob % kBStages), (ob / kBStages) & 1);
            }
            if (tid == 0) tc_trace(p, kb, 1);
            const uint4 w = wq[0];
#pragma unroll
            for (int i = 0; i < kStages - 1; ++i) wq[i] = wq[i + 1];
            wq[kStages - 1] = load_w(kb + kStages);
            const uint32_t dst = sa + (uint32_t)st * a_bytes + a_off;
            // word i (columns 16 i .. 16 i + 15 of the slab): K step 2 j + i / 2, half i % 2
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint32_t o[4];
                decode_word(ws[i], o);
                sts128(dst + (uint32_t)(i >> 1) * (kTM * 32) + (uint32_t)(i & 1) * 128u, o[0], o[1], o[2], o[3]);
            }
            fence_proxy_async_smem();  // this thread's generic stores -> the async proxy
            __syncwarp();
            if (lane == 0) mbar_arrive(afull + 8u * st);
            if (tid == 0) tc_trace(p, kb, 2);
        }
    }
    mbar_wait(bdone + 8u * ((nkb - 1) % kBStages), ((nkb - 1) / kBStages) & 1);  // all MMAs done
    tc_fence_after();
    if (tid == 0) tc_trace(p, 60, 1);  // epilogue start

    // split tiles: the CTAs of a tile form a cluster; once every CTA's MMAs are done (cluster
    // barrier: no CTA reads its shared memory any more) each share writes its accumulators
    // into share 0's shared memory (DSMEM), a second cluster barrier, and share 0 finishes the
    // tile from the exact int32 sums
    if (p.splits > 1) cluster_sync();
    if (tid == 0) tc_trace(p, 61, 0);
    // row of a lane: 3 limbs x cwp (2B padded to 4) words + 4, 16-byte aligned for the vector
    // stores into share 0
    const int cw = 2 * p.B, cwp = (cw + 3) & ~3, rs = 3 * cwp + 4;
    if (warp < 4) {
        // lane m = 32 warp + lane of the accumulator: output row m / 4, plane m % 4.
        // Dsm[share][m][l][c] = limb l of column c (= 2 b + comp), row stride 6B + 1 words
        // (conflict-free), in share 0's shared memory (the idle A ring)
        const int m = 32 * warp + lane;
        const int LW = N / kLimbs;
        const uint32_t dsm_local = base + (uint32_t)((share * 128 + m) * rs) * 4u;
        const uint32_t dsm = p.splits > 1 ? map_to_rank(dsm_local, 0) : dsm_local;
        const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll
        for (int l = 0; l < kLimbs; ++l) {
            int32_t D[32];
            tmem_ld32(tl + (uint32_t)(l * LW), D);  // limb l: columns l LW .. l LW + 2B - 1
#pragma unroll
            for (int c = 0; c < 32; c += 4)
                if (c < cw) st_cluster_v4(dsm + 4u * (uint32_t)(l * cwp + c), D[c], D[c + 1], D[c + 2], D[c + 3]);
        }
    }
    if (tid == 0) tc_trace(p, 61, 1);
    // every share's sums are in share 0 (and visible to all of its warps, which finish the tile)
    if (p.splits > 1) cluster_sync();
    else __syncthreads();
    if (tid == 0) tc_trace(p, 61, 2);
    if (warp < kDecodeWarps && share == 0) {
        // the 16 decode warps finish the tile: warp group grp = warp / 4 takes the vectors
        // b = grp, grp + 4, ... (summing their columns over the shares first); warp % 4 picks
        // the M-rows as in the accumulator (lane quarter)
        const int q = warp & 3, grp = warp >> 2;
        const int m = 32 * q + lane, rr = m >> 2, pl = m & 3;
        const int64_t row = row0 + rr;
        int32_t* Dsm = reinterpret_cast<int32_t*>(smem) + m * rs;
        if (tid == 0) tc_trace(p, 61, 3);
        {
            const double s = row < p.n ? (double)p.scales[p.per_row ? 4 * row + pl : pl] : 0.0;
            const bool eq1 = p.conv == WW_CONV_EQ1;
            for (int b = grp; b < p.B; b += 4) {
                for (int j = 1; j < p.splits; ++j)
#pragma unroll
                    for (int l = 0; l < kLimbs; ++l)
#pragma unroll
                        for (int comp = 0; comp < 2; ++comp) {
                            const int k = l * cwp + 2 * b + comp;
                            Dsm[k] += Dsm[j * 128 * rs + k];
                        }
                double S[2];
#pragma unroll
                for (int comp = 0; comp < 2; ++comp) {
                    const int c = 2 * b + comp;
                    const double v =
                        (double)Dsm[2 * cwp + c] * 65536.0 + (double)Dsm[cwp + c] * 256.0 + (double)Dsm[c];
                    S[comp] = v * __longlong_as_double((long long)(1023 - expo_s[c]) << 52) * s;  // 2^-E
                }
                // this plane's share of y (P:1002-1011 with the EQ1 / ALG1 signs of Eq. 1 / Eq. 3):
                // U_re: (re, im); U_im: (-im, re); W_re: (re, -+im); W_im: (im, +-re)
                double yre, yim;
                if (pl == 0) { yre = S[0]; yim = S[1]; }
                else if (pl == 1) { yre = -S[1]; yim = S[0]; }
                else if (pl == 2) { yre = S[0]; yim = eq1 ? -S[1] : S[1]; }
                else { yre = S[1]; yim = eq1 ? S[0] : -S[0]; }
                // sum over the four planes (lanes 4rr .. 4rr+3), fixed order: (0+1) + (2+3)
                yre += __shfl_xor_sync(0xffffffffu, yre, 1);
                yim += __shfl_xor_sync(0xffffffffu, yim, 1);
                yre += __shfl_xor_sync(0xffffffffu, yre, 2);
                yim += __shfl_xor_sync(0xffffffffu, yim, 2);
                if (pl == (b & 3) && row < p.n)
                    reinterpret_cast<float2*>(p.Y)[(int64_t)b * p.ldy + row] =
                        make_float2((float)yre, (float)yim);
            }
        }
    }
    if (tid == 0) tc_trace(p, 60, 2);  // epilogue end (warp 0)
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        uint32_t cols = 32;
        while ((int)cols < N) cols <<= 1;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols)
                     : "memory");
    }
}

}  // namespace

static unsigned long long* g_tc_trace = nullptr;
// Not part of the ABI: tools point CTA 0 of the tensor-core kernel at a trace buffer.
extern "C" void ww_debug_tc_trace(void* buf) { g_tc_trace = reinterpret_cast<unsigned long long*>(buf); }

// K splits per tile: enough CTAs to cover the SMs, at most 4, at least one K block each
static int tc_splits(int64_t n, int64_t m, int32_t B) {
    const int64_t tiles = (n + kRows - 1) / kRows, nkb = tc_kpad(m) / kKB;
    int64_t sp = ww::device_sms() / tiles;
    if (sp > 4) sp = 4;
    // the shares' accumulators (128 rows of 6B + 1 words each) must fit share 0's rings
    const int64_t ring = (int64_t)kStages * kTM * kKB + (int64_t)kBStages * tc_n(B) * kKB;
    const int64_t fit = ring / (128 * (3 * ((2 * (int64_t)B + 3) & ~3) + 4) * 4);
    if (sp > fit) sp = fit;
    if (sp > nkb) sp = nkb;
    return sp < 1 ? 1 : (int)sp;
}

extern "C" size_t ww_tc_workspace_bytes(int64_t n, int64_t m, int32_t B) {
    if (n < 1 || m < 1 || B < 1 || B > kMaxB) return 0;
    return (size_t)tc_kpad(m) * (size_t)tc_n(B) + 256;
}

extern "C" ww_status ww_wl_gemv_batched_tc(const ww_layer* L, const void* packed_d, const float* scales_d,
                                           const float* X_d, int64_t ldx, float* Y_d, int64_t ldy,
                                           int32_t B, void* workspace_d, void* stream) {
    const char* fn = "ww_wl_gemv_batched_tc";
    if (!L || !packed_d || !scales_d || !X_d || !Y_d || !workspace_d)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: null pointer", fn);
    if (L->n < 1 || L->m < 1 || L->n > ((int64_t)1 << 30) || L->m > kLimbMaxM)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: n=%lld m=%lld", fn, (long long)L->n, (long long)L->m);
    if (L->layout != WW_LAYOUT_TILE32)
        return ww::fail(WW_ERR_UNSUPPORTED, "%s: needs WW_LAYOUT_TILE32", fn);
    if (L->conv != WW_CONV_EQ1 && L->conv != WW_CONV_ALG1)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: conv %d", fn, L->conv);
    if (B < 1 || B > kMaxB)
        return ww::fail(WW_ERR_UNSUPPORTED, "%s: B=%d (1..16)", fn, B);
    if (ldx < L->m || ldy < L->n)
        return ww::fail(WW_ERR_DIMENSION_MISMATCH, "%s: ldx=%lld ldy=%lld", fn, (long long)ldx, (long long)ldy);
    if (((uintptr_t)packed_d & 15) || ((uintptr_t)X_d & 7) || ((uintptr_t)Y_d & 7) ||
        ((uintptr_t)scales_d & 3) || ((uintptr_t)workspace_d & 127))
        return ww::fail(WW_ERR_MISALIGNED, "%s: packed 16-B, x/y 8-B, workspace 128-B aligned", fn);
    const int N = tc_n(B);
    const int64_t kpad = tc_kpad(L->m);
    int8_t* limbs = reinterpret_cast<int8_t*>(workspace_d);
    int* expo = reinterpret_cast<int*>(reinterpret_cast<char*>(workspace_d) + (size_t)kpad * N);
    const int splits = tc_splits(L->n, L->m, B);
    cudaStream_t s = (cudaStream_t)stream;
    tc_limbs_kernel<<<2 * B + 1, kLimbThreads, 0, s>>>(X_d, ldx, B, L->m, kpad, N, limbs, expo);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return ww::fail(WW_ERR_CUDA, "%s: %s", fn, cudaGetErrorString(e));
    TcParams p;
    memset(&p, 0, sizeof p);
    p.packed = reinterpret_cast<const uint8_t*>(packed_d);
    p.scales = scales_d;
    p.limbs = limbs;
    p.expo = expo;
    p.Y = Y_d;
    p.n = L->n;
    p.S = ww::tile32_slabs(L->m);
    p.kpad = kpad;
    p.ldy = ldy;
    p.B = B;
    p.N = N;
    p.per_row = L->scale_mode == WW_SCALES_PER_ROW;
    p.conv = L->conv;
    p.trace = g_tc_trace;
    p.splits = splits;
    const int smem = (int)(kStages * kTM * kKB + kBStages * (int64_t)N * kKB + 16 * kBStages +
                           8 * kStages + 64 + 4 * 2 * kMaxB + 1024);
    const int pe = ww::prepare_kernel(reinterpret_cast<const void*>(wl_tc_kernel), 227 * 1024);
    if (pe) return ww::fail(WW_ERR_CUDA, "%s: %s", fn, cudaGetErrorString((cudaError_t)pe));
    const int grid = (int)((L->n + kRows - 1) / kRows) * splits;
    {
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof cfg);
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = (size_t)smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;  // the shares of a tile: one cluster
        attr[0].val.clusterDim.x = (unsigned)splits;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the limb kernel
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        e = cudaLaunchKernelEx(&cfg, wl_tc_kernel, p);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return ww::fail(WW_ERR_CUDA, "%s: %s", fn, cudaGetErrorString(e));
    return ww::ok();
}
