// Device building blocks shared by the WL-GEMV kernels (ww_kernels.cu) and the persistent
// program kernel (ww_program.cu): PTX wrappers (streaming loads, cp.async, mbarriers, TMA,
// PDL), and the sweep arithmetic of one 16-column COL4 chunk -- decode (a5, Eqs. 4-5
// P:911-929) into predicates and predicated FADD2 accumulation (a6, Eqs. 6-7) --
// plus the warp transpose-reduce of the row totals (a7).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// the same load, issued only when a < b (else zeros): one compare + one predicated LDG
__device__ __forceinline__ uint4 ldg_stream_lt(const uint4* p, int a, int b) {
    uint4 v = make_uint4(0, 0, 0, 0);
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %5, %6;\n\t"
        "@q ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
        : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
        : "l"(p), "r"(a), "r"(b));
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
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// L2 prefetch of the 16-byte chunk at p when a < b (one compare + one predicated PREFETCH)
__device__ __forceinline__ void prefetch_chunk_lt(const uint4* p, int a, int b) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %1, %2;\n\t@q prefetch.global.L2 [%0];\n\t}"
        :: "l"(p), "r"(a), "r"(b));
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }

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
__device__ __forceinline__ void mbar_wait0(uint32_t bar) { mbar_wait(bar, 0); }


// Accumulators: S column-parity sets of B x 4 pair sums.  For B <= 2 even and odd columns
// feed separate sets (more independent FADD2 chains per warp, half-length fp32 chains);
// larger B has ILP across vectors.  (Separate sums of the +1 and the -1 codes measured
// 5-10 % slower: register pressure.)
template <int B>
struct Acc {
#ifndef WW_ACC_POSNEG
#define WW_ACC_POSNEG 0  // experiment switch: B = 1 keeps +1 and -1 sums apart (S = 1, N = 2)
#endif
#ifndef WW_ACC_S_B4
#define WW_ACC_S_B4 1  // experiment switch: column-parity sets at 3 <= B <= 4
#endif
    static constexpr int S = (B == 1 && WW_ACC_POSNEG) ? 1 : (B <= 2 ? 2 : (B <= 4 ? WW_ACC_S_B4 : 1));
    static constexpr int N = (B == 1 && WW_ACC_POSNEG) ? 2 : 1;
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
    // sum over sets of plane q, vector b (pos - neg when N == 2)
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
// NEXT-2 ablation switches (tools/ablation_o1o4.py builds each as a separate library; all 0
// in the product): WW_ABL_NO_O1 -- no mask reuse, the real and the imaginary path decode
// their own predicates and add with scalar FADDs; WW_ABL_NO_O2 -- no input reuse, every
// plane re-loads its (x_re, x_im) pair from shared memory; WW_ABL_NO_O4 -- no register-
// resident accumulators, they are spilled to local memory and reloaded after every chunk.
#ifndef WW_ABL_NO_O1
#define WW_ABL_NO_O1 0
#endif
#ifndef WW_ABL_NO_O2
#define WW_ABL_NO_O2 0
#endif
#ifndef WW_ABL_NO_O4
#define WW_ABL_NO_O4 0
#endif

__device__ __forceinline__ float2 lds64v(uint32_t addr) {  // a load ptxas cannot merge
    float2 v;
    asm volatile("ld.volatile.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

template <int N>
__device__ __forceinline__ void column(float2 (&pos)[4], float2 (&neg)[4], uint32_t bits, float2 x,
                                       uint32_t bits_im = 0) {
#if WW_ABL_NO_O1
    // each path decodes its own predicates (two R2P + tests per column, bits_im extracted
    // from the code word by a second, different instruction so ptxas cannot share them)
    // and adds alone
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int q = k >> 1;
        if (bits & (1u << k)) pos[q].x = __fadd_rn(pos[q].x, (k & 1) ? x.x : -x.x);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int q = k >> 1;
        if (bits_im & (1u << k)) pos[q].y = __fadd_rn(pos[q].y, (k & 1) ? x.y : -x.y);
    }
    return;
#endif
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
// chunk: 64 codes x B vectors, 2 predicated FADD2 per code and vector.  xl = smem address of
// the chunk's x for vector 0 with the swizzle key in bits 4..6 (chunk base | (chunk & 7) << 4;
// vector b at + b*bstride): granule kk (columns 2kk, 2kk+1) sits at xl ^ (kk << 4), one LOP3
// per load (the 128B swizzle of the TMA boxes; 32 lanes on 32 chunks hit 32 banks).
template <int B>
__device__ __forceinline__ void chunk(Acc<B>& acc, const uint4 w, uint32_t xl, uint32_t bstride,
                                      uint32_t off = 0) {
    // off: a multiple of 4096 added after the swizzle (the chunk 32 sweeps later sits at the
    // same swizzle key), so two sweeps can share the swizzled addresses with immediate offsets
    constexpr int S = Acc<B>::S, N = Acc<B>::N;
    const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {  // column pair (2kk, 2kk+1)
        const uint32_t word = w4[kk >> 1];
        const uint32_t sh = (kk & 1) * 16;
        const uint32_t bits_a = (word >> sh) & 0xffu, bits_b = (word >> (sh + 8)) & 0xffu;
        const uint32_t xa = (xl ^ ((uint32_t)kk << 4)) + off;
#if WW_ABL_NO_O2
        if (B == 1) {  // every plane re-loads x: 4 loads per column instead of one per pair
#pragma unroll
            for (int c = 1; c >= 0; --c) {
                const uint32_t bits = c ? bits_b : bits_a;
                float2(&pos)[4] = acc.a[c ? S - 1 : 0][0][0];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 x = lds64v(xa + 8u * c);
                    if (bits & (2u << (2 * q))) pos[q] = fadd2(pos[q], x);
                    if (bits & (1u << (2 * q))) pos[q] = fadd2(pos[q], make_float2(-x.x, -x.y));
                }
            }
            continue;
        }
#endif
#pragma unroll
        for (int b = 0; b < B; ++b) {  // each decoded code drives all B vectors (a9)
            const float4 v = lds128(xa + b * bstride);
            // (odd column first: the same sums -- each column-parity set keeps its own
            // order -- but ptxas then needs no predicate spill across the R2Ps)
#if WW_ABL_NO_O1
            // the same bytes through PRMT (byte select), a second decode path
            const uint32_t ia = __byte_perm(word, 0u, 0x4440u | (2u * (kk & 1))),
                           ib = __byte_perm(word, 0u, 0x4440u | (2u * (kk & 1) + 1u));
            column<N>(acc.a[S - 1][0][b], acc.a[S - 1][N - 1][b], bits_b, make_float2(v.z, v.w), ib);
            column<N>(acc.a[0][0][b], acc.a[0][N - 1][b], bits_a, make_float2(v.x, v.y), ia);
#else
            column<N>(acc.a[S - 1][0][b], acc.a[S - 1][N - 1][b], bits_b, make_float2(v.z, v.w));
            column<N>(acc.a[0][0][b], acc.a[0][N - 1][b], bits_a, make_float2(v.x, v.y));
#endif
        }
    }
#if WW_ABL_NO_O4
    {  // accumulators leave the registers after every chunk: spill to local memory, reload
        volatile float2 spill[S][N][B][4];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int k = 0; k < N; ++k)
#pragma unroll
                for (int b = 0; b < B; ++b)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        spill[s][k][b][q].x = acc.a[s][k][b][q].x;
                        spill[s][k][b][q].y = acc.a[s][k][b][q].y;
                    }
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int k = 0; k < N; ++k)
#pragma unroll
                for (int b = 0; b < B; ++b)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        acc.a[s][k][b][q] = make_float2(spill[s][k][b][q].x, spill[s][k][b][q].y);
    }
#endif
}

// Transpose-reduce NV (power of 2) partial sums across the warp: after the halving rounds
// lane l holds NV>>H totals starting at index (bit4(l) bit3(l) ...)_2 * (NV>>H).  Every
// value is summed over the lanes in the same xor-butterfly order (16, 8, 4, 2, 1) for any
// NV, so the totals do not depend on how many values are reduced together.
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


// ---------------------------------------------------------------- fused decode-block ops
// (NEXT-3) on a staged, 128B-swizzled x region of 8*32*J 16-byte granules (2
// complex columns each), shared by the per-stage kernel and the program kernel so both give
// the same bits.  Granule gi of chunk c = gi >> 3 sits at physical slot gi & 7 and holds
// logical granule (gi & 7) ^ (c & 7), i.e. columns 16c + 2g, +1.

__device__ __forceinline__ void sts128_f4(uint32_t addr, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

// x <- x (.) x2 on the real view (re*re, im*im): SiLU(gate) (.) up
__device__ __forceinline__ void x_mul(uint32_t xa, uint32_t xb, int ng, int tid, int nthr) {
    for (int gi = tid; gi < ng; gi += nthr) {
        const float4 a = lds128(xa + 16u * gi), b = lds128(xb + 16u * gi);
        sts128_f4(xa + 16u * gi, make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w));
    }
}

// RMSNorm in one pass: x <- x * gamma in place while summing x^2 over the real
// 2m-vector; the scalar 1 / sqrt(mean(x^2) + eps) is applied to the row results in the
// epilogue (the map is linear: WL(r v) = r WL(v)).  g[k] = this thread's gamma granules,
// loaded before the readiness wait (gamma is a weight); returns the warp-reduced partial sum
// (xor butterfly, the same order for every caller).
constexpr int kGammaRegs = 4;  // gamma granules a thread holds in registers (J <= 8 at 512 thr.)
__device__ __forceinline__ void gamma_prefetch(float4 (&g)[kGammaRegs], const float* gamma,
                                               int64_t m, int J, int tid, int nthr) {
#pragma unroll
    for (int k = 0; k < kGammaRegs; ++k) {
        const int gi = tid + k * nthr;
        const int c = gi >> 3, gg = (gi & 7) ^ (c & 7);
        const int64_t col = 16 * (int64_t)c + 2 * gg;
        g[k] = (gi < 8 * 32 * J && col < m) ? __ldg(reinterpret_cast<const float4*>(gamma + 2 * col))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}
__device__ __forceinline__ float x_gamma_sumsq_warp(uint32_t xa, int ng, int tid, int nthr,
                                                    const float4 (&g)[kGammaRegs],
                                                    const float* gamma, int64_t m) {
    float ss = 0.f;
    auto one = [&](int gi, float4 gm) {
        const float4 a = lds128(xa + 16u * gi);
        ss = ss + a.x * a.x;
        ss = ss + a.y * a.y;
        ss = ss + a.z * a.z;
        ss = ss + a.w * a.w;
        sts128_f4(xa + 16u * gi, make_float4(a.x * gm.x, a.y * gm.y, a.z * gm.z, a.w * gm.w));
    };
#pragma unroll
    for (int k = 0; k < kGammaRegs; ++k)
        if (tid + k * nthr < ng) one(tid + k * nthr, g[k]);
    for (int gi = tid + kGammaRegs * nthr; gi < ng; gi += nthr) {  // wide x: load gamma here
        const int c = gi >> 3, gg = (gi & 7) ^ (c & 7);
        const int64_t col = 16 * (int64_t)c + 2 * gg;
        one(gi, col < m ? __ldg(reinterpret_cast<const float4*>(gamma + 2 * col))
                        : make_float4(0.f, 0.f, 0.f, 0.f));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    return ss;
}

// this thread's share of sum(x^2) over the real 2m-vector, then reduced over the warp
// (xor butterfly, the same order for every caller)
__device__ __forceinline__ float x_sumsq_warp(uint32_t xa, int ng, int tid, int nthr) {
    float ss = 0.f;
    for (int gi = tid; gi < ng; gi += nthr) {
        const float4 a = lds128(xa + 16u * gi);
        ss = ss + a.x * a.x;
        ss = ss + a.y * a.y;
        ss = ss + a.z * a.z;
        ss = ss + a.w * a.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    return ss;
}

// RMSNorm factor from the per-warp partial sums (fixed order: deterministic)
__device__ __forceinline__ float rms_factor(const float* part, int nwarps, int64_t m, float eps) {
    float tot = 0.f;
    for (int w = 0; w < nwarps; ++w) tot += part[w];
    return 1.0f / sqrtf(tot / (float)(2 * m) + eps);
}

// x <- (x * gamma) * r (gamma: 2m fp32 over the real view)
__device__ __forceinline__ void x_rms_scale(uint32_t xa, int ng, int tid, int nthr,
                                            const float* gamma, int64_t m, float r) {
    for (int gi = tid; gi < ng; gi += nthr) {
        const int c = gi >> 3, g = (gi & 7) ^ (c & 7);
        const int64_t col = 16 * (int64_t)c + 2 * g;
        if (col >= m) continue;  // zero padding stays zero
        const float4 a = lds128(xa + 16u * gi);
        const float4 gm = __ldg(reinterpret_cast<const float4*>(gamma + 2 * col));
        sts128_f4(xa + 16u * gi, make_float4(a.x * gm.x * r, a.y * gm.y * r, a.z * gm.z * r,
                                            a.w * gm.w * r));
    }
}

__device__ __forceinline__ float silu_f(float v) { return v / (1.0f + expf(-v)); }
}  // namespace
