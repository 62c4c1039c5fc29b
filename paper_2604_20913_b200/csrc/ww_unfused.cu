// Unfused ablation of the WL-GEMV (the paper's unfused baseline,
// P:308-335 and Table "fused vs unfused"): one *real* ternary GEMV per
// (plane, component of x) -- eight calls per widely-linear layer, each re-streaming its
// plane's codes and one real component of x -- followed by a combine kernel that applies the
// scales.  Built to measure the fusion speedup on B200 against the fused kernel
// (ww_kernels.cu), not as a product path: same launch style (one persistent CTA per SM,
// PDL, coalesced 32-bit code loads from the App. H planar layout, predicated fp32 adds,
// warp reduction), no multiplies in the accumulation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "ww.h"
#include "ww_internal.h"

namespace {

constexpr int kWarps = 16;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}
__device__ __forceinline__ uint32_t ldg_stream32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// acc[i] = sum_j t_ij * xc_j for one plane of the App. H planar layout (n x W words, slot k
// of word c = column 16c+k, bit 2k+1 = +1, bit 2k = -1) and one real component
// xc of the complex64 vector x (Eqs. 6-7: +1 adds, -1 subtracts, 0 / (1,1) contribute 0).
// Tuned like the fused kernel: a warp owns a row (contiguous per-warp row ranges), each lane
// streams one 128-bit load = 4 words = 64 consecutive columns per sweep (2048 columns per
// warp sweep, two sweeps in flight), predicated fp32 adds (R2P-decoded), x staged once per
// CTA with the lane blocks' 16 granules XOR-swizzled (granule g of 64-column block L at
// L*16 + (g ^ (L & 15))) so the 32 lanes' LDS.128 are conflict-free; the rows' four
// accumulators reduced by warp shuffles.  Needs a 16-B aligned plane (W % 4 == 0: 64 | m);
// other shapes take the word-per-lane kernel below.
__global__ void __launch_bounds__(kWarps * 32, 2)
tern_plane_v4_kernel(const uint32_t* __restrict__ plane, const float* __restrict__ X, int comp,
                     int64_t n, int64_t m, int64_t W, float* __restrict__ acc_out) {
    extern __shared__ __align__(16) float xs4[];  // nblk x 16 granules x 4 floats
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * n / gridDim.x;
    const int64_t r1 = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
    const int NRc = (int)(r1 - r0);
    const int ub = NRc / kWarps, ue = NRc - ub * kWarps;
    const int w0 = warp * ub + (warp < ue ? warp : ue), w1 = w0 + ub + (warp < ue ? 1 : 0);
    const int64_t W4 = W / 4;             // 64-column blocks per row
    const int J = (int)((W4 + 31) / 32);  // sweeps per row
    pdl_launch_dependents();
    const uint4* base = reinterpret_cast<const uint4*>(plane) + (r0 + w0) * W4 + lane;
    int pr = w0, pk = 0;
    auto load_next = [&]() -> uint4 {
        uint4 v = make_uint4(0, 0, 0, 0);
        const int64_t blk = (int64_t)pk * 32 + lane;
        if (pr < w1 && blk < W4)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "l"(base + (int64_t)(pr - w0) * W4 + (int64_t)pk * 32));
        if (++pk == J) {
            pk = 0;
            ++pr;
        }
        return v;
    };
    uint4 qa = load_next(), qb = load_next();
    pdl_wait();
    const int64_t nblk = (int64_t)J * 32;
    for (int64_t e = threadIdx.x; e < nblk * 16; e += blockDim.x) {  // stage xc, swizzled
        const int64_t L = e >> 4, g = e & 15;
        float4 v;
        float* vp = &v.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t col = L * 64 + g * 4 + q;
            vp[q] = col < m ? X[2 * col + comp] : 0.f;
        }
        reinterpret_cast<float4*>(xs4)[L * 16 + (g ^ (L & 15))] = v;
    }
    __syncthreads();
    for (int r = w0; r < w1; ++r) {
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        for (int k = 0; k < J; ++k) {
            const uint4 w = qa;
            qa = qb;
            qb = load_next();
            const int64_t L = (int64_t)k * 32 + lane;
            const float4* xb = reinterpret_cast<const float4*>(xs4) + L * 16;
            const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int g = 0; g < 16; ++g) {
                const float4 v = xb[g ^ (int)(L & 15)];
                const float xv[4] = {v.x, v.y, v.z, v.w};
                const uint32_t word = w4[g >> 2];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int slot = 4 * (g & 3) + q;
                    if (word & (2u << (2 * slot))) a[q] = __fadd_rn(a[q], xv[q]);
                    if (word & (1u << (2 * slot))) a[q] = __fadd_rn(a[q], -xv[q]);
                }
            }
        }
        float t = (a[0] + a[1]) + (a[2] + a[3]);
#pragma unroll
        for (int off = 16; off; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) acc_out[r0 + r] = t;
    }
}

// Word-per-lane variant (any m): a warp owns a row (rows round-robin over the CTA's 16 warps), lanes take 16-column words,
// 32 words per sweep; x is staged once per CTA transposed by granule (granule g of word c at
// (g*Wp + c)*16) so 32 lanes reading their words' granule g hit consecutive addresses.
__global__ void __launch_bounds__(kWarps * 32, 2)
tern_plane_kernel(const uint32_t* __restrict__ plane, const float* __restrict__ X, int comp,
                  int64_t n, int64_t m, int64_t W, float* __restrict__ acc_out) {
    extern __shared__ __align__(16) float xs[];  // 4 granules x Wp words x 4 floats
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * n / gridDim.x;
    const int64_t r1 = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
    const int64_t Wp = (W + 31) / 32 * 32;
    pdl_launch_dependents();
    // the warp's code words as one stream over its rows (row = r0 + warp + 16 t), sweep k
    // of a row = words [32k, 32k+32), one word per lane; four sweeps in flight in registers,
    // the first four requested before waiting (codes never depend on x)
    const int J = (int)((W + 31) / 32);
    int64_t prow = r0 + warp;
    int pk = 0;
    auto load_next = [&]() -> uint32_t {
        uint32_t v = 0u;
        const int64_t c = (int64_t)pk * 32 + lane;
        if (prow < r1 && c < W) v = ldg_stream32(plane + prow * W + c);
        if (++pk == J) {
            pk = 0;
            prow += kWarps;
        }
        return v;
    };
    uint32_t q0 = load_next(), q1 = load_next(), q2 = load_next(), q3 = load_next();
    pdl_wait();
    for (int64_t e = threadIdx.x; e < 4 * Wp * 4; e += blockDim.x) {  // stage xc
        const int64_t g = e / (Wp * 4), rem = e - g * Wp * 4, c = rem / 4, q = rem & 3;
        const int64_t col = c * 16 + g * 4 + q;
        xs[(g * Wp + c) * 4 + q] = col < m ? X[2 * col + comp] : 0.f;
    }
    __syncthreads();
    for (int64_t row = r0 + warp; row < r1; row += kWarps) {
        float a0 = 0.f, a1 = 0.f;
        for (int k = 0; k < J; ++k) {
            const uint32_t w = q0;
            q0 = q1;
            q1 = q2;
            q2 = q3;
            q3 = load_next();
            const int64_t c = (int64_t)k * 32 + lane;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const float4 v = *reinterpret_cast<const float4*>(xs + (g * Wp + c) * 4);
                const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int slot = 4 * g + q;
                    float& a = (q & 1) ? a1 : a0;
                    if (w & (2u << (2 * slot))) a = __fadd_rn(a, xv[q]);
                    if (w & (1u << (2 * slot))) a = __fadd_rn(a, -xv[q]);
                }
            }
        }
        float t = a0 + a1;
#pragma unroll
        for (int off = 16; off; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) acc_out[row] = t;
    }
}

// y_i from the eight real partial sums A[c][i], c = 2*plane + component (re 0, im 1),
// with the row's scales applied once: EQ1 (Eq. 1) or ALG1 (Eqs. 2-3)
__global__ void combine_kernel(const float* __restrict__ A, const float* __restrict__ scales,
                               int per_row, int conv, int64_t n, float* __restrict__ Y) {
    pdl_launch_dependents();
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float* s = scales + (per_row ? 4 * i : 0);
        const float Ur_re = A[0 * n + i], Ur_im = A[1 * n + i], Ui_re = A[2 * n + i],
                    Ui_im = A[3 * n + i], Wr_re = A[4 * n + i], Wr_im = A[5 * n + i],
                    Wi_re = A[6 * n + i], Wi_im = A[7 * n + i];
        const float yre = s[0] * Ur_re - s[1] * Ui_im + s[2] * Wr_re + s[3] * Wi_im;
        const float yim = conv == WW_CONV_EQ1
                              ? s[0] * Ur_im + s[1] * Ui_re - s[2] * Wr_im + s[3] * Wi_re
                              : s[0] * Ur_im + s[1] * Ui_re + s[2] * Wr_im - s[3] * Wi_re;
        reinterpret_cast<float2*>(Y)[i] = make_float2(yre, yim);
    }
}

int sm_count() { return ww::device_sms(); }  // cached per device (ww_device.cu)

template <typename K, typename... A>
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                       A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace

extern "C" ww_status ww_ternary_gemv_plane(int64_t n, int64_t m, const void* planar_d,
                                           int32_t plane, const float* x_d, int32_t comp,
                                           float* acc_d, uint32_t flags, void* stream) {
    if (!planar_d || !x_d || !acc_d)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_ternary_gemv_plane: null pointer");
    if (n < 1 || m < 1 || n > (int64_t)1 << 30 || m > (int64_t)1 << 24 || plane < 0 || plane > 3 ||
        comp < 0 || comp > 1)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_ternary_gemv_plane: n=%lld m=%lld plane=%d comp=%d",
                        (long long)n, (long long)m, plane, comp);
    if (((uintptr_t)planar_d & 3) || ((uintptr_t)x_d & 7) || ((uintptr_t)acc_d & 3))
        return ww::fail(WW_ERR_MISALIGNED, "ww_ternary_gemv_plane: misaligned pointer");
    const int64_t W = ww::words_per_row(m);
    const int64_t Wp = (W + 31) / 32 * 32;
    const size_t smem = (size_t)Wp * 16 * 4;
    if (smem > 200 * 1024)
        return ww::fail(WW_ERR_UNSUPPORTED, "ww_ternary_gemv_plane: m=%lld too large", (long long)m);
    // the 32-bit kernel is launched only when the 128-bit one below does not apply
    const auto prepare32 = [] {
        return ww::prepare_kernel(reinterpret_cast<const void*>(tern_plane_kernel), 200 * 1024);
    };
    const uint32_t* pl = reinterpret_cast<const uint32_t*>(planar_d) + (int64_t)plane * n * W;
    const int grid = (int)std::min<int64_t>(sm_count(), n);
    if (W % 4 == 0 && ((uintptr_t)planar_d & 15) == 0) {  // the 128-bit kernel
        const int64_t J = (W / 4 + 31) / 32;
        const size_t smem4 = (size_t)J * 32 * 16 * 16;
        if (smem4 <= 200 * 1024) {
            const int e4 = ww::prepare_kernel(reinterpret_cast<const void*>(tern_plane_v4_kernel),
                                              200 * 1024);
            if (e4)
                return ww::fail(WW_ERR_CUDA, "ww_ternary_gemv_plane: %s",
                                cudaGetErrorString((cudaError_t)e4));
            cudaError_t e = launch_pdl(tern_plane_v4_kernel, dim3(grid), dim3(kWarps * 32), smem4,
                                       (cudaStream_t)stream, (flags & WW_FLAG_PDL) != 0, pl, x_d,
                                       (int)comp, n, m, W, acc_d);
            if (e != cudaSuccess)
                return ww::fail(WW_ERR_CUDA, "ww_ternary_gemv_plane: %s", cudaGetErrorString(e));
            return ww::ok();
        }
    }
    if (const int e32 = prepare32())
        return ww::fail(WW_ERR_CUDA, "ww_ternary_gemv_plane: %s",
                        cudaGetErrorString((cudaError_t)e32));
    cudaError_t e = launch_pdl(tern_plane_kernel, dim3(grid), dim3(kWarps * 32), smem,
                               (cudaStream_t)stream, (flags & WW_FLAG_PDL) != 0, pl, x_d, (int)comp,
                               n, m, W, acc_d);
    if (e != cudaSuccess)
        return ww::fail(WW_ERR_CUDA, "ww_ternary_gemv_plane: %s", cudaGetErrorString(e));
    return ww::ok();
}

extern "C" ww_status ww_wl_combine(const ww_layer* L, const float* acc8_d, const float* scales_d,
                                   float* y_d, void* stream) {
    if (!L || !acc8_d || !scales_d || !y_d)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_combine: null pointer");
    if (L->n < 1 || (L->conv != WW_CONV_EQ1 && L->conv != WW_CONV_ALG1))
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_wl_combine: n=%lld conv=%d", (long long)L->n,
                        L->conv);
    if (((uintptr_t)y_d & 7) || ((uintptr_t)acc8_d & 3) || ((uintptr_t)scales_d & 3))
        return ww::fail(WW_ERR_MISALIGNED, "ww_wl_combine: misaligned pointer");
    const int grid = (int)std::min<int64_t>(sm_count() * 4, (L->n + 255) / 256);
    cudaError_t e = launch_pdl(combine_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream,
                               (L->flags & WW_FLAG_PDL) != 0, acc8_d, scales_d,
                               (int)(L->scale_mode == WW_SCALES_PER_ROW), (int)L->conv, L->n, y_d);
    if (e != cudaSuccess) return ww::fail(WW_ERR_CUDA, "ww_wl_combine: %s", cudaGetErrorString(e));
    return ww::ok();
}
