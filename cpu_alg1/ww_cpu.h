/* ww_cpu.h -- the paper's own CPU datapath: Algorithm 1
 * with AVX-512F masked add/sub and BMI2 pext (Table tab:intrinsics), OpenMP
 * over contiguous row ranges.  A like-for-like CPU baseline reported beside
 * the GPU kernel; it is NOT a fallback of the CUDA path (ww.h) and shares no code with it
 * or with the oracle.
 *
 * Input: App. H planar words (four planes U_re, U_im, W_re, W_im, each n x
 * ceil(m/16) uint32, slot k = bits 2k (-1) / 2k+1 (+1)); scales per row (n x 4 fp32
 * [sUr, sUi, sWr, sWi]) or per tensor (4 fp32); x: m complex64; y: n complex64.
 * conv 0 = Eq. 1 (y = U x + W conj x), 1 = Alg. 1 / Eqs. 2-3 ((U + conj W) x).
 * Returns 0, -1 on bad arguments, -2 when the CPU lacks AVX-512F or BMI2. */
#ifndef WW_CPU_H
#define WW_CPU_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int wwc_supported(void);
int wwc_max_threads(void);
int wwc_wl_gemv(const uint32_t* planar, int64_t n, int64_t m, const float* scales, int per_row,
                int conv, const float* x, float* y, int nthreads);
#ifdef __cplusplus
}
#endif
#endif
