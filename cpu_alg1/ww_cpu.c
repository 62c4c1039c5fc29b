/* ww_cpu.c -- Algorithm 1 of FairyFuse on AVX-512F + BMI2, see ww_cpu.h.
 * Per output row i (one OpenMP thread owns a contiguous row range):
 *   O4: eight 16-lane fp32 accumulators a^re_1..4, a^im_1..4 in zmm registers;
 *   O2: x_re / x_im chunks loaded once per 16 columns and shared by all four planes;
 *   O1: per plane word p, k+ = pext(p, 0xAAAAAAAA), k- = pext(p, 0x55555555) (Eqs. 4-5),
 *       applied to both the real and the imaginary path (Eqs. 6-7: masked add, then sub);
 *   then _mm512_reduce_add_ps and the scale-weighted sums (the only multiplies).
 * O3's neg_x_im is folded into the signs of the weighted sums, as Alg. 1 prints them
 * (R4). */
#include "ww_cpu.h"

#include <immintrin.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int wwc_supported(void) {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("bmi2");
}

int wwc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

__attribute__((target("avx512f,bmi2"))) static inline __m512 masked_as(__m512 a, uint32_t kp,
                                                                     uint32_t kn, __m512 X) {
    a = _mm512_mask_add_ps(a, (__mmask16)kp, a, X); /* Eq. 6 */
    a = _mm512_mask_sub_ps(a, (__mmask16)kn, a, X); /* Eq. 7 */
    return a;
}

__attribute__((target("avx512f,bmi2"))) static void rows(const uint32_t* planar, int64_t n,
                                                         int64_t W, const float* scales,
                                                         int per_row, int conv,
                                                         const float* xre, const float* xim,
                                                         float* y, int64_t i0, int64_t i1) {
    const uint32_t MP = 0xAAAAAAAAu, MN = 0x55555555u;
    const uint32_t* Ur = planar;
    const uint32_t* Ui = planar + n * W;
    const uint32_t* Wr = planar + 2 * n * W;
    const uint32_t* Wi = planar + 3 * n * W;
    for (int64_t i = i0; i < i1; ++i) {
        __m512 r1 = _mm512_setzero_ps(), r2 = r1, r3 = r1, r4 = r1;
        __m512 m1 = r1, m2 = r1, m3 = r1, m4 = r1;
        const int64_t o = i * W;
        for (int64_t j = 0; j < W; ++j) {
            const __m512 Xre = _mm512_loadu_ps(xre + 16 * j); /* O2 */
            const __m512 Xim = _mm512_loadu_ps(xim + 16 * j);
            uint32_t p = Ur[o + j];
            uint32_t kp = _pext_u32(p, MP), kn = _pext_u32(p, MN); /* O1 */
            r1 = masked_as(r1, kp, kn, Xre);
            m1 = masked_as(m1, kp, kn, Xim);
            p = Ui[o + j];
            kp = _pext_u32(p, MP), kn = _pext_u32(p, MN);
            r2 = masked_as(r2, kp, kn, Xim);
            m2 = masked_as(m2, kp, kn, Xre);
            p = Wr[o + j];
            kp = _pext_u32(p, MP), kn = _pext_u32(p, MN);
            r3 = masked_as(r3, kp, kn, Xre);
            m3 = masked_as(m3, kp, kn, Xim);
            p = Wi[o + j];
            kp = _pext_u32(p, MP), kn = _pext_u32(p, MN);
            r4 = masked_as(r4, kp, kn, Xim);
            m4 = masked_as(m4, kp, kn, Xre);
        }
        const float* s = scales + (per_row ? 4 * i : 0);
        const float h1 = _mm512_reduce_add_ps(r1), h2 = _mm512_reduce_add_ps(r2),
                    h3 = _mm512_reduce_add_ps(r3), h4 = _mm512_reduce_add_ps(r4);
        const float g1 = _mm512_reduce_add_ps(m1), g2 = _mm512_reduce_add_ps(m2),
                    g3 = _mm512_reduce_add_ps(m3), g4 = _mm512_reduce_add_ps(m4);
        y[2 * i] = s[0] * h1 - s[1] * h2 + s[2] * h3 + s[3] * h4;        /* Eq. 2 */
        y[2 * i + 1] = conv == 0 ? s[0] * g1 + s[1] * g2 - s[2] * g3 + s[3] * g4  /* Eq. 1 */
                                 : s[0] * g1 + s[1] * g2 + s[2] * g3 - s[3] * g4; /* Eq. 3 */
    }
}

int wwc_wl_gemv(const uint32_t* planar, int64_t n, int64_t m, const float* scales, int per_row,
                int conv, const float* x, float* y, int nthreads) {
    if (!planar || !scales || !x || !y || n < 1 || m < 1 || (conv != 0 && conv != 1)) return -1;
    if (!wwc_supported()) return -2;
    const int64_t W = (m + 15) / 16;
    /* O2 layout: x_re, x_im as separate zero-padded fp32 arrays (once per call) */
    float* xre = (float*)aligned_alloc(64, (size_t)(64 * W));
    float* xim = (float*)aligned_alloc(64, (size_t)(64 * W));
    if (!xre || !xim) {
        free(xre), free(xim);
        return -1;
    }
    memset(xre, 0, (size_t)(64 * W));
    memset(xim, 0, (size_t)(64 * W));
    for (int64_t j = 0; j < m; ++j) {
        xre[j] = x[2 * j];
        xim[j] = x[2 * j + 1];
    }
#ifdef _OPENMP
    const int T = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel num_threads(T)
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
        rows(planar, n, W, scales, per_row, conv, xre, xim, y, t * n / nt, (t + 1) * n / nt);
    }
#else
    (void)nthreads;
    rows(planar, n, W, scales, per_row, conv, xre, xim, y, 0, n);
#endif
    free(xre), free(xim);
    return 0;
}
