/* oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C99, fp64, slow on
 * purpose: every function follows the paper's definition in the paper's order so
 * it can be checked against PAPER.md by eye.  No blocking, no fusion, no SIMD. */
#include "oracle.h"
#include <complex.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int64_t orc_words_per_row(int64_t m) { return (m + 15) / 16; }

/* App. H */
int orc_pack_slots(const int8_t t[16], uint32_t* out) {
    uint32_t packed = 0;
    for (int k = 0; k < 16; ++k) {
        if (t[k] == 1)
            packed += (uint32_t)1 << (2 * k + 1);
        else if (t[k] == -1)
            packed += (uint32_t)1 << (2 * k);
        else if (t[k] != 0)
            return -1;
    }
    *out = packed;
    return 0;
}

/* inverse of App. H; (1,1) is "unused" and therefore rejected */
int orc_unpack_slots(uint32_t p, int8_t t[16]) {
    for (int k = 0; k < 16; ++k) {
        int pos = (p >> (2 * k + 1)) & 1;
        int neg = (p >> (2 * k)) & 1;
        if (pos && neg) return -2;
        t[k] = (int8_t)(pos - neg);
    }
    return 0;
}

/* pext(src, mask): the bits of src selected by mask, packed LSB-first (its definition) */
static uint32_t pext32(uint32_t src, uint32_t mask) {
    uint32_t out = 0;
    int o = 0;
    for (int b = 0; b < 32; ++b) {
        if ((mask >> b) & 1) {
            out |= ((src >> b) & 1u) << o;
            ++o;
        }
    }
    return out;
}

/* Eqs. 4-5 */
void orc_decode_masks(uint32_t p, uint32_t* k_pos, uint32_t* k_neg) {
    *k_pos = pext32(p, 0xAAAAAAAAu);
    *k_neg = pext32(p, 0x55555555u);
}

int orc_pack_plane(const int8_t* dense, int64_t n, int64_t m, int64_t ld, uint32_t* words) {
    if (n < 0 || m < 0 || ld < m || (!dense && n * m != 0) || (!words && n * m != 0)) return -1;
    const int64_t W = orc_words_per_row(m);
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t c = 0; c < W; ++c) {
            int8_t t[16];
            for (int k = 0; k < 16; ++k) {
                int64_t j = 16 * c + k;
                t[k] = j < m ? dense[i * ld + j] : 0; /* zero-code padding */
            }
            if (orc_pack_slots(t, &words[i * W + c]) != 0) return -1;
        }
    }
    return 0;
}

int orc_unpack_plane(const uint32_t* words, int64_t n, int64_t m, int8_t* dense, int64_t ld) {
    if (n < 0 || m < 0 || ld < m) return -1;
    const int64_t W = orc_words_per_row(m);
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t c = 0; c < W; ++c) {
            int8_t t[16];
            if (orc_unpack_slots(words[i * W + c], t) != 0) return -2;
            for (int k = 0; k < 16; ++k) {
                int64_t j = 16 * c + k;
                if (j < m) dense[i * ld + j] = t[k];
            }
        }
    }
    return 0;
}

/* the four scales of row i: [sUr, sUi, sWr, sWi] */
static void row_scales(const float* scales, int scale_mode, int64_t i, double s[4]) {
    const float* p = scale_mode == ORC_SCALES_PER_ROW ? scales + 4 * i : scales;
    for (int c = 0; c < 4; ++c) s[c] = (double)p[c];
}

/* unpack the four planes of row i into dense int8 rows t[4][m]; -2 on (1,1) */
static int unpack_row(const uint32_t* planar, int64_t n, int64_t m, int64_t i, int8_t* t) {
    const int64_t W = orc_words_per_row(m);
    for (int p = 0; p < 4; ++p) {
        int rc = orc_unpack_plane(planar + ((int64_t)p * n + i) * W, 1, m, t + p * m, m);
        if (rc != 0) return rc;
    }
    return 0;
}

static int check_args(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                      int scale_mode, int conv, const float* x, int64_t B, const int64_t* rows,
                      int64_t nrows, const double* y) {
    if (!planar || !scales || !x || !y || n < 1 || m < 1 || B < 1 || nrows < 0) return -1;
    if (scale_mode != ORC_SCALES_PER_ROW && scale_mode != ORC_SCALES_PER_TENSOR) return -1;
    if (conv != ORC_CONV_EQ1 && conv != ORC_CONV_ALG1) return -1;
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows ? rows[r] : r;
        if (i < 0 || i >= n) return -1;
    }
    return 0;
}

int orc_wl_direct(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                  int scale_mode, int conv, const float* x, int64_t B, const int64_t* rows,
                  int64_t nrows, double* y) {
    int rc = check_args(planar, n, m, scales, scale_mode, conv, x, B, rows, nrows, y);
    if (rc) return rc;
    int8_t* t = (int8_t*)malloc((size_t)(4 * m));
    double complex* U = (double complex*)malloc(sizeof(double complex) * (size_t)m);
    double complex* Wm = (double complex*)malloc(sizeof(double complex) * (size_t)m);
    if (!t || !U || !Wm) {
        free(t), free(U), free(Wm);
        return -3;
    }
    for (int64_t r = 0; r < nrows && rc == 0; ++r) {
        const int64_t i = rows ? rows[r] : r;
        rc = unpack_row(planar, n, m, i, t);
        if (rc) break;
        double s[4];
        row_scales(scales, scale_mode, i, s);
        /* dense complex rows U_i. and W_i. */
        for (int64_t j = 0; j < m; ++j) {
            U[j] = s[0] * t[0 * m + j] + I * (s[1] * t[1 * m + j]);
            Wm[j] = s[2] * t[2 * m + j] + I * (s[3] * t[3 * m + j]);
        }
        for (int64_t b = 0; b < B; ++b) {
            const float* xb = x + 2 * m * b;
            double complex acc = 0;
            for (int64_t j = 0; j < m; ++j) { /* left to right */
                double complex xj = (double)xb[2 * j] + I * (double)xb[2 * j + 1];
                if (conv == ORC_CONV_EQ1)
                    acc += U[j] * xj + Wm[j] * conj(xj);      /* Eq. 1 */
                else
                    acc += (U[j] + conj(Wm[j])) * xj;         /* Eqs. 2-3 */
            }
            y[2 * (b * nrows + r)] = creal(acc);
            y[2 * (b * nrows + r) + 1] = cimag(acc);
        }
    }
    free(t), free(U), free(Wm);
    return rc;
}

int orc_wl_embedding(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                     int scale_mode, int conv, const float* x, int64_t B, const int64_t* rows,
                     int64_t nrows, double* y) {
    int rc = check_args(planar, n, m, scales, scale_mode, conv, x, B, rows, nrows, y);
    if (rc) return rc;
    int8_t* t = (int8_t*)malloc((size_t)(4 * m));
    double* E = (double*)malloc(sizeof(double) * (size_t)(4 * m)); /* row i of A,B,C,D */
    if (!t || !E) {
        free(t), free(E);
        return -3;
    }
    double *A = E, *Bm = E + m, *C = E + 2 * m, *D = E + 3 * m;
    for (int64_t r = 0; r < nrows && rc == 0; ++r) {
        const int64_t i = rows ? rows[r] : r;
        rc = unpack_row(planar, n, m, i, t);
        if (rc) break;
        double s[4]; /* a, b, c, d = sUr, sUi, sWr, sWi */
        row_scales(scales, scale_mode, i, s);
        for (int64_t j = 0; j < m; ++j) {
            const double ur = t[j], ui = t[m + j], wr = t[2 * m + j], wi = t[3 * m + j];
            A[j] = s[0] * ur + s[2] * wr;
            Bm[j] = -s[1] * ui + s[3] * wi;
            if (conv == ORC_CONV_EQ1) {
                C[j] = s[1] * ui + s[3] * wi;
                D[j] = s[0] * ur - s[2] * wr;
            } else {
                C[j] = s[1] * ui - s[3] * wi;
                D[j] = s[0] * ur + s[2] * wr;
            }
        }
        for (int64_t b = 0; b < B; ++b) {
            const float* xb = x + 2 * m * b;
            double yre = 0, yim = 0;
            for (int64_t j = 0; j < m; ++j) {
                const double xr = xb[2 * j], xi = xb[2 * j + 1];
                yre += A[j] * xr + Bm[j] * xi;
                yim += C[j] * xr + D[j] * xi;
            }
            y[2 * (b * nrows + r)] = yre;
            y[2 * (b * nrows + r) + 1] = yim;
        }
    }
    free(t), free(E);
    return rc;
}

/* MaskedAS(a, k+, k-, X): Eq. 6 then Eq. 7 on 16 lanes */
static void masked_as(double a[16], uint32_t kp, uint32_t kn, const double X[16],
                      int64_t* counts) {
    for (int l = 0; l < 16; ++l)
        if ((kp >> l) & 1) a[l] = a[l] + X[l]; /* _mm512_mask_add_ps */
    for (int l = 0; l < 16; ++l)
        if ((kn >> l) & 1) a[l] = a[l] - X[l]; /* _mm512_mask_sub_ps */
    if (counts) {
        counts[0] += 16;
        for (int l = 0; l < 16; ++l) {
            counts[1] += (kp >> l) & 1;
            counts[2] += (kn >> l) & 1;
        }
    }
}

static double hsum(const double a[16]) {
    double s = 0;
    for (int l = 0; l < 16; ++l) s += a[l];
    return s;
}

int orc_wl_alg1(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                int scale_mode, const float* x, const int64_t* rows, int64_t nrows, double* y,
                int64_t counts[5]) {
    int rc = check_args(planar, n, m, scales, scale_mode, ORC_CONV_ALG1, x, 1, rows, nrows, y);
    if (rc) return rc;
    const int64_t W = orc_words_per_row(m);
    /* x_re, x_im zero-padded to 16*W; neg_x_im of O3 is loaded by Alg. 1 but unused
     * by its displayed updates (R4), so it is not formed here. */
    double* xre = (double*)calloc((size_t)(16 * W), sizeof(double));
    double* xim = (double*)calloc((size_t)(16 * W), sizeof(double));
    if (!xre || !xim) {
        free(xre), free(xim);
        return -3;
    }
    for (int64_t j = 0; j < m; ++j) {
        xre[j] = x[2 * j];
        xim[j] = x[2 * j + 1];
    }
    if (counts) memset(counts, 0, 5 * sizeof(int64_t));
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = rows ? rows[r] : r;
        double are[4][16], aim[4][16];
        memset(are, 0, sizeof are);
        memset(aim, 0, sizeof aim);
        for (int64_t j = 0; j < W; ++j) {
            const double* Xre = xre + 16 * j; /* O2 */
            const double* Xim = xim + 16 * j;
            uint32_t kp, kn, p;
            int8_t chk[16];
            for (int q = 0; q < 4; ++q) {
                p = planar[((int64_t)q * n + i) * W + j];
                if (orc_unpack_slots(p, chk) != 0) { /* (1,1) is not a valid code */
                    free(xre), free(xim);
                    return -2;
                }
                orc_decode_masks(p, &kp, &kn); /* O1 */
                /* U_re: (x_re, x_im); U_im: (x_im, x_re); W_re: (x_re, x_im); W_im: (x_im, x_re) */
                const double* Xa = (q == 0 || q == 2) ? Xre : Xim;
                const double* Xb = (q == 0 || q == 2) ? Xim : Xre;
                masked_as(are[q], kp, kn, Xa, counts);
                masked_as(aim[q], kp, kn, Xb, counts);
            }
        }
        double s[4];
        row_scales(scales, scale_mode, i, s);
        /* weighted horizontal sums */
        y[2 * r] = s[0] * hsum(are[0]) - s[1] * hsum(are[1]) + s[2] * hsum(are[2]) +
                   s[3] * hsum(are[3]);
        y[2 * r + 1] = s[0] * hsum(aim[0]) + s[1] * hsum(aim[1]) + s[2] * hsum(aim[2]) -
                       s[3] * hsum(aim[3]);
        if (counts) counts[3] += 8;
    }
    free(xre), free(xim);
    return 0;
}

/* ---- Dense two-phase form of orc_wl_direct, for timing the CPU baseline's phases
 * separately ((a) unpack + build dense, (b) evaluate).  Same arithmetic, same
 * order as orc_wl_direct.  Rows are independent, so an OpenMP build (-fopenmp,
 * liboracle_omp.so) splits them over threads; results do not depend on the thread count. */

int orc_build_dense(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                    int scale_mode, const int64_t* rows, int64_t nrows, double* U, double* Wd) {
    if (!planar || !scales || !U || !Wd || n < 1 || m < 1 || nrows < 0) return -1;
    if (scale_mode != ORC_SCALES_PER_ROW && scale_mode != ORC_SCALES_PER_TENSOR) return -1;
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows ? rows[r] : r;
        if (i < 0 || i >= n) return -1;
    }
    int rc = 0;
#pragma omp parallel for schedule(static) reduction(min : rc)
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = rows ? rows[r] : r;
        int8_t* t = (int8_t*)malloc((size_t)(4 * m));
        if (!t) {
            rc = -3;
            continue;
        }
        const int ur = unpack_row(planar, n, m, i, t);
        if (ur != 0) {
            rc = ur < rc ? ur : rc;
            free(t);
            continue;
        }
        double s[4];
        row_scales(scales, scale_mode, i, s);
        double complex* Ur = (double complex*)(U + 2 * m * r);
        double complex* Wr = (double complex*)(Wd + 2 * m * r);
        for (int64_t j = 0; j < m; ++j) {
            Ur[j] = s[0] * t[0 * m + j] + I * (s[1] * t[1 * m + j]);
            Wr[j] = s[2] * t[2 * m + j] + I * (s[3] * t[3 * m + j]);
        }
        free(t);
    }
    return rc;
}

int orc_eval_dense(const double* U, const double* Wd, int64_t nrows, int64_t m, int conv,
                   const float* x, int64_t B, double* y) {
    if (!U || !Wd || !x || !y || nrows < 0 || m < 1 || B < 1) return -1;
    if (conv != ORC_CONV_EQ1 && conv != ORC_CONV_ALG1) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {
        const double complex* Ur = (const double complex*)(U + 2 * m * r);
        const double complex* Wr = (const double complex*)(Wd + 2 * m * r);
        for (int64_t b = 0; b < B; ++b) {
            const float* xb = x + 2 * m * b;
            double complex acc = 0;
            for (int64_t j = 0; j < m; ++j) { /* left to right */
                double complex xj = (double)xb[2 * j] + I * (double)xb[2 * j + 1];
                if (conv == ORC_CONV_EQ1)
                    acc += Ur[j] * xj + Wr[j] * conj(xj); /* Eq. 1 */
                else
                    acc += (Ur[j] + conj(Wr[j])) * xj;    /* Eqs. 2-3 */
            }
            y[2 * (b * nrows + r)] = creal(acc);
            y[2 * (b * nrows + r) + 1] = cimag(acc);
        }
    }
    return 0;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
