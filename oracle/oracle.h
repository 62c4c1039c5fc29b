/* oracle.h — plain, slow, obviously-correct CPU oracle for the FairyFuse fused
 * ternary widely-linear GEMV (arXiv 2604.20913).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the product
 * (paper_2604_20913_b200/, include/ww.h) and neither side includes the other.
 *
 * Arithmetic is IEEE fp64 throughout; fp32 inputs (scales, activations) are
 * promoted exactly.  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
 *
 * Readings of the paper (DESIGN.md "Readings" R1-R6):
 *  - conv ORC_CONV_EQ1  : y = U x + W conj(x)                      Eq. 1
 *    conv ORC_CONV_ALG1 : y = (U + conj(W)) x  == Eqs. 2-3, Alg. 1
 *  - U = sUr*U_re + i*sUi*U_im,  W = sWr*W_re + i*sWi*W_im
 *    scales per row (n x 4 floats [sUr,sUi,sWr,sWi]) or per tensor (4 floats)
 *  - code (b1,b0): (1,0)=+1, (0,1)=-1, (0,0)=0, (1,1) unused -> rejected
 *  - slot k of a word: bit 2k+1 = "+1", bit 2k = "-1"
 *  - planes stored U_re, U_im, W_re, W_im, each row-major n x ceil(m/16) words
 *                                                                     P:588-590
 * Every entry point returns 0 on success and a negative code on bad input:
 *   -1 invalid argument, -2 invalid encoding (slot (1,1)), -3 out of memory.
 */
#ifndef WW_ORACLE_H
#define WW_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORC_CONV_EQ1 0
#define ORC_CONV_ALG1 1
#define ORC_SCALES_PER_TENSOR 0
#define ORC_SCALES_PER_ROW 1

int64_t orc_words_per_row(int64_t m);

/* App. H packing equation: packed = sum_k [t_k=+1] 2^(2k+1) + [t_k=-1] 2^(2k). */
int orc_pack_slots(const int8_t t[16], uint32_t* out);
/* inverse; -2 if any slot is (1,1) ("unused") */
int orc_unpack_slots(uint32_t p, int8_t t[16]);
/* Eqs. 4-5: k_pos = pext(p, 0xAAAAAAAA), k_neg = pext(p, 0x55555555),
 * pext written out as its definition (a bit loop). */
void orc_decode_masks(uint32_t p, uint32_t* k_pos, uint32_t* k_neg);

/* One plane: dense int8 n x m (leading dim ld) <-> n x ceil(m/16) words, zero-code padding. */
int orc_pack_plane(const int8_t* dense, int64_t n, int64_t m, int64_t ld, uint32_t* words);
int orc_unpack_plane(const uint32_t* words, int64_t n, int64_t m, int8_t* dense, int64_t ld);

/* Direct evaluation of the widely-linear map (P:1435 / P:1447-1452) for the
 * listed rows.  planar = 4 planes back to back (4*n*ceil(m/16) words).
 * x: B vectors of m complex64 (re,im interleaved), vector b at x + 2*m*b.
 * y: B x nrows complex128 (re,im interleaved), y[(b*nrows + r)*2 + {0,1}].
 * rows == NULL means rows 0..nrows-1. */
int orc_wl_direct(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                  int scale_mode, int conv, const float* x, int64_t B, const int64_t* rows,
                  int64_t nrows, double* y);

/* Same map through the real 2n x 2m embedding [[A,B],[C,D]] built with explicit
 * multiplies; an evaluation path independent of the complex one. */
int orc_wl_embedding(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                     int scale_mode, int conv, const float* x, int64_t B, const int64_t* rows,
                     int64_t nrows, double* y);

/* Algorithm 1 step by step for one vector, in fp64: 8 accumulators of 16
 * lanes, pext masks, MaskedAS = Eq. 6 then Eq. 7, hsum, weighted sums.  Computes the
 * ALG1 convention only (the algorithm as printed).  Counts (may be NULL):
 *   counts[0] element add/sub slots   (16 per MaskedAS: the App. D count)
 *   counts[1] lanes actually added    (k_pos bits)
 *   counts[2] lanes actually subtracted (k_neg bits)
 *   counts[3] scale multiplies        (8 per row)
 *   counts[4] multiplies inside the chunk loop (always 0) */
int orc_wl_alg1(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                int scale_mode, const float* x, const int64_t* rows, int64_t nrows, double* y,
                int64_t counts[5]);

/* The same map as orc_wl_direct in two phases (for timing them separately):
 * orc_build_dense unpacks the listed rows and builds the dense complex rows of U and W
 * as nrows x m complex128 (re,im interleaved) in U and Wd; orc_eval_dense
 * evaluates Eq. 1 (EQ1) or Eqs. 2-3 (ALG1) on them, left to right -- bitwise the result of
 * orc_wl_direct.  Rows are independent: liboracle_omp.so (built with -fopenmp) splits them
 * over threads, with results independent of the thread count. */
int orc_build_dense(const uint32_t* planar, int64_t n, int64_t m, const float* scales,
                    int scale_mode, const int64_t* rows, int64_t nrows, double* U, double* Wd);
int orc_eval_dense(const double* U, const double* Wd, int64_t nrows, int64_t m, int conv,
                   const float* x, int64_t B, double* y);
/* threads the library will use (1 unless built with OpenMP) */
int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
