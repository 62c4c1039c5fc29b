/* ww_inputs — seeded synthetic input generator shared by the oracle side and the
 * CUDA side of the WL-GEMV tests and benchmark.
 *
 * This module holds NO arithmetic of the method (no packing, no decode, no
 * accumulation, no scaling).  It only draws random numbers with the shapes and
 * distributions BASELINE.json's configs name:
 *
 *   ternary codes  t in {-1,0,+1}:  u < t0 -> 0 ; u < t1 -> +1 ; else -1
 *                  (config 1: t0=1/3, t1=2/3 ; configs 2-5: t0=0.4, t1=0.7)
 *   scales         lo + (hi-lo)*u, rounded to fp32
 *   activations    Box-Muller N(0,1) pairs, rounded to fp32 (host only)
 *
 * Generator: counter-based SplitMix64.  Draw k of stream s under seed S is
 *   key  = mix64(S + G*(s+1))
 *   h_k  = mix64(key + G*(k+1))          G = 0x9E3779B97F4A7C15
 *   u_k  = (h_k >> 11) * 2^-53           exact double in [0,1)
 * so any element can be regenerated independently (host C and device CUDA
 * implement the same formula; tests check they agree bit for bit).
 *
 * Stream numbering for one widely-linear layer:
 *   0..3 = code planes U_re, U_im, W_re, W_im   (index k = i*m + j)
 *   4    = scales                                (index k = i*4 + c, or c)
 *   5    = activation normals                    (pair index q = b*m + j)
 */
#ifndef WW_INPUTS_GEN_H
#define WW_INPUTS_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define WWI_STREAM_CODES(p) (p)
#define WWI_STREAM_SCALES 4
#define WWI_STREAM_X 5

uint64_t wwi_mix64(uint64_t z);
uint64_t wwi_draw(uint64_t seed, uint64_t stream, uint64_t k);
double   wwi_uniform(uint64_t seed, uint64_t stream, uint64_t k);
/* seed of projection `proj` (0..6 = q,k,v,o,gate,up,down) of decoder layer `layer` */
uint64_t wwi_layer_seed(uint64_t seed, int64_t layer, int64_t proj);

/* Dense ternary codes of one plane, rows [row0, row0+nrows) of an n x m plane,
 * written row-major with leading dimension ld (>= m). */
void wwi_gen_codes(uint64_t seed, uint64_t stream, int64_t m, int64_t row0, int64_t nrows,
                   double t0, double t1, int8_t* out, int64_t ld);
/* count fp32 draws lo + (hi-lo)*u_k, k = k0 .. k0+count-1 */
void wwi_gen_uniform_f32(uint64_t seed, uint64_t stream, int64_t k0, int64_t count,
                         double lo, double hi, float* out);
/* npairs complex N(0,1) values (re,im interleaved, fp32), pair index q0 .. q0+npairs-1 */
void wwi_gen_normal_c64(uint64_t seed, uint64_t stream, int64_t q0, int64_t npairs, float* out);

#ifdef __cplusplus
}
#endif
#endif
