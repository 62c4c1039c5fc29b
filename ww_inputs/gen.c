/* ww_inputs host generator (see gen.h).  Plain C99, no method arithmetic. */
#include "gen.h"
#include <math.h>

#define WWI_G 0x9E3779B97F4A7C15ULL

uint64_t wwi_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return wwi_mix64(seed + WWI_G * (stream + 1));
}

uint64_t wwi_draw(uint64_t seed, uint64_t stream, uint64_t k) {
    return wwi_mix64(stream_key(seed, stream) + WWI_G * (k + 1));
}

double wwi_uniform(uint64_t seed, uint64_t stream, uint64_t k) {
    return (double)(wwi_draw(seed, stream, k) >> 11) * 0x1.0p-53;
}

uint64_t wwi_layer_seed(uint64_t seed, int64_t layer, int64_t proj) {
    return seed ^ (WWI_G * (uint64_t)(7 * layer + proj + 1));
}

void wwi_gen_codes(uint64_t seed, uint64_t stream, int64_t m, int64_t row0, int64_t nrows,
                   double t0, double t1, int8_t* out, int64_t ld) {
    uint64_t key = stream_key(seed, stream);
    for (int64_t r = 0; r < nrows; ++r) {
        uint64_t base = (uint64_t)(row0 + r) * (uint64_t)m;
        for (int64_t j = 0; j < m; ++j) {
            double u = (double)(wwi_mix64(key + WWI_G * (base + (uint64_t)j + 1)) >> 11) * 0x1.0p-53;
            out[r * ld + j] = (int8_t)(u < t0 ? 0 : (u < t1 ? 1 : -1));
        }
    }
}

void wwi_gen_uniform_f32(uint64_t seed, uint64_t stream, int64_t k0, int64_t count,
                         double lo, double hi, float* out) {
    for (int64_t k = 0; k < count; ++k)
        out[k] = (float)(lo + (hi - lo) * wwi_uniform(seed, stream, (uint64_t)(k0 + k)));
}

void wwi_gen_normal_c64(uint64_t seed, uint64_t stream, int64_t q0, int64_t npairs, float* out) {
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t q = 0; q < npairs; ++q) {
        uint64_t k = 2 * (uint64_t)(q0 + q);
        double u1 = (double)((wwi_draw(seed, stream, k) >> 11) + 1) * 0x1.0p-53; /* (0,1] */
        double u2 = wwi_uniform(seed, stream, k + 1);
        double r = sqrt(-2.0 * log(u1));
        out[2 * q] = (float)(r * cos(two_pi * u2));
        out[2 * q + 1] = (float)(r * sin(two_pi * u2));
    }
}
