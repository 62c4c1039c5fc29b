// ww_inputs device generator: the same counter-based SplitMix64 code draw as
// gen.c, run on the GPU so the benchmark's 1.6 GB decode stack can be made in
// HBM without a host round trip.  No method arithmetic lives here.
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr uint64_t kG = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void gen_codes_kernel(uint64_t key, int64_t m, int64_t row0, int64_t nrows,
                                 double t0, double t1, int8_t* __restrict__ out, int64_t ld) {
    const int64_t total = nrows * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / m, j = e - r * m;
        const uint64_t k = (uint64_t)(row0 + r) * (uint64_t)m + (uint64_t)j;
        const double u = (double)(mix64(key + kG * (k + 1)) >> 11) * 0x1.0p-53;
        out[r * ld + j] = (int8_t)(u < t0 ? 0 : (u < t1 ? 1 : -1));
    }
}
}  // namespace

extern "C" int wwi_gen_codes_device(uint64_t seed, uint64_t stream, int64_t m, int64_t row0,
                                    int64_t nrows, double t0, double t1, int8_t* out_d,
                                    int64_t ld, void* cuda_stream) {
    if (nrows <= 0 || m <= 0) return 0;
    const uint64_t key = mix64(seed + kG * (stream + 1));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    gen_codes_kernel<<<sms * 8, 256, 0, (cudaStream_t)cuda_stream>>>(key, m, row0, nrows, t0, t1,
                                                                     out_d, ld);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
