// HBM streaming rate of the WL-GEMV weight access pattern on B200: 148 CTAs x 16 warps, every
// warp reading its own contiguous range of the CTA's contiguous slab in 512-byte sweeps (one
// 16-byte load per lane), D sweeps in flight, versus warps of a CTA reading interleaved
// 512-byte pieces of the slab.  Total bytes = a gate/up-sized layer (22.5 MB), cold (a new
// region of a 1 GB buffer every launch).  GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ uint4 ldg_stream(const uint4* p){ uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];":"=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w):"l"(p)); return v; }

// MODE 0: per-warp contiguous ranges; MODE 1: CTA-interleaved sweeps
template<int D, int MODE>
__global__ void __launch_bounds__(512) stream(const uint4* base, size_t slab_chunks, unsigned* out){
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint4* slab = base + (size_t)blockIdx.x * slab_chunks;
  const size_t sweeps = slab_chunks / 32;          // 512-B sweeps in the slab
  const size_t per = sweeps / nw;                  // per warp
  unsigned acc = 0;
  uint4 q[D];
  auto addr = [&](size_t s) -> const uint4* {
    return MODE == 0 ? slab + ((size_t)warp * per + s) * 32 + lane : slab + (s * nw + warp) * 32 + lane;
  };
  #pragma unroll
  for (int d = 0; d < D; ++d) q[d] = ldg_stream(addr(d));
  for (size_t s = 0; s < per; s += D) {
    #pragma unroll
    for (int d = 0; d < D; ++d) {
      acc ^= q[d].x ^ q[d].y ^ q[d].z ^ q[d].w;
      if (s + D + d < per) q[d] = ldg_stream(addr(s + D + d));
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template<int D, int MODE>
double run(const uint4* buf, size_t total_chunks, size_t layer_chunks, unsigned* out, int nsm){
  const size_t slab = layer_chunks / nsm / 512 * 512;
  const int reps = (int)(total_chunks / (slab * nsm));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  stream<D, MODE><<<nsm, 512>>>(buf, slab, out);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) stream<D, MODE><<<nsm, 512>>>(buf + (size_t)r * slab * nsm, slab, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return (double)reps * slab * nsm * 16 / (ms * 1e-3) / 1e9;
}

int main(){
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)1 << 30;  // 1 GB
  uint4* buf; CK(cudaMalloc(&buf, total)); CK(cudaMemset(buf, 1, total));
  unsigned* out; CK(cudaMalloc(&out, 4));
  const size_t tc = total / 16, lc = (size_t)11008 * 128;  // gate/up layer: 11008 rows x 128 chunks
  printf("one launch over 1 GB (steady state):\n");
  printf("per-warp contiguous: D=1 %.0f  D=2 %.0f  D=4 %.0f  D=8 %.0f GB/s\n",
         run<1,0>(buf, tc, tc, out, nsm), run<2,0>(buf, tc, tc, out, nsm), run<4,0>(buf, tc, tc, out, nsm), run<8,0>(buf, tc, tc, out, nsm));
  printf("CTA-interleaved:     D=1 %.0f  D=2 %.0f  D=4 %.0f  D=8 %.0f GB/s\n",
         run<1,1>(buf, tc, tc, out, nsm), run<2,1>(buf, tc, tc, out, nsm), run<4,1>(buf, tc, tc, out, nsm), run<8,1>(buf, tc, tc, out, nsm));
  printf("gate/up-sized launches (22.5 MB each, back to back, no PDL):\n");
  printf("per-warp contiguous: D=1 %.0f  D=2 %.0f  D=4 %.0f  D=8 %.0f GB/s\n",
         run<1,0>(buf, tc, lc, out, nsm), run<2,0>(buf, tc, lc, out, nsm), run<4,0>(buf, tc, lc, out, nsm), run<8,0>(buf, tc, lc, out, nsm));
  printf("CTA-interleaved:     D=1 %.0f  D=2 %.0f  D=4 %.0f  D=8 %.0f GB/s\n",
         run<1,1>(buf, tc, lc, out, nsm), run<2,1>(buf, tc, lc, out, nsm), run<4,1>(buf, tc, lc, out, nsm), run<8,1>(buf, tc, lc, out, nsm));
  return 0;
}
