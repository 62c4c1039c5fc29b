// Can the FP64 pipe carry part of the ternary accumulation beside the FP32 pipe on sm_100a?
// Pure pipe rates (DADD, FADD2, mixes) and a realistic inner loop where planes 0..K-1 of a
// column accumulate with predicated FADD2 (fp32 pairs) and planes K..3 with predicated DADD
// (fp64, re and im separately).  Prints warp-instr/clk/SM and codes/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
constexpr int ITERS = 16384;

template<int KIND>
__global__ void pipe_kern(float* out, unsigned seed){
  unsigned long long a[8]; double d[8];
  const unsigned long long X = 0x3f8000013f800001ull + threadIdx.x;
  const double XD = 1.0 + threadIdx.x * 1e-9;
  #pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = i; d[i] = i * 0.5; }
  for (int it = 0; it < ITERS; ++it) {
    if (KIND == 0) {        // DADD x16
      #pragma unroll
      for (int k = 0; k < 2; ++k)
      #pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(XD));
    } else if (KIND == 1) { // FADD2 x8 + DADD x8 interleaved
      #pragma unroll
      for (int i = 0; i < 8; ++i) {
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X));
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(XD));
      }
    } else if (KIND == 2) { // FADD2 x8 + DADD x4
      #pragma unroll
      for (int i = 0; i < 8; ++i) {
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X));
        if (i & 1) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(XD));
      }
    } else if (KIND == 3) { // FADD2 x16
      #pragma unroll
      for (int k = 0; k < 2; ++k)
      #pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X));
    } else if (KIND == 4) { // FADD2 x8 + DADD x2
      #pragma unroll
      for (int i = 0; i < 8; ++i) {
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X));
        if ((i & 3) == 3) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(XD));
      }
    }
  }
  double t = 0;
  #pragma unroll
  for (int i = 0; i < 8; ++i) t += (double)(a[i] & 0xffff) + d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)t;
}

// realistic: K planes by predicated FADD2, 4-K planes by predicated DADD (re, im separately)
template<int K>
__global__ void tern_kern(float* out){
  __shared__ uint4 wsm[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    unsigned h = (i * 2654435761u) ^ 0x1234567u; uint4 q;
    unsigned a = h * 0x9E3779B9u, b = h * 0x85EBCA6Bu, c = h * 0xC2B2AE35u, d = h * 0x27D4EB2Fu;
    q.x = (a & 0xAAAAAAAAu) | ((~(a >> 1)) & b & 0x55555555u); q.y = (b & 0xAAAAAAAAu) | ((~(b >> 1)) & c & 0x55555555u);
    q.z = (c & 0xAAAAAAAAu) | ((~(c >> 1)) & d & 0x55555555u); q.w = (d & 0xAAAAAAAAu) | ((~(d >> 1)) & a & 0x55555555u);
    wsm[i] = q;   // COL4-like: byte k = column k's 8 bits (2 per plane)
  }
  __syncthreads();
  float2 X[16]; double XR[16], XI[16];
  #pragma unroll
  for (int k = 0; k < 16; ++k) {
    X[k] = make_float2(1.0f + k * 0.001f + threadIdx.x * 1e-6f, 2.0f - k * 0.001f);
    XR[k] = X[k].x; XI[k] = X[k].y;
  }
  float2 acc[4]; double accr[4], acci[4];
  #pragma unroll
  for (int p = 0; p < 4; ++p) { acc[p] = make_float2(0.f, 0.f); accr[p] = 0; acci[p] = 0; }
  for (int it = 0; it < ITERS / 4; ++it) {
    const uint4 q = wsm[(it * 7 + threadIdx.x) & 255];
    const unsigned w[4] = {q.x, q.y, q.z, q.w};
    #pragma unroll
    for (int k = 0; k < 16; ++k) {
      const unsigned bits = (w[k >> 2] >> (8 * (k & 3))) & 0xffu;
      const float2 x = X[k], nx = make_float2(-x.x, -x.y);
      #pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int p = b >> 1;
        if (bits & (1u << b)) {
          if (p < K) acc[p] = __fadd2_rn(acc[p], (b & 1) ? x : nx);
          else if (b & 1) { accr[p] += XR[k]; acci[p] += XI[k]; }
          else { accr[p] -= XR[k]; acci[p] -= XI[k]; }
        }
      }
    }
  }
  double t = 0;
  #pragma unroll
  for (int p = 0; p < 4; ++p) t += acc[p].x + acc[p].y + accr[p] + acci[p];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)t;
}

template<typename F>
double time_it(F launch){
  launch(); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best * 1e-3;
}

int main(){
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; CK(cudaMalloc(&out, sizeof(float) * nsm * 2048));
  const double clk = 1.965e9;
  const int threads = 256, blocks = nsm * 8;  // 64 warps/SM
  auto wi = [&](double s, int ops){ return (double)blocks * threads / 32 * ITERS * ops / s / nsm / clk; };
  printf("pipe rates (warp-instr/clk/SM @1.965 GHz, 64 warps/SM):\n");
  printf("  DADD x16            %.3f\n", wi(time_it([&]{ pipe_kern<0><<<blocks, threads>>>(out, 1); }), 16));
  printf("  FADD2 x16           %.3f\n", wi(time_it([&]{ pipe_kern<3><<<blocks, threads>>>(out, 1); }), 16));
  printf("  FADD2 x8 + DADD x8  %.3f (total)\n", wi(time_it([&]{ pipe_kern<1><<<blocks, threads>>>(out, 1); }), 16));
  printf("  FADD2 x8 + DADD x4  %.3f (total)\n", wi(time_it([&]{ pipe_kern<2><<<blocks, threads>>>(out, 1); }), 12));
  printf("  FADD2 x8 + DADD x2  %.3f (total)\n", wi(time_it([&]{ pipe_kern<4><<<blocks, threads>>>(out, 1); }), 10));
  for (int bps : {1, 2, 4, 8}) {
    const int b = nsm * bps, t = 128;  // 4 warps per block
    const double codes = (double)b * t * (ITERS / 4) * 64;
    double s4 = time_it([&]{ tern_kern<4><<<b, t>>>(out); });
    double s3 = time_it([&]{ tern_kern<3><<<b, t>>>(out); });
    double s2 = time_it([&]{ tern_kern<2><<<b, t>>>(out); });
    printf("warps/SM=%2d  codes/clk/SM: fp32 only %.1f   3 fp32 + 1 fp64 planes %.1f   2 + 2 %.1f\n",
           bps * 4, codes / s4 / nsm / clk, codes / s3 / nsm / clk, codes / s2 / nsm / clk);
  }
  return 0;
}
