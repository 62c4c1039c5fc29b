// Would a shared-memory LUT for one plane lift the B=1 inner loop?  Baseline: the product's
// chunk (COL4 byte per column, R2P + bit test, 8 predicated FADD2 per column).  Hybrid:
// planes 0-2 predicated (R2P of 6 bits, no bit test) + plane 3 from a lane-interleaved table
// of 4-column subset sums (pos / neg nibbles of an extra PN16 word -> PRMT address, LDS.64,
// one FADD2 per 2 codes).  Weights and x from shared memory; codes/clk/SM at 1.965 GHz.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
constexpr int TC = 64;       // chunks of x in smem (1024 columns)
constexpr int ITERS = 2048;

__device__ __forceinline__ float4 lds128(uint32_t a){ float4 v; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];":"=f"(v.x),"=f"(v.y),"=f"(v.z),"=f"(v.w):"r"(a)); return v; }
__device__ __forceinline__ float2 lds64(uint32_t a){ float2 v; asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];":"=f"(v.x),"=f"(v.y):"r"(a)); return v; }
__device__ __forceinline__ uint4 lds128u(uint32_t a){ uint4 v; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];":"=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w):"r"(a)); return v; }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b){ return __fadd2_rn(a,b); }

template <int NP>  // NP predicated planes per column (4 = product, 3 = hybrid)
__device__ __forceinline__ void column(float2 (&acc)[4], uint32_t bits, float2 x) {
  const float2 nx = make_float2(-x.x, -x.y);
#pragma unroll
  for (int k = 0; k < 2 * NP; ++k) {
    const int q = k >> 1;
    if (bits & (1u << k)) acc[q] = fadd2(acc[q], (k & 1) ? x : nx);
  }
}

template <int HYB>
__global__ void __launch_bounds__(512, 2) kern(float* out) {
  extern __shared__ __align__(4096) unsigned char sm[];
  // x: TC chunks x 128 B (swizzled); table: TC/32 sweeps x 4 groups x 16 entries x 32 lanes x 8 B
  const uint32_t xs = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t tb = xs + TC * 128;                      // 4096-aligned
  const uint32_t wsm = tb + (TC / 32) * 4 * 16 * 32 * 8;  // weights: 8 rows x TC chunks x 20 B
  for (int i = threadIdx.x; i < TC * 32; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f + (i % 97) * 0.01f;
  for (int i = threadIdx.x; i < (TC / 32) * 4 * 16 * 32 * 2; i += blockDim.x)
    reinterpret_cast<float*>(sm + TC * 128)[i] = 0.5f + (i % 89) * 0.01f;
  unsigned* ws = reinterpret_cast<unsigned*>(sm + (wsm - xs));
  for (int i = threadIdx.x; i < 8 * TC * 5; i += blockDim.x) {
    unsigned h = (i * 2654435761u) ^ 0x9e3779b9u; h ^= h >> 15; h *= 0x85ebca6bu; h ^= h >> 13;
    unsigned pos = h & 0xAAAAAAAAu, h2 = h * 0xc2b2ae35u, neg = (h2 & 0x55555555u) & ~(pos >> 1);
    ws[i] = (i % 5 == 4) ? ((h & 0xffffu) | ((h2 & ~h & 0xffffu) << 16)) : (pos | neg);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2 acc[2][4];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[s][q] = make_float2(0, 0);
  const uint32_t l7 = (uint32_t)(lane & 7) << 4;
  for (int it = 0; it < ITERS; ++it) {
    const int tc = (lane + 32 * it) & (TC - 1);
    const int row = (warp + it) & 7;
    const uint32_t wa = wsm + (uint32_t)((row * TC + tc) * 20);
    const uint4 w = lds128u(wa & ~15u);  // (misaligned rows fold onto aligned reads: rate test only)
    const uint32_t a3 = *reinterpret_cast<const unsigned*>(sm + (wa - xs) + 16 - ((wa & 15u)));
    const uint32_t xc = (xs + (uint32_t)tc * 128u) | l7;
    const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t word = w4[kk >> 1], sh = (kk & 1) * 16;
      const float4 v = lds128(xc ^ ((uint32_t)kk << 4));
      if (HYB) {
        column<3>(acc[0], (word >> sh) & 0x3fu, make_float2(v.x, v.y));
        column<3>(acc[1], (word >> (sh + 8)) & 0x3fu, make_float2(v.z, v.w));
      } else {
        column<4>(acc[0], (word >> sh) & 0xffu, make_float2(v.x, v.y));
        column<4>(acc[1], (word >> (sh + 8)) & 0xffu, make_float2(v.z, v.w));
      }
    }
    if (HYB) {  // plane 3 via the table: 8 lookups per 16 columns
      const uint32_t base = tb + (uint32_t)(((tc >> 5) * 4) * 16 * 32 * 8) + (uint32_t)lane * 8u;
      const uint32_t lo = a3 & 0x0F0F0F0Fu, hi = (a3 >> 4) & 0x0F0F0F0Fu;
      // bytes of lo: pos g0, pos g2, neg g0, neg g2; hi: pos g1, pos g3, neg g1, neg g3
      float2 p0 = lds64(__byte_perm(lo, base, 0x7604) + 0 * 4096);
      float2 p1 = lds64(__byte_perm(hi, base, 0x7604) + 1 * 4096);
      float2 p2 = lds64(__byte_perm(lo, base, 0x7614) + 2 * 4096);
      float2 p3 = lds64(__byte_perm(hi, base, 0x7614) + 3 * 4096);
      float2 n0 = lds64(__byte_perm(lo, base, 0x7624) + 0 * 4096);
      float2 n1 = lds64(__byte_perm(hi, base, 0x7624) + 1 * 4096);
      float2 n2 = lds64(__byte_perm(lo, base, 0x7634) + 2 * 4096);
      float2 n3 = lds64(__byte_perm(hi, base, 0x7634) + 3 * 4096);
      acc[0][3] = fadd2(acc[0][3], p0); acc[1][3] = fadd2(acc[1][3], p1);
      acc[0][3] = fadd2(acc[0][3], p2); acc[1][3] = fadd2(acc[1][3], p3);
      acc[0][3] = fadd2(acc[0][3], make_float2(-n0.x, -n0.y)); acc[1][3] = fadd2(acc[1][3], make_float2(-n1.x, -n1.y));
      acc[0][3] = fadd2(acc[0][3], make_float2(-n2.x, -n2.y)); acc[1][3] = fadd2(acc[1][3], make_float2(-n3.x, -n3.y));
    }
  }
  float t = 0;
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) t += acc[s][q].x + acc[s][q].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; CK(cudaMalloc(&out, sizeof(float) * nsm * 2 * 512));
  const size_t smem = TC * 128 + (TC / 32) * 4 * 16 * 32 * 8 + 8 * TC * 20 + 64;
  CK(cudaFuncSetAttribute(kern<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int ctas : {1, 2}) {
    for (int hyb = 0; hyb < 2; ++hyb) {
      auto launch = [&] { if (hyb) kern<1><<<nsm * ctas, 512, smem>>>(out); else kern<0><<<nsm * ctas, 512, smem>>>(out); };
      launch(); CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
      const double codes = (double)nsm * ctas * 512 * ITERS * 64;
      printf("%s  CTAs/SM=%d (warps/SM=%d): %.1f codes/clk/SM\n", hyb ? "hybrid (3 pred + 1 LUT plane)" : "product chunk (4 pred planes)", ctas, ctas * 16, codes / (best * 1e-3) / nsm / 1.965e9);
    }
  }
  return 0;
}
