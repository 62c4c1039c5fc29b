// Shared-memory lookup-table (LUT) inner loops for the ternary WL-GEMV on sm_100a:
// can "one LDS.64 of a 16-entry subset-sum table + one FADD2 per 4-column nibble" beat the
// predicated-FADD2 datapath (chunk_rate.cu, ~25 codes/clk/SM)?
//
// Table layout under test: for every group of 4 columns one 128-byte table of 16 float2
// entries, entry e = sum_{k: bit k of e} (x_re, x_im)_k.  A lane = one output row; all 32
// lanes of a warp read the same table at a time, so a warp's LDS.64 touches <= 16 distinct
// 8-byte entries = at most one word per bank.  The weight word of one plane covers 16
// columns: bits 0..15 = "+1" bits, bits 16..31 = "-1" bits (a bit permutation of App. H).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
constexpr int NG = 256;          // 4-column groups in the table = 1024 columns, 32 KB
constexpr int NCH = NG / 4;      // 16-column chunks
constexpr int ITERS = 4096;      // chunks per warp

__device__ __forceinline__ float2 lds64(uint32_t a){ float2 v; asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];":"=f"(v.x),"=f"(v.y):"r"(a)); return v; }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b){ return __fadd2_rn(a,b); }
__device__ __forceinline__ float2 fsub2(float2 a, float2 b){ return __fadd2_rn(a,make_float2(-b.x,-b.y)); }
__device__ __forceinline__ uint4 ldg_stream(const uint4* p){ uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];":"=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w):"l"(p)); return v; }

// one plane word (16 columns = 4 groups) against the 4 tables at tb (1 KB aligned chunk base)
template<int V>
__device__ __forceinline__ void plane(float2& acc, float2& accn, uint32_t w, uint32_t tb){
  if (V == 0) {  // PRMT: spread nibbles to bytes (x8), then one PRMT per lookup builds the address
    const uint32_t lo = (w << 3) & 0x78787878u;   // bytes: pos g0, pos g2, neg g0, neg g2
    const uint32_t hi = (w >> 1) & 0x78787878u;   // bytes: pos g1, pos g3, neg g1, neg g3
    acc  = fadd2(acc,  lds64(__byte_perm(lo, tb, 0x7650) + 0));
    acc  = fadd2(acc,  lds64(__byte_perm(hi, tb, 0x7650) + 128));
    acc  = fadd2(acc,  lds64(__byte_perm(lo, tb, 0x7651) + 256));
    acc  = fadd2(acc,  lds64(__byte_perm(hi, tb, 0x7651) + 384));
    accn = fadd2(accn, lds64(__byte_perm(lo, tb, 0x7652) + 0));
    accn = fadd2(accn, lds64(__byte_perm(hi, tb, 0x7652) + 128));
    accn = fadd2(accn, lds64(__byte_perm(lo, tb, 0x7653) + 256));
    accn = fadd2(accn, lds64(__byte_perm(hi, tb, 0x7653) + 384));
  } else {       // plain shift/mask (compiler's choice)
    #pragma unroll
    for (int j = 0; j < 4; ++j) acc = fadd2(acc, lds64(tb + j * 128 + ((w >> (4 * j)) & 15u) * 8));
    #pragma unroll
    for (int j = 0; j < 4; ++j) accn = fadd2(accn, lds64(tb + j * 128 + ((w >> (16 + 4 * j)) & 15u) * 8));
  }
}

// V 0/1: LUT loop, weights hashed in registers; V 2/3: same with weights from global (L2)
template<int V, int LDG>
__global__ void __launch_bounds__(1024) lut_kern(float* out, const uint4* wg){
  __shared__ __align__(1024) float2 tab[NG * 16];
  for (int i = threadIdx.x; i < NG * 16; i += blockDim.x) tab[i] = make_float2(1.0f + (i % 97) * 0.01f, 0.5f);
  __syncthreads();
  const uint32_t t0 = (uint32_t)__cvta_generic_to_shared(tab);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float2 a[4], an[4];
  #pragma unroll
  for (int q = 0; q < 4; ++q) { a[q] = make_float2(0, 0); an[q] = make_float2(0, 0); }
  uint4 w = make_uint4(lane * 0x9E3779B1u, lane * 0x85EBCA6Bu + 7u, lane * 0xC2B2AE35u + 3u, lane * 0x27D4EB2Fu + 1u);
  const uint4* wp = wg + ((size_t)(blockIdx.x * nw + warp) * 1024) * 32 + lane;  // per-warp 512 KB window
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t tb = t0 + (uint32_t)(((it + warp) & (NCH - 1)) * 512);
    if (LDG) w = ldg_stream(wp + (size_t)(it & 1023) * 32);
    else { w.x = w.x * 0x9E3779B1u + 1u; w.y ^= w.x; w.z += w.y; w.w ^= w.z >> 3; }
    plane<V>(a[0], an[0], w.x, tb);
    plane<V>(a[1], an[1], w.y, tb);
    plane<V>(a[2], an[2], w.z, tb);
    plane<V>(a[3], an[3], w.w, tb);
  }
  float t = 0;
  #pragma unroll
  for (int q = 0; q < 4; ++q) t += a[q].x + a[q].y - an[q].x - an[q].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// raw LDS.64 rates: MODE 0 = random entries of one 128-B table per warp (<= 1 word/bank),
// 1 = all lanes one address, 2 = lane l reads table l (32 tables, bank conflicts), 3 = LDS.32
// random within a 64-B table, 4 = LDS.128 random within one 256-B table
template<int MODE>
__global__ void __launch_bounds__(1024) lds_kern(float* out){
  __shared__ __align__(1024) float2 tab[NG * 16];
  for (int i = threadIdx.x; i < NG * 16; i += blockDim.x) tab[i] = make_float2(1.0f + (i % 97) * 0.01f, 0.5f);
  __syncthreads();
  const uint32_t t0 = (uint32_t)__cvta_generic_to_shared(tab);
  const int lane = threadIdx.x & 31;
  uint32_t ad[8];
  #pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint32_t h = (lane * 2654435761u) ^ (k * 0x9E3779B9u); h ^= h >> 13; h *= 0x85EBCA6Bu; h ^= h >> 16;
    if (MODE == 0) ad[k] = t0 + (h & 15u) * 8;
    else if (MODE == 1) ad[k] = t0;
    else if (MODE == 2) ad[k] = t0 + lane * 128 + (h & 15u) * 8;
    else if (MODE == 3) ad[k] = t0 + (h & 15u) * 4;
    else ad[k] = t0 + (h & 15u) * 16;
  }
  float2 a[8];
  #pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = make_float2(0, 0);
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t off = (uint32_t)((it & (NG - 1)) * 128);
    #pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 3) {
        float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(ad[k] + off));
        a[k].x += v;
      } else if (MODE == 4) {
        float4 v; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x),"=f"(v.y),"=f"(v.z),"=f"(v.w) : "r"(ad[k] + (off & ~255u)));
        a[k] = fadd2(a[k], make_float2(v.x + v.z, v.y + v.w));
      } else {
        a[k] = fadd2(a[k], lds64(ad[k] + (MODE == 2 ? (off & 0x1000u) : off)));
      }
    }
  }
  float t = 0;
  #pragma unroll
  for (int k = 0; k < 8; ++k) t += a[k].x + a[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
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
  float* out; CK(cudaMalloc(&out, sizeof(float) * nsm * 1024 * 2));
  uint4* wg; const size_t wbytes = (size_t)nsm * 32 * 1024 * 32 * 16;  // enough windows for 32 warps/SM
  CK(cudaMalloc(&wg, wbytes)); CK(cudaMemset(wg, 0x5A, wbytes));
  const double clk = 1.965e9;
  for (int wps : {4, 8, 16, 32}) {
    const int threads = wps * 32;
    double lk = (double)nsm * threads * ITERS * 32;  // lookups
    double s0 = time_it([&]{ lut_kern<0,0><<<nsm, threads>>>(out, wg); });
    double s1 = time_it([&]{ lut_kern<1,0><<<nsm, threads>>>(out, wg); });
    double s2 = time_it([&]{ lut_kern<0,1><<<nsm, threads>>>(out, wg); });
    double s3 = time_it([&]{ lut_kern<1,1><<<nsm, threads>>>(out, wg); });
    printf("warps/SM=%2d  LUT prmt/reg %5.1f  shf/reg %5.1f  prmt/ldg %5.1f  shf/ldg %5.1f  codes/clk/SM (2 codes per lookup)\n",
           wps, 2 * lk / s0 / nsm / clk, 2 * lk / s1 / nsm / clk, 2 * lk / s2 / nsm / clk, 2 * lk / s3 / nsm / clk);
    double lds = (double)nsm * threads * ITERS * 8;
    double r0 = time_it([&]{ lds_kern<0><<<nsm, threads>>>(out); });
    double r1 = time_it([&]{ lds_kern<1><<<nsm, threads>>>(out); });
    double r2 = time_it([&]{ lds_kern<2><<<nsm, threads>>>(out); });
    double r3 = time_it([&]{ lds_kern<3><<<nsm, threads>>>(out); });
    double r4 = time_it([&]{ lds_kern<4><<<nsm, threads>>>(out); });
    auto wr = [&](double s){ return lds / 32.0 / s / nsm / clk; };  // warp-LDS per clk per SM
    printf("warps/SM=%2d  warp-LDS/clk/SM: .64 one-table %.3f  .64 bcast %.3f  .64 32-tables %.3f  .32 one-table %.3f  .128 256B-table %.3f\n",
           wps, wr(r0), wr(r1), wr(r2), wr(r3), wr(r4));
  }
  return 0;
}
