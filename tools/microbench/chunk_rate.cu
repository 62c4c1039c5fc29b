// Inner-loop capacity of WL-GEMV chunk variants on smem-resident data (no HBM): codes per
// SM-clock as a function of warps per SM, to separate ALU limits from latency / TLP limits.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
constexpr int TC = 128;      // chunks of x in smem (m = 2048)
constexpr int WROWS = 8;     // rows of words in smem
constexpr int ITERS = 2048;

__device__ __forceinline__ float4 lds128(uint32_t a){ float4 v; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];":"=f"(v.x),"=f"(v.y),"=f"(v.z),"=f"(v.w):"r"(a)); return v; }
__device__ __forceinline__ uint4 lds128u(uint32_t a){ uint4 v; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];":"=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w):"r"(a)); return v; }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b){ return __fadd2_rn(a,b); }

// N = 1: pos/neg into the same accumulator; N = 2: separate; S = column-parity sets
template<int N, int S, int R>
struct V {
  float2 a[R][S][N][4];
  __device__ void zero(){
    #pragma unroll
    for(int r=0;r<R;r++)
    #pragma unroll
    for(int s=0;s<S;s++)
    #pragma unroll
    for(int k=0;k<N;k++)
    #pragma unroll
    for(int q=0;q<4;q++) a[r][s][k][q]=make_float2(0,0);
  }
  __device__ __forceinline__ static void col(float2 (&pos)[4], float2 (&neg)[4], uint32_t bits, float2 x){
    #pragma unroll
    for(int q=0;q<4;q++){
      if (bits & (2u<<(2*q))) pos[q]=fadd2(pos[q],x);
      if (N==2){ if (bits & (1u<<(2*q))) neg[q]=fadd2(neg[q],x); }
      else { if (bits & (1u<<(2*q))) pos[q]=fadd2(pos[q],make_float2(-x.x,-x.y)); }
    }
  }
  __device__ __forceinline__ void chunk(const uint4 (&w)[R], uint32_t xs, int tc){
    const uint32_t sw = tc & 7;
    #pragma unroll
    for(int kk=0;kk<8;kk++){
      const float4 v = lds128(xs + (uint32_t)(((tc*8) + (kk ^ sw))*16));
      #pragma unroll
      for(int r=0;r<R;r++){
        const uint32_t w4[4]={w[r].x,w[r].y,w[r].z,w[r].w};
        const uint32_t word=w4[kk>>1], sh=(kk&1)*16;
        col(a[r][0][0], a[r][0][N-1], (word>>sh)&0xffu, make_float2(v.x,v.y));
        col(a[r][S-1][0], a[r][S-1][N-1], (word>>(sh+8))&0xffu, make_float2(v.z,v.w));
      }
    }
  }
  __device__ float sum(){ float t=0;
    #pragma unroll
    for(int r=0;r<R;r++)
    #pragma unroll
    for(int s=0;s<S;s++)
    #pragma unroll
    for(int k=0;k<N;k++)
    #pragma unroll
    for(int q=0;q<4;q++) t+=a[r][s][k][q].x+a[r][s][k][q].y; return t; }
};

template<int N, int S, int R>
__global__ void kern(float* out){
  __shared__ __align__(128) unsigned char sm[TC*128 + WROWS*TC*16];
  const uint32_t xs = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t ws = xs + TC*128;
  for(int i=threadIdx.x;i<TC*32;i+=blockDim.x) reinterpret_cast<float*>(sm)[i]= 1.0f + (i%97)*0.01f;
  for(int i=threadIdx.x;i<WROWS*TC*4;i+=blockDim.x){
    unsigned h=(i*2654435761u)^0x9e3779b9u; h^=h>>15; h*=0x85ebca6bu; h^=h>>13;
    unsigned pos=h & 0xAAAAAAAAu; unsigned h2=h*0xc2b2ae35u; unsigned neg=(h2 & 0x55555555u) & ~(pos>>1);
    reinterpret_cast<unsigned*>(sm+TC*128)[i]=pos|neg;
  }
  __syncthreads();
  const int lane=threadIdx.x&31, warp=threadIdx.x>>5;
  V<N,S,R> acc; acc.zero();
  for(int it=0; it<ITERS; ++it){
    const int tc=(lane + 32*it) & (TC-1);
    uint4 w[R];
    #pragma unroll
    for(int r=0;r<R;r++) w[r]=lds128u(ws + (uint32_t)((((warp*R+r+it)&(WROWS-1))*TC + tc)*16));
    acc.chunk(w, xs, tc);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc.sum();
}

template<int N,int S,int R> int run(const char* name, int nsm){
  float* out; CK(cudaMalloc(&out, sizeof(float)*nsm*32*1024));
  for (int bps : {1,2,3,4,6,8,16}) {
    int blocks = nsm*bps, threads=128;
    kern<N,S,R><<<blocks,threads>>>(out); CK(cudaDeviceSynchronize());
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kern<N,S,R><<<blocks,threads>>>(out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double codes=(double)blocks*threads*ITERS*64*R;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s warps/SM=%3d  %.2f T codes/s  = %5.1f codes/clk/SM @1.965GHz\n", name, bps*4, codes/(ms*1e-3)*1e-12, codes/(ms*1e-3)/nsm/1.965e9);
  }
  cudaFree(out); return 0;
}
int main(){
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run<1,1,1>("N1 S1 R1", nsm);
  run<1,2,1>("N1 S2 R1 (old B=1)", nsm);
  run<2,2,1>("N2 S2 R1 (new B=1)", nsm);
  run<2,1,1>("N2 S1 R1", nsm);
  run<1,1,2>("N1 S1 R2", nsm);
  run<2,1,2>("N2 S1 R2", nsm);
  run<1,1,4>("N1 S1 R4", nsm);
  return 0;
}
