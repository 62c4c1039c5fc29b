// Inner-loop capacity of WL-GEMV chunk variants (lane = 16-column chunk, x from swizzled smem,
// weights from smem) when part of the accumulation moves to the FP64 pipe:
//   F0: all 4 planes predicated FADD2 (the product loop)
//   F1: planes 0-2 predicated FADD2, plane 3 predicated DADD (x converted with F2F.F64.F32)
//   F2: planes 0-1 FADD2, planes 2-3 DADD
// plus raw F2F.F64.F32 / DADD / FADD2 pipe rates.  codes/clk/SM at 1.965 GHz.
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

// predicated double add: acc += (bit ? x : 0) as one @P DADD
__device__ __forceinline__ void dadd_if(double& acc, double x, uint32_t bits, uint32_t mask){
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %2, %3;\n\tsetp.ne.b32 p, t, 0;\n\t@p add.rn.f64 %0, %0, %1;\n\t}"
               : "+d"(acc) : "d"(x), "r"(bits), "r"(mask));
}

template<int F>  // F = number of planes on the FP64 pipe (the last F planes)
struct V {
  static constexpr int S = 2;
  float2 a[S][4];
  double dr[S][2], di[S][2];
  __device__ void zero(){
    #pragma unroll
    for(int s=0;s<S;s++){
      #pragma unroll
      for(int q=0;q<4;q++) a[s][q]=make_float2(0,0);
      #pragma unroll
      for(int q=0;q<2;q++){ dr[s][q]=0; di[s][q]=0; }
    }
  }
  __device__ __forceinline__ void col(int s, uint32_t bits, float2 x){
    const float2 nx = make_float2(-x.x, -x.y);
    #pragma unroll
    for(int k=0;k<8;k++){
      const int q=k>>1;
      if (q < 4 - F) {
        if (bits & (1u<<k)) a[s][q]=fadd2(a[s][q], (k&1)? x : nx);
      }
    }
    if (F > 0) {
      const double xr = (double)x.x, xi = (double)x.y, nxr = -xr, nxi = -xi;
      #pragma unroll
      for(int k=0;k<8;k++){
        const int q=k>>1;
        if (q >= 4 - F) {
          const int d = q - (4 - F);
          dadd_if(dr[s][d], (k&1)? xr : nxr, bits, 1u<<k);
          dadd_if(di[s][d], (k&1)? xi : nxi, bits, 1u<<k);
        }
      }
    }
  }
  __device__ __forceinline__ void chunk(const uint4 w, uint32_t xs, int tc){
    const uint32_t sw = tc & 7;
    const uint32_t w4[4]={w.x,w.y,w.z,w.w};
    #pragma unroll
    for(int kk=0;kk<8;kk++){
      const float4 v = lds128(xs + (uint32_t)(((tc*8) + (kk ^ sw))*16));
      const uint32_t word=w4[kk>>1], sh=(kk&1)*16;
      col(0, (word>>sh)&0xffu, make_float2(v.x,v.y));
      col(1, (word>>(sh+8))&0xffu, make_float2(v.z,v.w));
    }
  }
  __device__ float sum(){ double t=0;
    #pragma unroll
    for(int s=0;s<S;s++){
      #pragma unroll
      for(int q=0;q<4;q++) t+=a[s][q].x+a[s][q].y;
      #pragma unroll
      for(int q=0;q<2;q++) t+=dr[s][q]+di[s][q];
    }
    return (float)t; }
};

template<int F>
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
  V<F> acc; acc.zero();
  for(int it=0; it<ITERS; ++it){
    const int tc=(lane + 32*it) & (TC-1);
    const uint4 w=lds128u(ws + (uint32_t)((((warp+it)&(WROWS-1))*TC + tc)*16));
    acc.chunk(w, xs, tc);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc.sum();
}

__global__ void f2f_kern(float* out){
  float x[8]; double d[8];
  #pragma unroll
  for(int i=0;i<8;i++){ x[i]=threadIdx.x*0.001f+i; d[i]=0; }
  for(int it=0; it<ITERS*8; ++it){
    #pragma unroll
    for(int i=0;i<8;i++){ double t; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(x[i])); d[i]+=0.0; asm volatile("mov.b64 %0, %0;" : "+d"(t)); x[i] = (float)__double2hiint(t) * 0.0f + x[i]; }
  }
  double t=0;
  #pragma unroll
  for(int i=0;i<8;i++) t+=x[i]+d[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=(float)t;
}

template<int F> int run(const char* name, int nsm){
  float* out; CK(cudaMalloc(&out, sizeof(float)*nsm*32*1024));
  for (int bps : {2,4,8}) {
    int blocks = nsm*bps, threads=128;
    kern<F><<<blocks,threads>>>(out); CK(cudaDeviceSynchronize());
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kern<F><<<blocks,threads>>>(out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double codes=(double)blocks*threads*ITERS*64;
    printf("%-34s warps/SM=%3d  %5.1f codes/clk/SM @1.965GHz\n", name, bps*4, codes/(ms*1e-3)/nsm/1.965e9);
  }
  cudaFree(out); return 0;
}
int main(){
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  run<0>("F0 4 FADD2 planes", nsm);
  run<1>("F1 3 FADD2 + 1 DADD plane (F2F)", nsm);
  run<2>("F2 2 FADD2 + 2 DADD planes (F2F)", nsm);
  return 0;
}
