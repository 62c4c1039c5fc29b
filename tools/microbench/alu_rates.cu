// Pipe-rate microbenchmark for sm_100a (B200): FADD, FADD2, predicated FADD2,
// LOP3, FADD2+LOP3 mixes, FFMA2.  Pure register work, no memory in the loop.
// Prints warp-instructions per SM-clock for each pattern, so the WL-GEMV
// inner-loop design (SURVEY §8d "issue ceiling") can be chosen from data.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ unsigned long long f2u(float a, float b){
  return ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
}

// each kernel: ITERS iterations x 16 ops per thread; record SM cycles per block
template<int KIND>
__global__ void kern(float* out, unsigned long long* cyc, unsigned seed){
  unsigned long long a[8];
  unsigned r[8];
  float s[16];
  unsigned long long X = f2u(1.0f + threadIdx.x*1e-7f, 2.0f);
  unsigned M1 = seed ^ threadIdx.x, M2 = seed * 3u + threadIdx.x;
  #pragma unroll
  for(int i=0;i<8;i++){ a[i]=f2u(i,i+1); r[i]=seed+i*7u+threadIdx.x; }
  #pragma unroll
  for(int i=0;i<16;i++) s[i]=i*0.5f;
  unsigned pbits = (threadIdx.x*2654435761u) ^ seed;
  __syncthreads();
  long long t0 = clock64();
  for(int it=0; it<ITERS; ++it){
    if (KIND==0){ // FADD2 x16
      #pragma unroll
      for(int k=0;k<2;k++)
      #pragma unroll
      for(int i=0;i<8;i++) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X));
    } else if (KIND==1){ // FADD x16
      #pragma unroll
      for(int i=0;i<16;i++) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(s[i]) : "f"(1.0f+it));
    } else if (KIND==2){ // LOP3 x16
      #pragma unroll
      for(int k=0;k<2;k++)
      #pragma unroll
      for(int i=0;i<8;i++) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(M1), "r"(M2));
    } else if (KIND==3){ // FADD2 x8 + LOP3 x8 interleaved
      #pragma unroll
      for(int i=0;i<8;i++){
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(M1), "r"(M2));
      }
    } else if (KIND==4){ // predicated FADD2 x16, predicates from bits of a word that changes per iteration
      pbits = __funnelshift_l(pbits, pbits, 3);
      #pragma unroll
      for(int k=0;k<2;k++)
      #pragma unroll
      for(int i=0;i<8;i++){
        unsigned long long t;
        if (pbits & (1u<<(i*2+k))) { asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X)); }
      }
    } else if (KIND==5){ // FFMA2 x16
      #pragma unroll
      for(int k=0;k<2;k++)
      #pragma unroll
      for(int i=0;i<8;i++) asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(a[i]) : "l"(X));
    } else if (KIND==6){ // FADD2 x16 with 2 LOP3 each (1:2 mix, LOP3-masked datapath shape)
      #pragma unroll
      for(int i=0;i<8;i++){
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(M1), "r"(M2));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[(i+1)&7]) : "r"(M1), "r"(M2));
      }
    } else if (KIND==7){ // FADD x8 + LOP3 x8 interleaved
      #pragma unroll
      for(int i=0;i<8;i++){
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(s[i]) : "f"(1.0f+it));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(M1), "r"(M2));
      }
    }
  }
  long long t1 = clock64();
  float acc=0; unsigned ra=0;
  #pragma unroll
  for(int i=0;i<8;i++){ acc += __uint_as_float((unsigned)a[i]) + __uint_as_float((unsigned)(a[i]>>32)); ra ^= r[i]; }
  #pragma unroll
  for(int i=0;i<16;i++) acc += s[i];
  out[blockIdx.x*blockDim.x+threadIdx.x] = acc + (float)ra;
  if(threadIdx.x==0) cyc[blockIdx.x] = (unsigned long long)(t1-t0);
}

template<int K> int run(const char* name, int ops_per_iter, int nsm, int threads){
  int blocks = nsm * (2048/threads);
  float* out; unsigned long long* cyc;
  CK(cudaMalloc(&out, sizeof(float)*blocks*threads));
  CK(cudaMalloc(&cyc, sizeof(unsigned long long)*blocks));
  kern<K><<<blocks,threads>>>(out,cyc,1u); CK(cudaDeviceSynchronize());
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<K><<<blocks,threads>>>(out,cyc,2u);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  unsigned long long* h = new unsigned long long[blocks];
  CK(cudaMemcpy(h,cyc,sizeof(unsigned long long)*blocks,cudaMemcpyDeviceToHost));
  double mean=0; for(int i=0;i<blocks;i++) mean+=h[i]; mean/=blocks;
  // warp-instructions per SM over the timed loop: (blocks/nsm)*(threads/32)*ITERS*ops
  double wi_per_sm = (double)(blocks/nsm)*(threads/32)*ITERS*ops_per_iter;
  double ipc = wi_per_sm / mean;  // blocks are co-resident (2048 threads/SM)
  double lane_ops_per_s = (double)blocks*threads*ITERS*ops_per_iter/(ms*1e-3);
  printf("%-34s  warp-instr/clk/SM = %.3f   (kernel %.3f ms, %.2f T lane-instr/s, eff clk %.0f MHz)\n",
         name, ipc, ms, lane_ops_per_s*1e-12, mean/(ms*1e3));
  cudaFree(out); cudaFree(cyc); delete[] h; return 0;
}

int main(){
  int nsm=0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs=%d\n", nsm);
  for(int th : {256, 1024}){
    printf("-- threads/block %d (2048 threads/SM)\n", th);
    run<0>("FADD2 (add.f32x2)", 16, nsm, th);
    run<1>("FADD", 16, nsm, th);
    run<2>("LOP3", 16, nsm, th);
    run<3>("FADD2+LOP3 1:1", 16, nsm, th);
    run<4>("pred FADD2 x16 (+pred setup, see SASS)", 16, nsm, th);
    run<5>("FFMA2", 16, nsm, th);
    run<6>("FADD2+2xLOP3 1:2", 24, nsm, th);
    run<7>("FADD+LOP3 1:1", 16, nsm, th);
  }
  return 0;
}
