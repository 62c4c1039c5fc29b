// Pipe-rate microbenchmark for sm_100a (B200): FADD, FADD2, predicated FADD2,
// LOP3, FADD2+LOP3 mixes, FFMA2.  Pure register work, no memory in the loop.
// Prints warp-instructions per SM-clock for each pattern, so the WL-GEMV
// inner-loop design (SURVEY §8d "issue ceiling") can be chosen from data.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 65536
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
  unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for(int it=0; it<ITERS; ++it){
    if (KIND==0){ // FADD2 x16
      #pragma unroll
      for(int k=0;k<2;k++)
      #pragma unroll
      for(int i=0;i<8;i++) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(X));
    } else if (KIND==1){ // FADD x16
      #pragma unroll
      for(int i=0;i<16;i++) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(s[i]) : "f"(__uint_as_float((unsigned)X)));
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
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(s[i]) : "f"(__uint_as_float((unsigned)X)));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(M1), "r"(M2));
      }
    }
  }
  long long t1 = clock64();
  unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  float acc=0; unsigned ra=0;
  #pragma unroll
  for(int i=0;i<8;i++){ acc += __uint_as_float((unsigned)a[i]) + __uint_as_float((unsigned)(a[i]>>32)); ra ^= r[i]; }
  #pragma unroll
  for(int i=0;i<16;i++) acc += s[i];
  out[blockIdx.x*blockDim.x+threadIdx.x] = acc + (float)ra;
  if(threadIdx.x==0){ cyc[2*blockIdx.x] = (unsigned long long)(t1-t0); cyc[2*blockIdx.x+1] = g1-g0; }
}

template<int K> int run(const char* name, int ops_per_iter, int nsm, int threads){
  int blocks = nsm * (2048/threads);
  float* out; unsigned long long* cyc;
  CK(cudaMalloc(&out, sizeof(float)*blocks*threads));
  CK(cudaMalloc(&cyc, 2*sizeof(unsigned long long)*blocks));
  kern<K><<<blocks,threads>>>(out,cyc,1u); CK(cudaDeviceSynchronize());
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<K><<<blocks,threads>>>(out,cyc,2u);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  unsigned long long* h = new unsigned long long[2*blocks];
  CK(cudaMemcpy(h,cyc,2*sizeof(unsigned long long)*blocks,cudaMemcpyDeviceToHost));
  double mean=0, ns=0; for(int i=0;i<blocks;i++){ mean+=h[2*i]; ns+=h[2*i+1]; } mean/=blocks; ns/=blocks;
  double mhz = mean/ns*1e3;
  // warp-instructions per SM over the timed loop: (blocks/nsm)*(threads/32)*ITERS*ops
  double wi_per_sm = (double)(blocks/nsm)*(threads/32)*ITERS*ops_per_iter;
  double lane_ops = (double)blocks*threads*ITERS*ops_per_iter;
  double ipc = lane_ops/32.0/nsm/(ms*1e-3)/(mhz*1e6);  // warp-instr per SM-clock at the measured clock
  double lane_ops_per_s = (double)blocks*threads*ITERS*ops_per_iter/(ms*1e-3);
  printf("%-34s  warp-instr/clk/SM = %.3f   (kernel %.3f ms, %.2f T lane-instr/s, SM clk %.0f MHz)\n",
         name, ipc, ms, lane_ops_per_s*1e-12, mhz);
  cudaFree(out); cudaFree(cyc); delete[] h; return 0;
}


// ---- realistic ternary inner loops: one uint4 (4 planes x 16 codes) per iteration from smem,
// 16 x-pairs in registers; counts codes/clk/SM.
#define TITERS 8192
template<int V>
__global__ void tern(float* out, unsigned long long* cyc, unsigned seed){
  __shared__ uint4 wsm[256];
  for(int i=threadIdx.x;i<256;i+=blockDim.x){
    unsigned h=(i*2654435761u)^seed; uint4 q;
    // random codes with no (1,1): pos bits from h, neg bits = ~pos & h2
    unsigned a=h*0x9E3779B9u, b=h*0x85EBCA6Bu, c=h*0xC2B2AE35u, d=h*0x27D4EB2Fu;
    q.x=(a&0xAAAAAAAAu)|((~(a>>1))&b&0x55555555u); q.y=(b&0xAAAAAAAAu)|((~(b>>1))&c&0x55555555u);
    q.z=(c&0xAAAAAAAAu)|((~(c>>1))&d&0x55555555u); q.w=(d&0xAAAAAAAAu)|((~(d>>1))&a&0x55555555u);
    wsm[i]=q;
  }
  __syncthreads();
  float2 X[16];
  #pragma unroll
  for(int k=0;k<16;k++) X[k]=make_float2(1.0f+k*0.001f+threadIdx.x*1e-6f, 2.0f-k*0.001f);
  float2 acc[4]; 
  #pragma unroll
  for(int p=0;p<4;p++) acc[p]=make_float2(0.f,0.f);
  long long t0 = clock64();
  unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for(int it=0; it<TITERS; ++it){
    uint4 q = wsm[(it*7+threadIdx.x)&255];
    unsigned w[4]={q.x,q.y,q.z,q.w};
    if (V==0){ // predicated add / sub
      #pragma unroll
      for(int k=0;k<16;k++){
        #pragma unroll
        for(int p=0;p<4;p++){
          if (w[p] & (2u<<(2*k))) acc[p]=__fadd2_rn(acc[p], X[k]);
          if (w[p] & (1u<<(2*k))) acc[p]=__fadd2_rn(acc[p], make_float2(-X[k].x,-X[k].y));
        }
      }
    } else if (V==1){ // LOP3-masked: v = (x ^ S) & M, one FADD2 per code
      #pragma unroll
      for(int p=0;p<4;p++){
        unsigned nz = (w[p] | (w[p]>>1)) & 0x55555555u;  // bit 2k = nonzero
        #pragma unroll
        for(int k=0;k<16;k++){
          unsigned S = (w[p] << (31-2*k)) & 0x80000000u;           // neg bit -> sign
          unsigned M = 0u - ((nz >> (2*k)) & 1u);                 // all ones if nonzero
          float2 v = make_float2(__uint_as_float((__float_as_uint(X[k].x)^S)&M),
                                 __uint_as_float((__float_as_uint(X[k].y)^S)&M));
          acc[p]=__fadd2_rn(acc[p], v);
        }
      }
    } else if (V==2){ // predicated on nonzero, sign by LOP3 xor
      #pragma unroll
      for(int p=0;p<4;p++){
        unsigned nz = (w[p] | (w[p]>>1)) & 0x55555555u;
        #pragma unroll
        for(int k=0;k<16;k++){
          unsigned S = (w[p] << (31-2*k)) & 0x80000000u;
          float2 v = make_float2(__uint_as_float(__float_as_uint(X[k].x)^S),
                                 __uint_as_float(__float_as_uint(X[k].y)^S));
          if (nz & (1u<<(2*k))) acc[p]=__fadd2_rn(acc[p], v);
        }
      }

    } else if (V==4 || V==5 || V==6){ // PTX predicated add.f32x2 on u64 accumulators
      unsigned long long A[4];
      #pragma unroll
      for(int p=0;p<4;p++) A[p]=((unsigned long long)__float_as_uint(acc[p].y)<<32)|__float_as_uint(acc[p].x);
      if (V==5) { w[0]=w[1]=w[2]=w[3]=it&0x100000u; }            // all predicates false (except rare)
      if (V==6) { w[0]|=0xFFFFFFFFu; w[1]|=0xFFFFFFFFu; w[2]|=0xFFFFFFFFu; w[3]|=0xFFFFFFFFu; }
      #pragma unroll
      for(int k=0;k<16;k++){
        unsigned long long XX=((unsigned long long)__float_as_uint(X[k].y)<<32)|__float_as_uint(X[k].x);
        unsigned long long NX=XX^0x8000000080000000ull;
        #pragma unroll
        for(int p=0;p<4;p++){
          asm volatile("{.reg .pred pp, pn; .reg .b32 t0, t1;\n\t"
                       "and.b32 t0, %2, %3; and.b32 t1, %2, %4;\n\t"
                       "setp.ne.b32 pp, t0, 0; setp.ne.b32 pn, t1, 0;\n\t"
                       "@pp add.rn.f32x2 %0, %0, %1;\n\t"
                       "@pn add.rn.f32x2 %0, %0, %5;}"
                       : "+l"(A[p]) : "l"(XX), "r"(w[p]), "r"(2u<<(2*k)), "r"(1u<<(2*k)), "l"(NX));
        }
      }
      #pragma unroll
      for(int p=0;p<4;p++) acc[p]=make_float2(__uint_as_float((unsigned)A[p]), __uint_as_float((unsigned)(A[p]>>32)));
    } else if (V==3){ // mixed: planes 0,1 predicated; planes 2,3 masked
      #pragma unroll
      for(int k=0;k<16;k++){
        #pragma unroll
        for(int p=0;p<2;p++){
          if (w[p] & (2u<<(2*k))) acc[p]=__fadd2_rn(acc[p], X[k]);
          if (w[p] & (1u<<(2*k))) acc[p]=__fadd2_rn(acc[p], make_float2(-X[k].x,-X[k].y));
        }
      }
      #pragma unroll
      for(int p=2;p<4;p++){
        unsigned nz = (w[p] | (w[p]>>1)) & 0x55555555u;
        #pragma unroll
        for(int k=0;k<16;k++){
          unsigned S = (w[p] << (31-2*k)) & 0x80000000u;
          unsigned M = 0u - ((nz >> (2*k)) & 1u);
          float2 v = make_float2(__uint_as_float((__float_as_uint(X[k].x)^S)&M),
                                 __uint_as_float((__float_as_uint(X[k].y)^S)&M));
          acc[p]=__fadd2_rn(acc[p], v);
        }
      }
    }
  }
  long long t1 = clock64();
  unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  float s=0;
  #pragma unroll
  for(int p=0;p<4;p++) s+=acc[p].x+acc[p].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if(threadIdx.x==0){ cyc[2*blockIdx.x]=(unsigned long long)(t1-t0); cyc[2*blockIdx.x+1]=g1-g0; }
}

template<int V> int run_tern(const char* name, int nsm, int threads, int blocks_per_sm){
  int blocks = nsm*blocks_per_sm;
  float* out; unsigned long long* cyc;
  CK(cudaMalloc(&out, sizeof(float)*blocks*threads));
  CK(cudaMalloc(&cyc, 2*sizeof(unsigned long long)*blocks));
  tern<V><<<blocks,threads>>>(out,cyc,1u); CK(cudaDeviceSynchronize());
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tern<V><<<blocks,threads>>>(out,cyc,2u);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  unsigned long long* h = new unsigned long long[2*blocks];
  CK(cudaMemcpy(h,cyc,2*sizeof(unsigned long long)*blocks,cudaMemcpyDeviceToHost));
  double cy=0, ns=0; for(int i=0;i<blocks;i++){ cy+=h[2*i]; ns+=h[2*i+1]; } cy/=blocks; ns/=blocks;
  double mhz = cy/ns*1e3;
  double codes = (double)blocks*threads*TITERS*64;
  double cps = codes/(ms*1e-3);
  printf("tern %-28s warps/SM=%2d  codes/clk/SM = %6.2f  (%.2f T codes/s = %.2f TB/s-equiv, %.3f ms, SM clk %.0f MHz)\n",
         name, blocks_per_sm*threads/32, cps/nsm/(mhz*1e6), cps*1e-12, cps/4*1e-12, ms, mhz);
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
  for(int bps : {2, 4, 8}){
    run_tern<0>("predicated add/sub", nsm, 256, bps);
    run_tern<1>("LOP3 masked", nsm, 256, bps);
    run_tern<2>("pred nz + LOP3 sign", nsm, 256, bps);
    run_tern<3>("mixed 2 pred + 2 masked", nsm, 256, bps);
    run_tern<4>("PTX pred add.f32x2 (u64 acc)", nsm, 256, bps);
    run_tern<5>("PTX pred, all preds false", nsm, 256, bps);
    run_tern<6>("PTX pred, all preds true", nsm, 256, bps);
  }
  return 0;
}
