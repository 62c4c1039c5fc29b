// Grid-barrier latency on B200 (tools only): a persistent cooperative kernel of one CTA per
// SM runs `iters` barriers (optionally after each CTA stores `stores` floats to global, as a
// stage epilogue would) and reports ns per barrier for several signal / poll variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o grid_barrier grid_barrier.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned* p) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void red_rlx(unsigned* p) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

template <int V>
__global__ void bar_kernel(unsigned* ctr, float* out, int iters, int stores, int sleep_ns) {
    const unsigned T = gridDim.x;
    for (int it = 0; it < iters; ++it) {
        for (int i = threadIdx.x; i < stores; i += blockDim.x)
            out[((size_t)it * gridDim.x + blockIdx.x) * stores + i] = (float)it;
        __syncthreads();
        if (threadIdx.x == 0) {
            if (V == 0) red_rel(ctr);
            else if (V == 1) { __threadfence(); red_rlx(ctr); }
            else { __threadfence(); atomicAdd(ctr, 1u); }
            const unsigned target = (unsigned)(it + 1) * T;
            if (V == 0 || V == 2) {
                while ((int)(ld_acq(ctr) - target) < 0) if (sleep_ns) __nanosleep(sleep_ns);
            } else {
                while ((int)(ld_rlx(ctr) - target) < 0) if (sleep_ns) __nanosleep(sleep_ns);
                __threadfence();
            }
        }
        __syncthreads();
    }
}

__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// V = 3: per-CTA flags (own 128-B line, epoch value, no atomics), warp 0 reads all flags.
// V = 4: K = 8 counters on separate lines (CTA b adds to counter b % 8), warp 0 sums them.
template <int V>
__global__ void bar2_kernel(unsigned* ctr, float* out, int iters, int stores, int sleep_ns) {
    const unsigned T = gridDim.x;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
        for (int i = threadIdx.x; i < stores; i += blockDim.x)
            out[((size_t)it * gridDim.x + blockIdx.x) * stores + i] = (float)it;
        __syncthreads();
        if (threadIdx.x < 32) {
            if (V == 3) {
                if (lane == 0) st_rel(ctr + 32 * blockIdx.x, (unsigned)it + 1);
                while (true) {
                    bool ok = true;
                    for (unsigned b = lane; b < T; b += 32) ok &= (int)(ld_acq(ctr + 32 * b) - (unsigned)(it + 1)) >= 0;
                    if (__all_sync(0xffffffffu, ok)) break;
                    if (sleep_ns) __nanosleep(sleep_ns);
                }
            } else {
                if (lane == 0) red_rel(ctr + 32 * (blockIdx.x % 8));
                while (true) {
                    unsigned v = lane < 8 ? ld_acq(ctr + 32 * lane) : 0u;
                    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if ((int)(v - (unsigned)(it + 1) * T) >= 0) break;
                    if (sleep_ns) __nanosleep(sleep_ns);
                }
            }
        }
        __syncthreads();
    }
}

template <int V>
float run2(int grid, int iters, int stores, int sleep_ns, unsigned* ctr, float* out) {
    cudaMemset(ctr, 0, 4 * 32 * 160);
    void* args[] = {&ctr, &out, &iters, &stores, &sleep_ns};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)bar2_kernel<V>, grid, 512, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e6f / iters;
}

template <int V>
float run(int grid, int iters, int stores, int sleep_ns, unsigned* ctr, float* out) {
    cudaMemset(ctr, 0, 4);
    void* args[] = {&ctr, &out, &iters, &stores, &sleep_ns};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)bar_kernel<V>, grid, 512, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e6f / iters;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* ctr;
    float* out;
    const int iters = 2000;
    cudaMalloc(&ctr, 4 * 32 * 160);
    cudaMalloc(&out, (size_t)iters * sms * 64 * 4);
    const char* names[] = {"red.release + ld.acquire poll", "fence + red.relaxed + relaxed poll + fence",
                           "fence + atomicAdd + ld.acquire poll"};
    for (int stores : {0, 16, 64})
        for (int sl : {0, 32, 256}) {
            run<0>(sms, 50, stores, sl, ctr, out);  // warm
            printf("stores/CTA %2d sleep %3d ns: %6.0f | %6.0f | %6.0f ns per barrier\n", stores, sl,
                   run<0>(sms, iters, stores, sl, ctr, out), run<1>(sms, iters, stores, sl, ctr, out),
                   run<2>(sms, iters, stores, sl, ctr, out));
        }
    printf("columns: %s | %s | %s\n", names[0], names[1], names[2]);
    for (int stores : {0, 64})
        for (int sl : {0, 32}) {
            run2<3>(sms, 50, stores, sl, ctr, out);
            printf("stores/CTA %2d sleep %3d ns: per-CTA flags, warp reads all %6.0f | 8 counters %6.0f ns\n",
                   stores, sl, run2<3>(sms, iters, stores, sl, ctr, out), run2<4>(sms, iters, stores, sl, ctr, out));
        }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
