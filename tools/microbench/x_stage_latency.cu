// x-staging latency on B200 (tools only): every CTA (one per SM) loads a 16 KB activation
// into shared memory (4 TMA-like bulk copies of 4 KB on one mbarrier, or plain 16-B loads by
// all threads) and records globaltimer from issue to arrival.  "shared": all CTAs load the
// SAME 16 KB (as every stage of the WL-GEMV does); "distinct": each CTA its own 16 KB.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o x_stage_latency x_stage_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <algorithm>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(512, 1) k_bulk(const char* x, int distinct, unsigned long long* out,
                                                 int nbytes, int pieces) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
    const char* src = x + (distinct ? (size_t)blockIdx.x * nbytes : 0);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0 = 0;
    if (threadIdx.x == 0) {
        t0 = gt();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nbytes));
        const int pb = nbytes / pieces;
        for (int i = 0; i < pieces; ++i)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    d + i * pb),
                "l"(src + i * pb), "r"(pb), "r"(b)
                : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(done)
                         : "r"(b));
        out[blockIdx.x] = gt() - t0;
    }
}

__global__ void __launch_bounds__(512, 1) k_ldg(const char* x, int distinct, unsigned long long* out,
                                                int nbytes) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const float4* src = reinterpret_cast<const float4*>(x + (distinct ? (size_t)blockIdx.x * nbytes : 0));
    __syncthreads();
    const unsigned long long t0 = gt();
    for (int i = threadIdx.x; i < nbytes / 16; i += blockDim.x)
        reinterpret_cast<float4*>(sm)[i] = __ldcg(src + i);
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = gt() - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nbytes = 16384;
    char* x;
    cudaMalloc(&x, (size_t)sms * nbytes);
    cudaMemset(x, 1, (size_t)sms * nbytes);
    char* flush;
    const size_t fb = 512u << 20;
    cudaMalloc(&flush, fb);
    unsigned long long* out;
    cudaMalloc(&out, sms * 8);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    std::vector<unsigned long long> h(sms);
    for (int cold = 0; cold < 2; ++cold)
        for (int distinct = 0; distinct < 2; ++distinct)
            for (int mode = 0; mode < 3; ++mode) {
                std::vector<double> med;
                for (int rep = 0; rep < 5; ++rep) {
                    if (cold) cudaMemset(flush, rep, fb);  // evict x from L2
                    if (mode == 0) k_bulk<<<sms, 512, 64 * 1024>>>(x, distinct, out, nbytes, 4);
                    else if (mode == 1) k_bulk<<<sms, 512, 64 * 1024>>>(x, distinct, out, nbytes, 1);
                    else k_ldg<<<sms, 512, 64 * 1024>>>(x, distinct, out, nbytes);
                    cudaDeviceSynchronize();
                    cudaMemcpy(h.data(), out, sms * 8, cudaMemcpyDeviceToHost);
                    std::sort(h.begin(), h.end());
                    med.push_back((double)h[sms / 2]);
                    if (rep == 4)
                        printf("%s x, %s, %-28s: median CTA %6.0f ns, max %6.0f ns\n", cold ? "L2-cold" : "L2-hot ",
                               distinct ? "distinct per CTA" : "shared by all  ",
                               mode == 0 ? "bulk copy, 4 x 4 KB" : (mode == 1 ? "bulk copy, 1 x 16 KB" : "LDG.128 by 512 threads"),
                               (double)h[sms / 2], (double)h[sms - 1]);
                }
            }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
