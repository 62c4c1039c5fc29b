// tcgen05.mma throughput for the small-N shapes of the tensor-core WL-GEMV: back-to-back
// MMAs into one accumulator (M = 128), A from tensor memory (.ts) or shared memory (.ss),
// kind::i8 / kind::f8f6f4 (e4m3) / kind::f16, N = 16..256.  One CTA per SM, all SMs.
// Tools only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((256u >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
    return pred != 0;
}
template <int KIND, bool TS, bool CONV = false>  // KIND 0 = i8, 1 = f8f6f4 e4m3, 2 = f16
__global__ void __launch_bounds__(128, 1) rate(int N, int iters, int per_commit, unsigned long long* out,
                                               int inner_commit = 0) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 64 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = slot;
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar[0]);
    unsigned long long t0 = 0, t1 = 0;
    if (CONV ? warp == 0 : tid == 0) {
        uint32_t idesc;
        if (KIND == 0) idesc = (2u << 4) | (1u << 7) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        else if (KIND == 1) idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        else idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm);
        const uint64_t ad = desc(sa), bd = desc(sa + 32768);
        uint32_t phase = 0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < per_commit; ++k) {
                const uint32_t acc = (it | k) ? 1u : 0u;
                if (CONV && !elect_one()) { __syncwarp(); continue; }
                if (inner_commit && k && (k % inner_commit) == 0)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a + 8)
                                 : "memory");
                if (TS) {
                    if (KIND == 0)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                                     "r"(tm + 256u + 8u * (k & 7)), "l"(bd), "r"(idesc), "r"(acc) : "memory");
                    else if (KIND == 1)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                                     "r"(tm + 256u + 8u * (k & 7)), "l"(bd), "r"(idesc), "r"(acc) : "memory");
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                                     "r"(tm + 256u + 8u * (k & 7)), "l"(bd), "r"(idesc), "r"(acc) : "memory");
                } else {
                    if (KIND == 0)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                                     "l"(ad + 256 * (k & 7)), "l"(bd), "r"(idesc), "r"(acc) : "memory");
                    else if (KIND == 1)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                                     "l"(ad + 256 * (k & 7)), "l"(bd), "r"(idesc), "r"(acc) : "memory");
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                                     "l"(ad + 256 * (k & 7)), "l"(bd), "r"(idesc), "r"(acc) : "memory");
                }
                if (CONV) __syncwarp();
            }
            if (!CONV || elect_one())
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a)
                             : "memory");
            __syncwarp();
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                             : "=r"(done) : "r"(bar_a), "r"(phase) : "memory");
            phase ^= 1;
        }
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (blockIdx.x == 0 && (tid & 31) == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int KIND, bool TS, bool CONV = false>
void run(const char* name, int N, int iters, int per, int inner = 0) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate<KIND, TS, CONV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    rate<KIND, TS, CONV><<<148, 128, 64 * 1024>>>(N, 2, per, d);
    cudaDeviceSynchronize();
    rate<KIND, TS, CONV><<<148, 128, 64 * 1024>>>(N, iters, per, d, inner);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double per_mma = (double)h / (iters * per);
    const int K = KIND == 2 ? 16 : 32;
 printf("%-18s inner=%2d N=%3d per_commit=%3d: %8.1f ns/MMA  %7.1f clk  (%s) -> %.1f TOPS (all SMs)\n", name, inner, N, per,
           per_mma, per_mma * 1.965, e == cudaSuccess ? "ok" : cudaGetErrorString(e),
           2.0 * 128 * N * K * 148 / per_mma * 1e-3);
    cudaFree(d);
}

int main() {
    for (int inner : {0, 1, 2, 4, 16}) run<0, true, true>("i8 tmem CONV", 16, 100, 64, inner);
    for (int inner : {1, 2, 4, 8, 16}) run<0, true>("i8 A=tmem", 16, 100, 64, inner);
    run<0, true>("i8 A=tmem", 16, 100, 128);
    run<0, true>("i8 A=tmem", 32, 100, 128);
    run<0, true>("i8 A=tmem", 64, 100, 128);
    for (int N : {16, 64, 256}) {
        run<0, true>("i8 A=tmem", N, 200, 16);
        run<0, false>("i8 A=smem", N, 200, 16);
        run<1, true>("e4m3 A=tmem", N, 200, 16);
        run<1, false>("e4m3 A=smem", N, 200, 16);
        run<2, false>("f16 A=smem", N, 200, 16);
    }
    run<0, true>("i8 A=tmem", 16, 200, 2);
    run<0, true>("i8 A=tmem", 16, 200, 64);
    return 0;
}
