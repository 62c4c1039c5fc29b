// Does a packed 4-bit A operand halve the tensor core's A-read time per code?  Back-to-back
// unrolled MMAs (commit every 8, wait per 64), M = 128, A and B from shared memory (K-major,
// no swizzle), one issuing thread per SM on all SMs: kind::i8 (K = 32 = 32 bytes of A per
// row) vs kind::mxf4.block_scale.block32 (K = 64 packed e2m1 = 32 bytes of A per row; scale
// factors from TMEM, values irrelevant for timing).  Tools only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND, int N>  // KIND 0 = i8, 1 = mxf4
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
    __shared__ __align__(1024) uint8_t sa[8192];
    __shared__ __align__(1024) uint8_t sbm[8192];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 2048; i += 128) {
        reinterpret_cast<uint32_t*>(sa)[i] = 0x22222222u;
        reinterpret_cast<uint32_t*>(sbm)[i] = 0x22222222u;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < 2; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = slot;
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
    auto desc = [](uint32_t a) {
        return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | ((uint64_t)1 << 46);
    };
    const uint64_t ad = desc((uint32_t)__cvta_generic_to_shared(sa)), bd = desc((uint32_t)__cvta_generic_to_shared(sbm));
    const uint32_t idesc_i8 = (2u << 4) | (1u << 7) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint32_t idesc_f4 = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | (8u << 24);
    if (tid == 0) {
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        uint32_t phase = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 64; ++q) {
                const uint32_t acc = (it | q) ? 1u : 0u;
                const uint64_t a = ad + (uint64_t)(256 * (q & 3));  // 4 K-steps of A (4 KB each)
                if (KIND == 0)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                                 "l"(a), "l"(bd), "r"(idesc_i8), "r"(acc) : "memory");
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tm),
                                 "l"(a), "l"(bd), "r"(idesc_f4), "r"(acc), "r"(tm + 256u), "r"(tm + 320u) : "memory");
                if ((q & 7) == 7 && q != 63)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0 + 8)
                                 : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0)
                         : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                             : "=r"(done) : "r"(b0), "r"(phase) : "memory");
            phase ^= 1;
        }
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int KIND, int N>
void run() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    k<KIND, N><<<148, 128>>>(2, d);
    cudaDeviceSynchronize();
    const int iters = 200;
    k<KIND, N><<<148, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double ns = (double)h / (iters * 64);
    const double codes = 128.0 * (KIND ? 64 : 32);  // A elements per MMA
    printf("%s N=%3d: %6.1f ns/MMA, %6.1f clk, %6.1f A-elements/clk/SM (%s)\n", KIND ? "mxf4 " : "i8   ", N, ns,
           ns * 1.965, codes / (ns * 1.965), e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<0, 16>(); run<1, 16>(); run<0, 32>(); run<1, 32>(); run<0, 64>(); run<1, 64>();
    run<1, 128>(); run<1, 256>();
    return 0;
}
