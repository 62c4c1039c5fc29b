// tcgen05.commit inside a tcgen05.mma stream, variants (tools only).  64 MMAs (kind::i8,
// A in TMEM, M = 128, N = 16, K = 32) per round, one final commit + wait per round.
//   V=0: no inner commit; V=1: commit every 8 to bar1 (nobody waits);
//   V=2: commit every 8 to bar1, a second warp waits on every phase of bar1;
//   V=3: commit every 8 to one of 4 barriers in turn;
//   V=4: commit every 8, MMAs alternate between two accumulators;
//   V=5: commit every 8, generic-address form;
//   V=6: commit every 8 with .multicast::cluster mask 1.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
    __shared__ __align__(1024) uint8_t sb[4096];
    __shared__ __align__(8) uint64_t bar[6];
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 1024; i += 128) reinterpret_cast<uint32_t*>(sb)[i] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < 6; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = slot;
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
    uint64_t bd = 0;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sb);
    bd |= (uint64_t)((sa >> 4) & 0x3FFFu) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | ((uint64_t)1 << 46);
    const uint32_t idesc = (2u << 4) | (1u << 7) | ((16u >> 3) << 17) | (8u << 24);
    if (tid == 0) {
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        uint32_t phase = 0;
        int nc = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 64; ++q) {
                const uint32_t acc = (it | q) ? 1u : 0u;
                const uint32_t d = (V == 4) ? tm + 16u * (q & 1) : tm;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                             "r"(tm + 256u + 8u * (q & 7)), "l"(bd), "r"(idesc), "r"((V == 4 && q < 2 && it == 0) ? 0u : acc)
                             : "memory");
                if (V != 0 && (q & 7) == 7 && q != 63) {
                    const uint32_t tb = b0 + 8u * (V == 3 ? 1 + (nc & 3) : 1);
                    ++nc;
                    if (V == 5)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)tb)
                                     : "memory");
                    else if (V == 6)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(tb),
                                     "h"((uint16_t)1) : "memory");
                    else
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tb)
                                     : "memory");
                }
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
    } else if (V == 2 && tid == 32) {
        uint32_t ph = 0;
        for (int n = 0; n < iters * 7; ++n) {
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                             : "=r"(done) : "r"(b0 + 8), "r"(ph) : "memory");
            ph ^= 1;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int V>
void run() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    k<V><<<148, 128>>>(2, d);
    cudaDeviceSynchronize();
    const int iters = 100;
    k<V><<<148, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %7.1f ns/MMA (%s)\n", V, (double)h / (iters * 64), e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<0>(); run<1>(); run<2>(); run<3>(); run<4>(); run<5>(); run<6>();
    return 0;
}
