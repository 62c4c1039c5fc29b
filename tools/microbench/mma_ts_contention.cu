// tcgen05.mma kind::i8 (A in TMEM, M = 128, N = 16, K = 32) issue rate under the conditions of
// wl_tcv_kernel (tools only): V=0 fixed B address; V=1 B address advancing 512 B per MMA over
// 32 KB; V=2 as 1 plus 16 warps storing 16 TMEM columns each (tcgen05.st.32x32b.x16, other
// columns) continuously; V=3 as 1 plus 16 warps doing LDS.128 + PRMT work (no TMEM traffic).
// 64 MMAs per round, commit every 8 (unrolled), wait at the end of each round.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__global__ void __launch_bounds__(544, 1) k(int iters, unsigned long long* out, unsigned* sink) {
    extern __shared__ __align__(1024) uint8_t sb[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = i * 2654435761u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        stop = 0;
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
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sb);
    const uint32_t idesc = (2u << 4) | (1u << 7) | ((16u >> 3) << 17) | (8u << 24);
    if (tid == 0) {
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        uint32_t phase = 0;
        for (int it = 0; it < iters; ++it) {
            const uint32_t boff = (uint32_t)(it & 1) * 32768u;
#pragma unroll
            for (int q = 0; q < 64; ++q) {
                const uint32_t acc = (it | q) ? 1u : 0u;
                const uint32_t baddr = V == 0 ? sa : sa + ((boff + 512u * q) & 32767u);
                const uint64_t bd = (uint64_t)((baddr >> 4) & 0x3FFFu) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) |
                                    ((uint64_t)1 << 46);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                             "r"(tm + 32u + 8u * (q & 7)), "l"(bd), "r"(idesc), "r"(acc) : "memory");
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
        stop = 1;
    } else if (warp >= 1 && (V == 2 || V == 3)) {
        // background load: warps 1..16 (TMEM lane quarter warp % 4), columns 96 + 16 (warp / 4)
        const int q = warp & 3, c = (warp - 1) >> 2;
        uint32_t acc = 0;
        while (!stop) {
#pragma unroll 1
            for (int r = 0; r < 16; ++r) {
                uint4 w;
                asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                             : "r"(sa + 49152u + (uint32_t)((tid * 16 + r * 4096) & 16383)));
                uint32_t o[16];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t x = j == 0 ? w.x : j == 1 ? w.y : j == 2 ? w.z : w.w;
                    const uint32_t e = x & 0x33333333u, d = (x >> 2) & 0x33333333u;
                    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(o[4 * j]) : "r"(0x0001FF00u), "r"(e));
                    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(o[4 * j + 1]) : "r"(0x0001FF00u), "r"(e >> 16));
                    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(o[4 * j + 2]) : "r"(0x0001FF00u), "r"(d));
                    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(o[4 * j + 3]) : "r"(0x0001FF00u), "r"(d >> 16));
                }
                if (V == 2) {
                    asm volatile(
                        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                        "%14,%15,%16};" ::"r"(tm + ((uint32_t)(32 * q) << 16) + 96u + 16u * c),
                        "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]),
                        "r"(o[9]), "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15])
                        : "memory");
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc += o[j];
                }
            }
        }
        if (acc == 0x12345) sink[0] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int V>
void run() {
    unsigned long long* d;
    unsigned* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<V><<<148, 544, 64 * 1024>>>(2, d, sink);
    cudaDeviceSynchronize();
    const int iters = 200;
    k<V><<<148, 544, 64 * 1024>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %7.1f ns/MMA (%s)\n", V, (double)h / (iters * 64), e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

int main() {
    run<0>(); run<1>(); run<2>(); run<3>();
    return 0;
}
