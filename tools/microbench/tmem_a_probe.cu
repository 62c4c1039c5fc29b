// Probe: tcgen05.mma kind::i8 with the A operand in tensor memory (M = 128, N = 16, K = 32),
// A signed 8-bit, B unsigned 8-bit in shared memory (canonical K-major, no swizzle).
// Checks the assumed TMEM layout of A (lane = row, 32-bit column c holds K = 4c..4c+3,
// byte b = K 4c+b) against a host reference.  Tools only.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((256u >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__global__ void probe(const int8_t* A, const uint8_t* B, int32_t* D, uint32_t bsigned) {
    __shared__ __align__(1024) uint8_t sb[16 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // B canonical: k-step tile N x 32 bytes: (n>>3)*256 + h*128 + (n&7)*16 + c
    for (int e = tid; e < 16 * 32; e += blockDim.x) {
        int n = e / 32, k = e % 32;
        sb[(n >> 3) * 256 + ((k >> 4) & 1) * 128 + (n & 7) * 16 + (k & 15)] = B[n * 32 + k];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = slot;
    // A row 32w + lane -> TMEM lane 32w + lane, columns 0..7
    uint32_t v[8];
    const int row = 32 * warp + lane;
    for (int c = 0; c < 8; ++c) v[c] = *reinterpret_cast<const uint32_t*>(A + row * 32 + 4 * c);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tm + ((uint32_t)(32 * warp) << 16)),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        const uint32_t idesc = (2u << 4) | (1u << 7) | (bsigned << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t bd = desc((uint32_t)__cvta_generic_to_shared(sb));
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 32u),
                     "r"(tm), "l"(bd), "r"(idesc), "r"(0u) : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tm + 32u + ((uint32_t)(32 * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int c = 0; c < 16; ++c) D[row * 16 + c] = (int32_t)r[c];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm) : "memory");
}

int main() {
    int8_t hA[128 * 32];
    uint8_t hB[16 * 32];
    srand(1);
    for (int i = 0; i < 128 * 32; ++i) hA[i] = (int8_t)(rand() % 7 - 3);
    for (int i = 0; i < 16 * 32; ++i) hB[i] = (uint8_t)(rand() & 255);
    int8_t* dA; uint8_t* dB; int32_t* dD;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, 128 * 16 * 4);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    for (uint32_t bs = 0; bs < 2; ++bs) {
        cudaMemset(dD, 0, 128 * 16 * 4);
        probe<<<1, 128>>>(dA, dB, dD, bs);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        int32_t hD[128 * 16];
        cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
        long bad = 0;
        for (int i = 0; i < 128; ++i)
            for (int n = 0; n < 16; ++n) {
                long s = 0;
                for (int k = 0; k < 32; ++k) s += (long)hA[i * 32 + k] * (bs ? (long)(int8_t)hB[n * 32 + k] : (long)hB[n * 32 + k]);
                if (s != hD[i * 16 + n]) { if (bad < 5) printf("  mismatch row %d n %d: got %d want %ld\n", i, n, hD[i * 16 + n], s); ++bad; }
            }
        printf("B %s: %ld mismatches of 2048 (D[0][0..3] = %d %d %d %d)\n", bs ? "signed" : "unsigned", bad, hD[0], hD[1], hD[2], hD[3]);
    }
    return 0;
}
