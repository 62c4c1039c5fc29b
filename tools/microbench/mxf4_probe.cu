// Probe (tools only): tcv-style exact ternary x digit products on kind::mxf4 (packed e2m1):
// A = 128 x 64 ternary {-1, 0, +1}, B = 16 x 64 digits {0, 1, 2, 3}, both K-major canonical
// (8-row x 16-byte core matrices, the two 16-byte K halves LBO = 128 B apart, 8-row groups
// SBO = 256 B apart), element k of a row in byte k / 2, nibble k % 2 (low first = variant 0,
// high first = variant 1); all scale factors E8M0 1.0 (0x7F in every byte of the TMEM
// columns given as SFA / SFB).  D (fp32) must equal the integer dot products exactly.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | ((uint64_t)1 << 46);
}

__global__ void probe(const uint8_t* A, const uint8_t* B, float* D, int variant) {
    __shared__ __align__(1024) uint8_t sa[128 * 32];
    __shared__ __align__(1024) uint8_t sb[16 * 32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < 128 * 32; e += blockDim.x) {
        const int r = e / 32, b = e % 32;
        sa[(r >> 3) * 256 + (b >> 4) * 128 + (r & 7) * 16 + (b & 15)] = A[e];
    }
    for (int e = tid; e < 16 * 32; e += blockDim.x) {
        const int r = e / 32, b = e % 32;
        sb[(r >> 3) * 256 + (b >> 4) * 128 + (r & 7) * 16 + (b & 15)] = B[e];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
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
    // scale factors: columns 64..191 of every lane = 0x7F7F7F7F (E8M0 1.0)
    {
        uint32_t v[16];
        for (int i = 0; i < 16; ++i) v[i] = 0x7F7F7F7Fu;
        for (int c = 64; c < 192; c += 16)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                    tm + ((uint32_t)(32 * warp) << 16) + (uint32_t)c),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | (1u << 23) | (8u << 24);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tm),
                     "l"(desc((uint32_t)__cvta_generic_to_shared(sa))), "l"(desc((uint32_t)__cvta_generic_to_shared(sb))),
                     "r"(idesc), "r"(0u), "r"(tm + 64u), "r"(tm + 128u) : "memory");
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
                 : "r"(tm + ((uint32_t)(32 * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int c = 0; c < 16; ++c) D[(32 * warp + lane) * 16 + c] = __uint_as_float(r[c]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm) : "memory");
    (void)variant;
}

static uint8_t e2m1(int v) {  // v in {-1, 0, 1, 2, 3}
    switch (v) {
        case -1: return 0xA;
        case 0: return 0x0;
        case 1: return 0x2;
        case 2: return 0x4;
        default: return 0x5;
    }
}

int main() {
    int a[128][64], b[16][64];
    srand(7);
    for (int i = 0; i < 128; ++i)
        for (int k = 0; k < 64; ++k) a[i][k] = rand() % 3 - 1;
    for (int n = 0; n < 16; ++n)
        for (int k = 0; k < 64; ++k) b[n][k] = rand() % 4;
    uint8_t *dA, *dB;
    float* dD;
    cudaMalloc(&dA, 128 * 32);
    cudaMalloc(&dB, 16 * 32);
    cudaMalloc(&dD, 128 * 16 * 4);
    for (int variant = 0; variant < 2; ++variant) {
        uint8_t hA[128 * 32], hB[16 * 32];
        for (int i = 0; i < 128; ++i)
            for (int k = 0; k < 64; k += 2) {
                const uint8_t lo = e2m1(a[i][k]), hi = e2m1(a[i][k + 1]);
                hA[i * 32 + k / 2] = variant == 0 ? (uint8_t)(lo | hi << 4) : (uint8_t)(hi | lo << 4);
            }
        for (int n = 0; n < 16; ++n)
            for (int k = 0; k < 64; k += 2) {
                const uint8_t lo = e2m1(b[n][k]), hi = e2m1(b[n][k + 1]);
                hB[n * 32 + k / 2] = variant == 0 ? (uint8_t)(lo | hi << 4) : (uint8_t)(hi | lo << 4);
            }
        cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        cudaMemset(dD, 0, 128 * 16 * 4);
        probe<<<1, 128>>>(dA, dB, dD, variant);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("variant %d: %s\n", variant, cudaGetErrorString(e)); return 1; }
        float hD[128 * 16];
        cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 128; ++i)
            for (int n = 0; n < 16; ++n) {
                int s = 0;
                for (int k = 0; k < 64; ++k) s += a[i][k] * b[n][k];
                if ((float)s != hD[i * 16 + n]) {
                    if (bad < 4) printf("  v%d row %d col %d: got %g want %d\n", variant, i, n, hD[i * 16 + n], s);
                    ++bad;
                }
            }
        printf("variant %d (%s nibble first): %d mismatches of 2048; D[0][0..3] = %g %g %g %g\n", variant,
               variant ? "high" : "low", bad, hD[0], hD[1], hD[2], hD[3]);
    }
    return 0;
}
