// Persistent, stage-chained WL-GEMV "program" (ww.h ww_program_*): one launch runs a whole
// sequence of widely-linear layers -- e.g. one decode step of the config-4 stack, 128
// stages -- with the true data dependency between stages kept by a grid-wide (and, with
// several ranks, GPU-wide) readiness counter instead of kernel boundaries.
//
// Per CTA (one per SM, cooperative launch so all CTAs are co-resident):
//   * 16 consumer warps run the sweep of the single-layer kernel (decode + predicated FADD2,
//     ww_sweep.cuh; a5/a6, Eqs. 4-7), one row per warp at a time, whole rows,
//     contiguous balanced row ranges per CTA and per warp;
//   * 1 producer warp streams the CTA's packed rows, stage after stage, into a shared-memory
//     ring with cp.async.bulk (one bulk copy per row, mbarrier full/empty pairs per slot).
//     Weights never depend on earlier stages, so the producer runs ahead across stage
//     boundaries: while the consumers wait for stage s to finish everywhere, the ring fills
//     with stage s+1's rows (the dead time between dependent GEMVs);
//   * x of a stage is staged once per CTA by TMA (128B swizzle) after the readiness wait;
//   * fused prologue ops on the staged x: RMSNorm (x * gamma / rms) or the
//     elementwise product of two vectors (SiLU(gate) (.) up); fused epilogue ops
//     per row: residual add, or SiLU of the gate rows;
//   * the epilogue stores every output row into the gathered output buffer of every rank
//     (peer-mapped pointers over NVLink at world > 1): the all-gather is fused into the
//     GEMV and the readiness counter of every rank is bumped once per
//     CTA and stage (red.release.sys), so no NCCL call sits between stages.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "ww.h"
#include "ww_internal.h"
#include "ww_sweep.cuh"

namespace {

constexpr int kCW = 16;                  // consumer warps
constexpr int kThreads = (kCW + 1) * 32;  // + one producer warp
constexpr int kMaxSlots = 64;
constexpr int kSmemMax = 227 * 1024;
constexpr int kSyncWords = 128;  // per rank: counter at [0], epoch at [32], exit at [64]

struct alignas(128) StageDev {
    CUtensorMap xmap;   // x as [1][W][32 floats] (ww::encode_x_map)
    CUtensorMap xmap2;  // WW_PRO_MUL: second operand
    const uint4* packed;
    const float* scales;
    const float* residual;
    const float* gamma;
    float* ydst[WW_PROG_MAX_RANKS];
    int64_t n_local, row0, m, W, silu_rows;
    int32_t J, conv, per_row, pro, epi, wait, ndst;
    float eps;
};

struct ProgParams {
    const StageDev* stages;               // [ranks_in_launch][nstages]
    uint32_t* sync[WW_PROG_MAX_RANKS];    // every rank's sync words
    int32_t nstages, world, rank_base, ranks_in_launch, ctas_per_rank;
    int32_t nslot, slot_bytes, x_bytes, has_mul;
    int32_t off_ring, off_scratch, off_part, off_bars;
    unsigned long long* trace;  // tools only (ww_debug_program_trace): per CTA and stage,
                                // globaltimer at [start, polled, x ready, rows done, producer]
};

__device__ __forceinline__ void ptrace(const ProgParams& p, int s, int ev) {
    if (p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[((size_t)blockIdx.x * p.nstages + s) * 8 + ev] = t;
    }
}

// ------------------------------------------------------------------ PTX helpers (program only)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint4 lds128u(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ void bar_consumers() {  // named barrier 1: the 16 consumer warps
    asm volatile("bar.sync 1, %0;" ::"n"(kCW * 32) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ float2 ldcg2(const float* p) {  // L2 only: written by other CTAs
    float2 v;
    asm volatile("ld.global.cg.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

// whole rows of a stage packed into one ring slot (one bulk copy, one full/empty pair)
__host__ __device__ __forceinline__ int rows_per_slot(int slot_bytes, int row_bytes) {
    const int r = slot_bytes / row_bytes;
    return r < 1 ? 1 : r;
}

// per-warp contiguous row range [w0, w1) of a CTA's NRc rows (sizes differ by <= 1, the
// longer ranges on the first warps: equal work per SM sub-partition, +-1 row)
__device__ __forceinline__ void warp_rows(int NRc, int warp, int& w0, int& w1) {
    const int ub = NRc / kCW, ue = NRc - ub * kCW;
    w0 = warp * ub + (warp < ue ? warp : ue);
    w1 = w0 + ub + (warp < ue ? 1 : 0);
}

__global__ void __launch_bounds__(kThreads, 1) wl_program_kernel(const __grid_constant__ ProgParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* smem = smem_raw + (base - raw);
    const uint32_t xa = base, xb = base + (uint32_t)p.x_bytes;  // x regions (xb: WW_PRO_MUL)
    const uint32_t ring = base + (uint32_t)p.off_ring;
    const uint32_t bars = base + (uint32_t)p.off_bars;  // full[nslot], empty[nslot], xbar
    const uint32_t xbar = bars + 16u * (uint32_t)p.nslot;
    float* part = reinterpret_cast<float*>(smem + p.off_part);  // [kCW] + norm factor

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rl = blockIdx.x / p.ctas_per_rank;  // rank within this launch
    const int ci = blockIdx.x - rl * p.ctas_per_rank;
    const int me = p.rank_base + rl;
    const StageDev* SD = p.stages + (size_t)rl * p.nstages;
    uint32_t* my_sync = p.sync[me];
    const uint32_t T = (uint32_t)(p.world * p.ctas_per_rank);  // signals per stage per rank

    if (threadIdx.x == 0) {
        for (int k = 0; k < p.nslot; ++k) {
            mbar_init(bars + 8u * k, 1);                       // full[k]: producer expect_tx
            mbar_init(bars + 8u * (p.nslot + k), 1);           // empty[k]: consumer lane 0
        }
        mbar_init(xbar, 1);
        fence_barrier_init();
    }
    // epoch of this launch (advanced by the last CTA of the previous launch on this rank)
    const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(my_sync + 32);
    __syncthreads();

    if (warp == kCW) {
        // ---------------------------------------------------------------- producer warp
        if (lane == 0) {
            uint32_t seq = 0;
            for (int s = 0; s < p.nstages; ++s) {
                const StageDev& D = SD[s];
                const int64_t n = D.n_local;
                const int64_t r0 = ci * n / p.ctas_per_rank, r1 = (ci + 1) * n / p.ctas_per_rank;
                const int NRc = (int)(r1 - r0);
                const int ub = NRc / kCW, ue = NRc - ub * kCW;
                const uint32_t rb = (uint32_t)(16 * D.W);
                const int rps = rows_per_slot(p.slot_bytes, (int)rb);
                const int U0 = (ub + rps - 1) / rps, U1 = (ub + rps) / rps;  // units per warp
                const uint4* src0 = D.packed + r0 * D.W;
                for (int u = 0; u < (ue ? U1 : U0); ++u) {
                    for (int w = 0; w < kCW; ++w) {
                        const int nr = ub + (w < ue ? 1 : 0);  // the warp's rows
                        if (u * rps >= nr) break;  // warps holding unit u are a prefix
                        const int q0 = u * rps;
                        const int cnt = nr - q0 < rps ? nr - q0 : rps;
                        const int r = w * ub + (w < ue ? w : ue) + q0;
                        const int k = (int)(seq % (uint32_t)p.nslot);
                        const uint32_t use = seq / (uint32_t)p.nslot;
                        if (use > 0) mbar_wait(bars + 8u * (p.nslot + k), (use - 1) & 1);
                        mbar_expect_tx(bars + 8u * k, rb * (uint32_t)cnt);
                        bulk_g2s(ring + (uint32_t)k * p.slot_bytes, src0 + (int64_t)r * D.W,
                                 rb * (uint32_t)cnt, bars + 8u * k);
                        ++seq;
                    }
                }
                ptrace(p, s, 4);
            }
        }
        return;
    }

    // -------------------------------------------------------------------- consumer warps
    float* scratch = reinterpret_cast<float*>(smem + p.off_scratch) + warp * 8;
    const uint32_t l7 = (uint32_t)(lane & 7) << 4;
    const uint32_t xl = (xa + (uint32_t)lane * 128u) | l7;  // lane's chunk, swizzle key
    uint32_t seq_base = 0, xphase = 0;
    Acc<1> acc;
    acc.zero();
    for (int s = 0; s < p.nstages; ++s) {
        const StageDev& D = SD[s];
        const int64_t n = D.n_local;
        const int J = D.J, pro = D.pro, epi = D.epi;
        const int64_t r0 = ci * n / p.ctas_per_rank, r1 = (ci + 1) * n / p.ctas_per_rank;
        const int NRc = (int)(r1 - r0);
        int w0, w1;
        warp_rows(NRc, warp, w0, w1);

        // ---- readiness: stage s reads what stage s-1 wrote on every rank
        if (threadIdx.x == 0) ptrace(p, s, 0);
        if (s > 0) {
            bar_consumers();  // this CTA's rows of stage s-1 are stored
            if (threadIdx.x == 0) {
                // release (cumulative over the CTA's stores ordered before bar.sync): GPU
                // scope on one GPU, system scope when peers read the stored rows
                if (p.world == 1)
                    red_release_gpu(p.sync[0], 1u);
                else
                    for (int g = 0; g < p.world; ++g) red_release_sys(p.sync[g], 1u);
            }
        }
        float4 gam[kGammaRegs];  // RMSNorm gamma (a weight): loaded before the wait
        float rnorm = 1.0f;
        if (pro == WW_PRO_RMSNORM) gamma_prefetch(gam, D.gamma, D.m, J, threadIdx.x, kCW * 32);
        if (D.wait && threadIdx.x == 0) {
            const uint32_t target = epoch * (uint32_t)(p.nstages - 1) * T + (uint32_t)s * T;
            if (p.world == 1)
                while ((int32_t)(ld_acquire_gpu(my_sync) - target) < 0) __nanosleep(32);
            else
                while ((int32_t)(ld_acquire_sys(my_sync) - target) < 0) __nanosleep(32);
        }
        if (threadIdx.x == 0) ptrace(p, s, 1);
        bar_consumers();
        // ---- x (and the second operand) by TMA into the swizzled x regions
        if (threadIdx.x == 0) {
            fence_proxy_async();
            const uint32_t nb = (uint32_t)J * 4096u * (pro == WW_PRO_MUL ? 2u : 1u);
            mbar_expect_tx(xbar, nb);
            for (int j = 0; j < J; ++j) {
                tma_load_3d(xa + (uint32_t)j * 4096u, &D.xmap, 0, 32 * j, 0, xbar);
                if (pro == WW_PRO_MUL) tma_load_3d(xb + (uint32_t)j * 4096u, &D.xmap2, 0, 32 * j, 0, xbar);
            }
        }
        mbar_wait(xbar, xphase);
        xphase ^= 1u;
        if (threadIdx.x == 0) ptrace(p, s, 2);
        // (event 3: prologue done, below)
        // ---- fused prologue ops on the staged x (granule gi = 16 B = 2 complex columns)
        if (pro != WW_PRO_NONE) {
            const int ng = 8 * 32 * J;
            if (pro == WW_PRO_MUL) {  // x = a (.) b, re and im separately (real view)
                x_mul(xa, xb, ng, threadIdx.x, kCW * 32);
            } else {  // RMSNorm over the real 2m-vector: x * gamma, 1/rms in the epilogue
                const float ss =
                    x_gamma_sumsq_warp(xa, ng, threadIdx.x, kCW * 32, gam, D.gamma, D.m);
                if (lane == 0) part[warp] = ss;
            }
            bar_consumers();
            if (pro == WW_PRO_RMSNORM) rnorm = rms_factor(part, kCW, D.m, D.eps);
        }

        // ---- the warp's rows, in units of up to rps consecutive rows per ring slot:
        // weights from the ring, x from shared memory.  The stage's fields are copied to
        // registers once (the mbarrier asm clobbers memory: no reloads in the row loop).
        const uint32_t rb = (uint32_t)(16 * D.W);
        const int rps = rows_per_slot(p.slot_bytes, (int)rb);
        const float* const scl = D.scales + (D.per_row ? 4 * r0 : 0);
        const int sstep = D.per_row ? 4 : 0;
        const float* const resid = D.residual;
        const int conv = D.conv, ndst = D.ndst;
        const int64_t grow0 = D.row0 + r0, silu_rows = D.silu_rows;
        float2* const ydst0 = reinterpret_cast<float2*>(D.ydst[0]);
        unsigned long long waited = 0;
        int j = rps;  // row within the current unit (rps: start a new unit)
        uint32_t useq = seq_base + (uint32_t)warp - kCW, slot = 0;
        for (int r = w0; r < w1; ++r) {
            if (j == rps) {  // next unit: its ring slot, wait until the bulk copy landed
                j = 0;
                useq += kCW;
                const uint32_t k = useq % (uint32_t)p.nslot;
                slot = k;
                unsigned long long t0 = 0;
                if (p.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                mbar_wait(bars + 8u * k, (useq / (uint32_t)p.nslot) & 1);
                if (p.trace) {
                    unsigned long long t1;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                    waited += t1 - t0;
                }
            }
            const bool last_in_unit = j == rps - 1 || r == w1 - 1;
            const int64_t grow = grow0 + r;  // global row index of the stage
            float4 sc = make_float4(0.f, 0.f, 0.f, 0.f);
            float2 res = make_float2(0.f, 0.f);
            if (lane == 0) {  // row operands of the epilogue, fetched a row ahead of use
                sc = __ldg(reinterpret_cast<const float4*>(scl + sstep * r));
                if (epi == WW_EPI_RESIDUAL) res = ldcg2(resid + 2 * grow);
            }
            const uint32_t wl = ring + slot * (uint32_t)p.slot_bytes + (uint32_t)j * rb + (uint32_t)lane * 16u;
            uint32_t xc = xl;
            uint4 cur = lds128u(wl);
#pragma unroll 1
            for (int kk = 0; kk < J; ++kk) {
                const uint4 nxt = lds128u(wl + 512u * (kk + 1));  // (ring has a 512-B tail)
                chunk<1>(acc, cur, xc, 0);
                cur = nxt;
                xc += 4096u;
            }
            __syncwarp();
            if (last_in_unit && lane == 0) mbar_arrive(bars + 8u * (p.nslot + slot));  // free
            ++j;
            reduce_to<1>(acc, scratch);
            acc.zero();
            if (lane == 0) {
                float Tt[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) Tt[i] = scratch[i];
                float yre = sc.x * Tt[0] - sc.y * Tt[3] + sc.z * Tt[4] + sc.w * Tt[7];  // Eq. 2
                float yim = conv == WW_CONV_EQ1
                                ? sc.x * Tt[1] + sc.y * Tt[2] - sc.z * Tt[5] + sc.w * Tt[6]   // Eq. 1
                                : sc.x * Tt[1] + sc.y * Tt[2] + sc.z * Tt[5] - sc.w * Tt[6];  // Eq. 3
                if (pro == WW_PRO_RMSNORM) {  // RMSNorm scalar (linear map)
                    yre = yre * rnorm;
                    yim = yim * rnorm;
                }
                if (epi == WW_EPI_RESIDUAL) {
                    yre = yre + res.x;
                    yim = yim + res.y;
                } else if (epi == WW_EPI_SILU && grow < silu_rows) {
                    yre = silu_f(yre);
                    yim = silu_f(yim);
                }
                ydst0[grow] = make_float2(yre, yim);
                for (int g = 1; g < ndst; ++g)
                    reinterpret_cast<float2*>(SD[s].ydst[g])[grow] = make_float2(yre, yim);
            }
        }
        if (warp == 0 && lane == 0 && p.trace)
            p.trace[((size_t)blockIdx.x * p.nstages + s) * 8 + 3] = waited;  // (replaces event 3)
        {
            const int ub = NRc / kCW, ue = NRc - ub * kCW;
            const int U0 = (ub + rps - 1) / rps, U1 = (ub + rps) / rps;
            seq_base += (uint32_t)(kCW * U0 + (U1 > U0 ? ue : 0));  // units of the stage
        }
        if (lane == 0 && (warp == 0 || warp == 8 || warp == kCW - 1))
            ptrace(p, s, warp == 0 ? 5 : (warp == 8 ? 7 : 6));
    }

    // ---- exit: the last CTA of this rank advances the epoch for the next launch
    bar_consumers();
    if (threadIdx.x == 0) {
        const uint32_t old = atomicAdd(my_sync + 64, 1u);
        if (old == (uint32_t)p.ctas_per_rank - 1) {
            my_sync[64] = 0;
            *reinterpret_cast<volatile uint32_t*>(my_sync + 32) = epoch + 1;
        }
    }
}

}  // namespace

// ---------------------------------------------------------------------------- host side
static unsigned long long* g_prog_trace = nullptr;  // tools only
// Not part of the ABI (no declaration in ww.h): tools/prog_trace.py points the program kernel
// at a device buffer of grid x nstages x 8 u64 globaltimer stamps (NULL: off, the default).
extern "C" void ww_debug_program_trace(void* dev_buf) {
    g_prog_trace = reinterpret_cast<unsigned long long*>(dev_buf);
}

static_assert(sizeof(StageDev) % 128 == 0, "descriptor alignment");

extern "C" size_t ww_program_workspace_bytes(int32_t nstages, int32_t ranks_in_launch) {
    if (nstages < 1 || ranks_in_launch < 1) return 0;
    return sizeof(StageDev) * (size_t)nstages * (size_t)ranks_in_launch;
}

extern "C" size_t ww_program_sync_bytes(void) { return kSyncWords * sizeof(uint32_t) * 4; }

extern "C" ww_status ww_program_init(const ww_stage* stages, int32_t nstages, int32_t world,
                                     int32_t rank_base, int32_t ranks_in_launch,
                                     uint32_t* const* sync_d, void* workspace_d, ww_program* out) {
    const char* fn = "ww_program_init";
    if (!stages || !sync_d || !workspace_d || !out)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: null pointer", fn);
    if (nstages < 1 || world < 1 || world > WW_PROG_MAX_RANKS || ranks_in_launch < 1 ||
        rank_base < 0 || rank_base + ranks_in_launch > world)
        return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: nstages=%d world=%d rank_base=%d ranks=%d", fn,
                        nstages, world, rank_base, ranks_in_launch);
    if ((uintptr_t)workspace_d & 127) return ww::fail(WW_ERR_MISALIGNED, "%s: workspace", fn);
    for (int g = 0; g < world; ++g)
        if (!sync_d[g] || ((uintptr_t)sync_d[g] & 127))
            return ww::fail(WW_ERR_MISALIGNED, "%s: sync words of rank %d", fn, g);
    const int sms = ww::device_sms();
    const int cpr = sms / ranks_in_launch;
    if (cpr < 1) return ww::fail(WW_ERR_UNSUPPORTED, "%s: %d ranks on %d SMs", fn, ranks_in_launch, sms);

    std::vector<StageDev> dev((size_t)nstages * ranks_in_launch);
    int64_t Wmax = 1, Jmax = 1;
    bool has_mul = false;
    for (int r = 0; r < ranks_in_launch; ++r) {
        for (int s = 0; s < nstages; ++s) {
            const ww_stage& S = stages[(size_t)r * nstages + s];
            StageDev& D = dev[(size_t)r * nstages + s];
            memset(&D, 0, sizeof D);
            if (S.m < 16 || S.m % 16 || S.m > WW_PROG_MAX_M || S.n_local < 0 || S.row0 < 0 ||
                (S.n_local > 0 && (!S.packed || !S.scales)) || !S.x)
                return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: stage %d rank %d: m=%lld n_local=%lld",
                                fn, s, rank_base + r, (long long)S.m, (long long)S.n_local);
            if (S.scale_mode != WW_SCALES_PER_ROW && S.scale_mode != WW_SCALES_PER_TENSOR)
                return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: stage %d scale_mode", fn, s);
            if (S.conv != WW_CONV_EQ1 && S.conv != WW_CONV_ALG1)
                return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: stage %d conv", fn, s);
            if (S.prologue < WW_PRO_NONE || S.prologue > WW_PRO_MUL || S.epilogue < WW_EPI_NONE ||
                S.epilogue > WW_EPI_SILU || (S.prologue == WW_PRO_MUL && !S.x2) ||
                (S.prologue == WW_PRO_RMSNORM && (!S.gamma || !(S.eps >= 0.f))) ||
                (S.epilogue == WW_EPI_RESIDUAL && !S.residual))
                return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: stage %d ops", fn, s);
            if (((uintptr_t)S.packed & 15) || ((uintptr_t)S.scales & 15) || ((uintptr_t)S.x & 15) ||
                ((uintptr_t)S.x2 & 15) || ((uintptr_t)S.residual & 7) || ((uintptr_t)S.gamma & 15))
                return ww::fail(WW_ERR_MISALIGNED, "%s: stage %d pointers", fn, s);
            for (int g = 0; g < world; ++g)
                if (!S.y[g] || ((uintptr_t)S.y[g] & 7))
                    return ww::fail(WW_ERR_MISALIGNED, "%s: stage %d y[%d]", fn, s, g);
            D.packed = reinterpret_cast<const uint4*>(S.packed);
            D.scales = S.scales;
            D.residual = S.residual;
            D.gamma = S.gamma;
            for (int g = 0; g < world; ++g) D.ydst[g] = S.y[g];
            D.ndst = world;
            D.n_local = S.n_local;
            D.row0 = S.row0;
            D.m = S.m;
            D.W = S.m / 16;
            D.J = (int32_t)((D.W + 31) / 32);
            D.silu_rows = S.silu_rows;
            D.conv = S.conv;
            D.per_row = S.scale_mode == WW_SCALES_PER_ROW;
            D.pro = S.prologue;
            D.epi = S.epilogue;
            D.wait = S.wait != 0;
            D.eps = S.eps;
            if (ww::encode_x_map(&D.xmap, S.x, D.W, 1, S.m) != 0 ||
                (S.prologue == WW_PRO_MUL && ww::encode_x_map(&D.xmap2, S.x2, D.W, 1, S.m) != 0))
                return ww::fail(WW_ERR_CUDA, "%s: stage %d: tensor map encoding failed", fn, s);
            Wmax = D.W > Wmax ? D.W : Wmax;
            Jmax = D.J > Jmax ? D.J : Jmax;
            has_mul |= S.prologue == WW_PRO_MUL;
        }
    }
    // shared memory: x (+ x2) regions, weight ring (+ 512-B tail read by the sweep's
    // one-ahead load), per-warp totals, norm partials, mbarriers
    const int x_bytes = (int)(Jmax * 4096);
    const int slot = (int)((16 * Wmax + 127) / 128 * 128);
    const int off_ring = x_bytes * (has_mul ? 2 : 1);
    const int fixed = 512 + kCW * 8 * 4 + 32 * 4 + 8 * (2 * kMaxSlots + 1) + 1024 + 64;
    int nslot = (kSmemMax - off_ring - fixed) / slot;
    if (nslot > kMaxSlots) nslot = kMaxSlots;
    if (nslot < 2)
        return ww::fail(WW_ERR_UNSUPPORTED, "%s: m=%lld leaves no room for the weight ring", fn,
                        (long long)(16 * Wmax));
    const int off_scratch = off_ring + nslot * slot + 512;
    const int off_part = off_scratch + kCW * 8 * 4;
    const int off_bars = (off_part + 32 * 4 + 7) / 8 * 8;
    const int smem = off_bars + 8 * (2 * nslot + 1) + 1024;  // + base alignment slack

    cudaError_t e = cudaMemcpy(workspace_d, dev.data(), dev.size() * sizeof(StageDev),
                               cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return ww::fail(WW_ERR_CUDA, "%s: %s", fn, cudaGetErrorString(e));
    ww_program P;
    memset(&P, 0, sizeof P);
    P.nstages = nstages;
    P.world = world;
    P.rank_base = rank_base;
    P.ranks_in_launch = ranks_in_launch;
    P.ctas_per_rank = cpr;
    P.grid = cpr * ranks_in_launch;
    P.block = kThreads;
    P.smem_bytes = smem;
    P.nslot = nslot;
    P.slot_bytes = slot;
    P.x_bytes = x_bytes;
    P.has_mul = has_mul;
    P.workspace = workspace_d;
    for (int g = 0; g < world; ++g) P.sync[g] = sync_d[g];
    *out = P;
    return ww::ok();
}

extern "C" ww_status ww_program_run(const ww_program* P, void* stream) {
    const char* fn = "ww_program_run";
    if (!P || !P->workspace) return ww::fail(WW_ERR_INVALID_ARGUMENT, "%s: null program", fn);
    ProgParams p;
    memset(&p, 0, sizeof p);
    p.stages = reinterpret_cast<const StageDev*>(P->workspace);
    for (int g = 0; g < P->world; ++g) p.sync[g] = P->sync[g];
    p.nstages = P->nstages;
    p.world = P->world;
    p.rank_base = P->rank_base;
    p.ranks_in_launch = P->ranks_in_launch;
    p.ctas_per_rank = P->ctas_per_rank;
    p.nslot = P->nslot;
    p.slot_bytes = P->slot_bytes;
    p.x_bytes = P->x_bytes;
    p.has_mul = P->has_mul;
    p.off_ring = P->x_bytes * (P->has_mul ? 2 : 1);
    p.off_scratch = p.off_ring + P->nslot * P->slot_bytes + 512;
    p.off_part = p.off_scratch + kCW * 8 * 4;
    p.off_bars = (p.off_part + 32 * 4 + 7) / 8 * 8;
    p.trace = g_prog_trace;
    const int pe = ww::prepare_kernel(reinterpret_cast<const void*>(wl_program_kernel), kSmemMax);
    if (pe) return ww::fail(WW_ERR_CUDA, "%s: %s", fn, cudaGetErrorString((cudaError_t)pe));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P->grid);
    cfg.blockDim = dim3((unsigned)P->block);
    cfg.dynamicSmemBytes = (size_t)P->smem_bytes;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, wl_program_kernel, p);
    if (e != cudaSuccess) return ww::fail(WW_ERR_CUDA, "%s: launch failed: %s", fn, cudaGetErrorString(e));
    return ww::ok();
}
