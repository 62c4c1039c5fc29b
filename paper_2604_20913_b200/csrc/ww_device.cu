// Per-device launch state of libww: SM counts and the one-time kernel attributes (maximum
// dynamic shared memory, shared-memory carveout).  Both are properties of a (device,
// function) pair, so they are cached per device behind a mutex: a process that drives
// several GPUs from one or many threads gets each device's own values (ww.h: thread-safe,
// no global state besides caches keyed by device and the thread-local error string).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>
#include <set>
#include <utility>

#include "ww_internal.h"

namespace ww {
namespace {
std::mutex g_mu;
std::set<std::pair<int, const void*>> g_prepared;  // (device, kernel) attributes set
constexpr int kMaxDevices = 64;
int g_sms[kMaxDevices] = {};  // 0 = not queried yet (guarded by g_mu)
}  // namespace

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    return dev;
}

int device_sms() {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev < 0 || dev >= kMaxDevices) {
        int c = 0;
        return cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && c > 0
                   ? c
                   : 148;
    }
    if (!g_sms[dev]) {
        int c = 0;
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || c <= 0)
            c = 148;  // B200
        g_sms[dev] = c;
    }
    return g_sms[dev];
}

int prepare_kernel(const void* fn, int max_dynamic_smem) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_prepared.count({dev, fn})) return 0;
    cudaError_t e =
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dynamic_smem);
    if (e != cudaSuccess) return (int)e;
    // always the largest shared-memory carveout: consecutive launches of different shapes then
    // never force an L1/shared reconfiguration, and a PDL-launched next kernel can co-reside
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return (int)e;
    g_prepared.insert({dev, fn});
    return 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link); the
// entry point is process-wide (not per device): resolved once, thread-safe
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        return nullptr;
    }();
    return fn;
}

// x viewed as a [B][W][32 floats] tensor (one 128-byte row per 16-column chunk); boxes of
// 32 chunks x 128 B land 128B-swizzled, i.e. granule g of chunk tc at g ^ (tc & 7) -- the
// layout the sweep reads.  Chunks past W (the last box's tail) are zero-filled.  Needs a
// 16-B aligned x and 16 | m (checked by the callers).
int encode_x_map(void* map, const float* X, int64_t W, int64_t B, int64_t ldx) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return -1;
    const cuuint64_t dims[3] = {32, (cuuint64_t)W, (cuuint64_t)B};
    const cuuint64_t strides[2] = {128, (cuuint64_t)ldx * 8};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(reinterpret_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                     const_cast<float*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)r;
}

}  // namespace ww

// Keep [ptr, ptr + bytes) resident in L2 for kernels launched on `stream` (and kernel nodes
// captured from it): an access-policy window with hit ratio 1 (persisting) and streaming
// misses, after reserving that much persisting L2 (capped by the device's maximum).  For the
// activations of a decode step, which every CTA of the next stage re-reads while the weights
// stream through L2.  bytes == 0 clears the window.
extern "C" ww_status ww_stream_keep_in_l2(void* stream, const void* ptr, size_t bytes) {
    cudaStreamAttrValue v;
    memset(&v, 0, sizeof v);
    if (bytes) {
        if (!ptr) return ww::fail(WW_ERR_INVALID_ARGUMENT, "ww_stream_keep_in_l2: null pointer");
        int dev = ww::current_device(), maxp = 0, maxw = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        if (maxp <= 0 || maxw <= 0)
            return ww::fail(WW_ERR_UNSUPPORTED, "ww_stream_keep_in_l2: no persisting L2 on this device");
        const size_t want = bytes < (size_t)maxp ? bytes : (size_t)maxp;
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        if (cur < want) {
            cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
            if (e != cudaSuccess)
                return ww::fail(WW_ERR_CUDA, "ww_stream_keep_in_l2: %s", cudaGetErrorString(e));
        }
        v.accessPolicyWindow.base_ptr = const_cast<void*>(ptr);
        v.accessPolicyWindow.num_bytes = bytes < (size_t)maxw ? bytes : (size_t)maxw;
        v.accessPolicyWindow.hitRatio = 1.0f;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
    cudaError_t e = cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &v);
    if (e != cudaSuccess) return ww::fail(WW_ERR_CUDA, "ww_stream_keep_in_l2: %s", cudaGetErrorString(e));
    return ww::ok();
}
