// Per-device launch state of libww: SM counts and the one-time kernel attributes (maximum
// dynamic shared memory, shared-memory carveout).  Both are properties of a (device,
// function) pair, so they are cached per device behind a mutex: a process that drives
// several GPUs from one or many threads gets each device's own values (ww.h: thread-safe,
// no global state besides caches keyed by device and the thread-local error string).
#include <cuda_runtime.h>

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

}  // namespace ww
