// Internal helpers shared by the host (.cc) and CUDA (.cu) translation units of libww.
#pragma once
#include <cstdarg>
#include <cstdint>

#include "ww.h"

namespace ww {
inline int64_t words_per_row(int64_t m) { return (m + 15) / 16; }  // 16 codes per word
ww_status fail(ww_status s, const char* fmt, ...);                  // sets ww_last_error()
ww_status ok();
// per-device launch state (ww_device.cu; cached per device, mutex-guarded)
int current_device();
int device_sms();                                          // SM count of the current device
int prepare_kernel(const void* fn, int max_dynamic_smem);  // cudaError_t of the attribute calls
}  // namespace ww
