// Internal helpers shared by the host (.cc) and CUDA (.cu) translation units of libww.
#pragma once
#include <cstdarg>
#include <cstdint>

#include "ww.h"

namespace ww {
inline int64_t words_per_row(int64_t m) { return (m + 15) / 16; }  // 16 codes per word
// WW_LAYOUT_TILE32 geometry: tiles of 32 rows, slabs of 64 columns (4 words)
inline int64_t tile32_tiles(int64_t n) { return (n + 31) / 32; }
inline int64_t tile32_slabs(int64_t m) { return (words_per_row(m) + 3) / 4; }
ww_status fail(ww_status s, const char* fmt, ...);                  // sets ww_last_error()
ww_status ok();
// per-device launch state (ww_device.cu; cached per device, mutex-guarded)
int current_device();
int device_sms();                                          // SM count of the current device
int prepare_kernel(const void* fn, int max_dynamic_smem);  // cudaError_t of the attribute calls
// CUtensorMap of x as [B][W][32 floats], 32 x 32 boxes, 128B swizzle (0 on success)
int encode_x_map(void* map, const float* X, int64_t W, int64_t B, int64_t ldx);
// WW_LAYOUT_LUT81 device packer (ww_lut.cu); returns the cudaError_t of the launch
int pack_lut81_device(const int8_t* planes_d, int64_t n, int64_t m, int64_t ld, uint32_t* out_d,
                      int32_t* bad_d, void* stream);
}  // namespace ww
