// Internal helpers shared by the host (.cc) and CUDA (.cu) translation units of libww.
#pragma once
#include <cstdarg>
#include <cstdint>

#include "ww.h"

namespace ww {
inline int64_t words_per_row(int64_t m) { return (m + 15) / 16; }  // 16 codes per word
ww_status fail(ww_status s, const char* fmt, ...);                  // sets ww_last_error()
ww_status ok();
}  // namespace ww
