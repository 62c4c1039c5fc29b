// Host side of the C ABI (include/ww.h): error reporting, the App. H packer and its
// inverse for both layouts, re-layout, and the row-shard planner.  Pure host C++.
#include <cstdio>
#include <cstring>
#include <string>

#include "ww.h"
#include "ww_internal.h"

namespace {
thread_local std::string g_last_error;
}

namespace ww {
ww_status fail(ww_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}
ww_status ok() {
    g_last_error.clear();
    return WW_OK;
}
}  // namespace ww

using ww::fail;

extern "C" const char* ww_status_string(ww_status s) {
    switch (s) {
        case WW_OK: return "WW_OK";
        case WW_ERR_INVALID_ARGUMENT: return "WW_ERR_INVALID_ARGUMENT";
        case WW_ERR_DIMENSION_MISMATCH: return "WW_ERR_DIMENSION_MISMATCH";
        case WW_ERR_INVALID_CODE: return "WW_ERR_INVALID_CODE";
        case WW_ERR_INVALID_ENCODING: return "WW_ERR_INVALID_ENCODING";
        case WW_ERR_NONFINITE_SCALE: return "WW_ERR_NONFINITE_SCALE";
        case WW_ERR_MISALIGNED: return "WW_ERR_MISALIGNED";
        case WW_ERR_UNSUPPORTED: return "WW_ERR_UNSUPPORTED";
        case WW_ERR_CUDA: return "WW_ERR_CUDA";
    }
    return "WW_ERR_UNKNOWN";
}

extern "C" const char* ww_last_error(void) { return g_last_error.c_str(); }
extern "C" int32_t ww_version(void) { return WW_VERSION; }

extern "C" size_t ww_packed_bytes(int64_t n, int64_t m) {
    if (n < 0 || m < 0) return 0;
    return (size_t)16 * (size_t)n * (size_t)ww::words_per_row(m);
}

extern "C" size_t ww_packed_bytes_layout(int64_t n, int64_t m, int32_t layout) {
    if (n < 0 || m < 0) return 0;
    if (layout == WW_LAYOUT_PLANAR || layout == WW_LAYOUT_COL4) return ww_packed_bytes(n, m);
    if (layout == WW_LAYOUT_TILE32)
        return (size_t)ww::tile32_tiles(n) * (size_t)ww::tile32_slabs(m) * 2048u;
    if (layout == WW_LAYOUT_LUT81) return (size_t)n * (size_t)((m + 511) / 512) * 512u;
    return 0;
}

namespace {

// 2-bit code of value t (App. H): +1 -> 0b10, -1 -> 0b01, 0 -> 0b00
inline bool code_of(int8_t t, uint32_t* c) {
    if (t == 1) { *c = 2u; return true; }
    if (t == -1) { *c = 1u; return true; }
    if (t == 0) { *c = 0u; return true; }
    return false;
}

inline bool value_of(uint32_t c, int8_t* t) {
    if (c == 3u) return false;  // (1,1) unused
    *t = (int8_t)((int)(c >> 1) - (int)(c & 1u));
    return true;
}

// word index and bit shift of (row i, column j, plane p) in a layout
inline void locate(int32_t layout, int64_t n, int64_t W, int64_t i, int64_t j, int p,
                   int64_t* word, int* shift) {
    const int64_t c = j >> 4;
    const int k = (int)(j & 15);
    if (layout == WW_LAYOUT_PLANAR) {
        *word = ((int64_t)p * n + i) * W + c;
        *shift = 2 * k;
    } else if (layout == WW_LAYOUT_TILE32) {  // App. H word c of (p, i), re-tiled (ww.h)
        const int64_t S = (W + 3) / 4;
        *word = (((i >> 5) * S + (c >> 2)) * 128 + 4 * (i & 31) + p) * 4 + (c & 3);
        *shift = 2 * k;
    } else {  // COL4: byte k of the 16-byte chunk (i, c); slot p within the byte
        *word = (i * W + c) * 4 + (k >> 2);
        *shift = 8 * (k & 3) + 2 * p;
    }
}

bool layout_ok(int32_t l) { return l == WW_LAYOUT_PLANAR || l == WW_LAYOUT_COL4 || l == WW_LAYOUT_TILE32; }

}  // namespace

extern "C" ww_status ww_pack_ternary(const int8_t* u_re, const int8_t* u_im, const int8_t* w_re,
                                     const int8_t* w_im, int64_t n, int64_t m, int64_t ld,
                                     int32_t layout, uint32_t* out) {
    if (!u_re || !u_im || !w_re || !w_im || !out)
        return fail(WW_ERR_INVALID_ARGUMENT, "ww_pack_ternary: null pointer");
    if (n < 1 || m < 1 || ld < m)
        return fail(WW_ERR_INVALID_ARGUMENT, "ww_pack_ternary: n=%lld m=%lld ld=%lld",
                    (long long)n, (long long)m, (long long)ld);
    if (!layout_ok(layout)) return fail(WW_ERR_INVALID_ARGUMENT, "ww_pack_ternary: layout %d", layout);
    const int64_t W = ww::words_per_row(m);
    std::memset(out, 0, ww_packed_bytes_layout(n, m, layout));  // zero codes everywhere, incl. padding
    const int8_t* planes[4] = {u_re, u_im, w_re, w_im};
    for (int p = 0; p < 4; ++p) {
        for (int64_t i = 0; i < n; ++i) {
            const int8_t* row = planes[p] + i * ld;
            for (int64_t j = 0; j < m; ++j) {
                uint32_t c;
                if (!code_of(row[j], &c))
                    return fail(WW_ERR_INVALID_CODE,
                                "ww_pack_ternary: plane %d row %lld col %lld value %d not in {-1,0,1}",
                                p, (long long)i, (long long)j, (int)row[j]);
                int64_t w;
                int s;
                locate(layout, n, W, i, j, p, &w, &s);
                out[w] |= c << s;
            }
        }
    }
    return ww::ok();
}

extern "C" ww_status ww_unpack_ternary(const uint32_t* packed, int64_t n, int64_t m,
                                       int32_t layout, int8_t* u_re, int8_t* u_im, int8_t* w_re,
                                       int8_t* w_im, int64_t ld) {
    if (!packed || !u_re || !u_im || !w_re || !w_im)
        return fail(WW_ERR_INVALID_ARGUMENT, "ww_unpack_ternary: null pointer");
    if (n < 1 || m < 1 || ld < m)
        return fail(WW_ERR_INVALID_ARGUMENT, "ww_unpack_ternary: n=%lld m=%lld ld=%lld",
                    (long long)n, (long long)m, (long long)ld);
    if (!layout_ok(layout)) return fail(WW_ERR_INVALID_ARGUMENT, "ww_unpack_ternary: layout %d", layout);
    const int64_t W = ww::words_per_row(m);
    int8_t* planes[4] = {u_re, u_im, w_re, w_im};
    for (int p = 0; p < 4; ++p) {
        for (int64_t i = 0; i < n; ++i) {
            for (int64_t j = 0; j < 16 * W; ++j) {  // padding slots are validated too
                int64_t w;
                int s;
                locate(layout, n, W, i, j, p, &w, &s);
                int8_t t;
                if (!value_of((packed[w] >> s) & 3u, &t))
                    return fail(WW_ERR_INVALID_ENCODING,
                                "ww_unpack_ternary: slot (1,1) at plane %d row %lld col %lld", p,
                                (long long)i, (long long)j);
                if (j < m) planes[p][i * ld + j] = t;
            }
        }
    }
    return ww::ok();
}

extern "C" ww_status ww_repack(const uint32_t* src, int32_t src_layout, int64_t n, int64_t m,
                               uint32_t* dst, int32_t dst_layout) {
    if (!src || !dst || src == dst) return fail(WW_ERR_INVALID_ARGUMENT, "ww_repack: bad pointers");
    if (n < 1 || m < 1) return fail(WW_ERR_INVALID_ARGUMENT, "ww_repack: n=%lld m=%lld", (long long)n, (long long)m);
    if (!layout_ok(src_layout) || !layout_ok(dst_layout))
        return fail(WW_ERR_INVALID_ARGUMENT, "ww_repack: layouts %d -> %d", src_layout, dst_layout);
    const int64_t W = ww::words_per_row(m);
    std::memset(dst, 0, ww_packed_bytes_layout(n, m, dst_layout));
    for (int p = 0; p < 4; ++p)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < 16 * W; ++j) {
                int64_t ws, wd;
                int ss, sd;
                locate(src_layout, n, W, i, j, p, &ws, &ss);
                locate(dst_layout, n, W, i, j, p, &wd, &sd);
                dst[wd] |= ((src[ws] >> ss) & 3u) << sd;
            }
    return ww::ok();
}

// Ceil-block row partition (S:240-248 balanced split when world | n; equal counts for the
// NCCL all-gather otherwise).
extern "C" ww_status ww_shard_plan(int64_t n, int64_t m, int32_t world, int32_t rank,
                                   ww_shard* out) {
    if (!out) return fail(WW_ERR_INVALID_ARGUMENT, "ww_shard_plan: null out");
    if (n < 1 || m < 1 || world < 1 || rank < 0 || rank >= world)
        return fail(WW_ERR_INVALID_ARGUMENT, "ww_shard_plan: n=%lld m=%lld world=%d rank=%d",
                    (long long)n, (long long)m, world, rank);
    const int64_t rpr = (n + world - 1) / world;
    ww_shard s;
    s.world = world;
    s.rank = rank;
    s.n = n;
    s.rows_per_rank = rpr;
    s.n_padded = rpr * world;
    s.row_begin = rpr * rank < n ? rpr * rank : n;
    s.row_end = rpr * (rank + 1) < n ? rpr * (rank + 1) : n;
    const int64_t row_bytes = 16 * ww::words_per_row(m);
    s.packed_offset_bytes = s.row_begin * row_bytes;
    s.packed_bytes = (s.row_end - s.row_begin) * row_bytes;
    s.scale_offset_floats = 4 * s.row_begin;
    s.scale_count = 4 * (s.row_end - s.row_begin);
    s.y_offset_complex = rpr * rank;
    *out = s;
    return ww::ok();
}
