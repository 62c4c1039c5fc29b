/* ww.h — C ABI of the B200-native fused ternary widely-linear GEMV
 * (FairyFuse, arXiv 2604.20913).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
 *
 * Operation (Eq. 1; Eqs. 2-3; Alg. 1):
 *   y = U x + W conj(x)                     (WW_CONV_EQ1, default)
 *   y = (U + conj(W)) x   == Eqs. 2-3        (WW_CONV_ALG1)
 *   U = diag(sUr) U_re + i diag(sUi) U_im,  W = diag(sWr) W_re + i diag(sWi) W_im,
 *   U_re, U_im, W_re, W_im in {-1,0,+1}^{n x m}; the only multiplies are the 8 scale
 *   multiplies per output row after accumulation.
 *
 * Ternary code (App. H): 2 bits (b1,b0), (1,0) = +1, (0,1) = -1,
 * (0,0) = 0, (1,1) unused.  Layouts of the packed weights (all little-endian uint32):
 *   WW_LAYOUT_PLANAR: the paper's App. H format.  Four planes back to back in the order
 *     U_re, U_im, W_re, W_im; each plane row-major n x W words, W = ceil(m/16);
 *     column j of a row is slot (j % 16) of word (j / 16): bit 2k+1 = +1, bit 2k = -1;
 *     padding columns carry the zero code.
 *   WW_LAYOUT_COL4 (device layout, consumed by the GPU kernels): row-major n x W "chunks"
 *     of 16 bytes (one uint4 per 16 columns); byte k of chunk c of row i holds the four
 *     codes of column 16c+k with the App. H bit rule applied per plane:
 *     bit 2p+1 = (plane p code == +1), bit 2p = (plane p code == -1), p = 0..3 =
 *     U_re, U_im, W_re, W_im.  Same 2 bits per code (n*W*16 bytes = n*m when 16 | m);
 *     the bit order is chosen so one R2P decodes a column's predicates.
 *   WW_LAYOUT_TILE32 (device layout of the tensor-core path, ww_wl_gemv_tc): the App. H
 *     words themselves, re-tiled.  Rows are grouped in tiles of 32, columns in slabs of 64
 *     (4 words), S = ceil(W/4); the 512 words of (tile t, slab s) are contiguous, M-row
 *     major: word index ((t*S + s)*128 + 4*(i%32) + p)*4 + (w%4) holds App. H word w of
 *     plane p, row i (t = i/32, s = w/4).  Rows past n and words past W are zero codes.
 *     ww_packed_bytes_layout(): ceil(n/32) * S * 2048 bytes (2 bits per code, the same bytes
 *     as the other layouts when 32 | n and 64 | m).
 *   WW_LAYOUT_LUT81 (device layout of the lookup path, ww_wl_gemv_lut): one byte per 4 codes
 *     of one plane, byte = sum_k (code_k + 1) 3^k over columns 4g..4g+3 (0..80; 40 = four
 *     zero codes) -- a bijection of the four App. H bit pairs, still 2 bits per code.  Rows
 *     are T = ceil(m/512) steps of 512 bytes: byte 16*((i*T + t)*32 + l) + 4*p + k holds
 *     plane p, row i, columns 512t + 128k + 4l .. +3 (padding columns are zero codes).
 *     Converted on the host from / to WW_LAYOUT_PLANAR (ww_lut81_from_planar / _to_planar);
 *     ww_lut81_packed_bytes(): n * T * 512.
 *
 * Scales (R2): WW_SCALES_PER_ROW = n x 4 fp32 [sUr, sUi, sWr, sWi] row-major;
 *   WW_SCALES_PER_TENSOR = 4 fp32 shared by all rows.
 * Activations / outputs: complex64 = interleaved (re, im) fp32 pairs (torch.complex64).
 *
 * Conventions: every buffer is caller-allocated; the library never allocates or frees
 * and holds no global state besides a thread-local error string.  Host functions are
 * synchronous and thread-safe.  GPU entry points are asynchronous on `stream`
 * (a cudaStream_t passed as void*, NULL = legacy default stream), never synchronize,
 * validate arguments before launching, and map launch failures to WW_ERR_CUDA (faults
 * inside a kernel surface at the caller's next synchronization).  Numerics: fp32
 * round-to-nearest accumulation in an unspecified but deterministic order (bitwise
 * repeatable for a given shape and batch), no FTZ, no fast-math.
 */
#ifndef WW_H
#define WW_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define WW_VERSION 1

typedef enum {
    WW_OK = 0,
    WW_ERR_INVALID_ARGUMENT = 1,   /* null pointer, n<1, m<1, B<1, ld<m, world<1, rank out of range */
    WW_ERR_DIMENSION_MISMATCH = 2, /* e.g. ldx < m, ldy < n */
    WW_ERR_INVALID_CODE = 3,       /* dense weight value not in {-1,0,+1} */
    WW_ERR_INVALID_ENCODING = 4,   /* slot pattern (1,1) met while unpacking */
    WW_ERR_NONFINITE_SCALE = 5,    /* reserved: scales live on the device and are not inspected */
    WW_ERR_MISALIGNED = 6,         /* packed not 16-B aligned, x / y not 8-B aligned */
    WW_ERR_UNSUPPORTED = 7,        /* B > WW_MAX_BATCH, layout not COL4 on the GPU, ... */
    WW_ERR_CUDA = 8                /* a CUDA runtime call failed; see ww_last_error() */
} ww_status;

typedef enum { WW_LAYOUT_PLANAR = 0, WW_LAYOUT_COL4 = 1, WW_LAYOUT_TILE32 = 2, WW_LAYOUT_LUT81 = 3 } ww_layout;
typedef enum { WW_CONV_EQ1 = 0, WW_CONV_ALG1 = 1 } ww_convention;
typedef enum { WW_SCALES_PER_TENSOR = 0, WW_SCALES_PER_ROW = 1 } ww_scale_mode;

/* launch flags (ww_layer.flags) */
#define WW_FLAG_PDL 1u /* programmatic dependent launch: the kernel starts streaming its
                          packed weights while the previous kernel on the stream finishes
                          (so that kernel must not write the packed weights), and waits
                          (griddepcontrol.wait) before touching x, y or the scales, which the
                          previous kernel may therefore produce */

#define WW_MAX_BATCH 16

/* One widely-linear layer (complex n x m).  Fields are fixed-width for a stable ABI. */
typedef struct {
    int64_t n;          /* complex output rows, >= 1 */
    int64_t m;          /* complex input columns, >= 1 */
    int32_t layout;     /* ww_layout of the packed weights (GPU: WW_LAYOUT_COL4) */
    int32_t scale_mode; /* ww_scale_mode */
    int32_t conv;       /* ww_convention */
    uint32_t flags;     /* WW_FLAG_* */
} ww_layer;

/* Bytes of packed weights for an n x m layer in WW_LAYOUT_PLANAR or WW_LAYOUT_COL4:
 * 16 * n * ceil(m/16). */
size_t ww_packed_bytes(int64_t n, int64_t m);
/* Bytes of packed weights in any layout (WW_LAYOUT_TILE32: ceil(n/32) * ceil(m/64) * 2048;
 * WW_LAYOUT_LUT81: n * ceil(m/512) * 512);
 * 0 for an unknown layout or negative sizes. */
size_t ww_packed_bytes_layout(int64_t n, int64_t m, int32_t layout);

/* Host packer (App. H).  u_re..w_im: dense int8 n x m planes, row stride ld
 * (>= m) elements; values must be in {-1,0,+1} (else WW_ERR_INVALID_CODE, nothing
 * promised about `out`).  out: ww_packed_bytes_layout(n,m,layout) bytes, caller-owned host
 * memory.  Every layout (PLANAR, COL4, TILE32) is accepted by the three host functions. */
ww_status ww_pack_ternary(const int8_t* u_re, const int8_t* u_im, const int8_t* w_re,
                          const int8_t* w_im, int64_t n, int64_t m, int64_t ld, int32_t layout,
                          uint32_t* out);

/* Host unpacker (inverse).  Rejects slot (1,1) with WW_ERR_INVALID_ENCODING. */
ww_status ww_unpack_ternary(const uint32_t* packed, int64_t n, int64_t m, int32_t layout,
                            int8_t* u_re, int8_t* u_im, int8_t* w_re, int8_t* w_im, int64_t ld);

/* Host re-layout between any two layouts (src and dst distinct; sizes per layout). */
ww_status ww_repack(const uint32_t* src, int32_t src_layout, int64_t n, int64_t m,
                    uint32_t* dst, int32_t dst_layout);

/* Device packer: dense int8 planes on the GPU -> WW_LAYOUT_COL4 on the GPU.
 * planes_d: 4 planes (U_re, U_im, W_re, W_im) of n x ld int8 back to back (plane p at
 * planes_d + p*n*ld).  out_d: ww_packed_bytes(n,m) bytes, 16-B aligned.  bad_d (may be
 * NULL): device int32 set to 1 if any value is outside {-1,0,+1} (that column then packs
 * as zero); it is never cleared by the library.  Asynchronous on `stream`. */
ww_status ww_pack_ternary_device(const int8_t* planes_d, int64_t n, int64_t m, int64_t ld,
                                 uint32_t* out_d, int32_t* bad_d, void* stream);
/* The same device packer for any GPU layout: WW_LAYOUT_COL4 (== ww_pack_ternary_device) or
 * WW_LAYOUT_TILE32 (out_d: ww_packed_bytes_layout(n,m,WW_LAYOUT_TILE32) bytes, 16-B aligned;
 * an invalid value packs its 16-column word of that plane as zero and sets *bad_d) or
 * WW_LAYOUT_LUT81 (out_d: ww_packed_bytes_layout(n,m,WW_LAYOUT_LUT81) bytes, 16-B aligned; an
 * invalid value packs as the zero code and sets *bad_d). */
ww_status ww_pack_ternary_device_layout(const int8_t* planes_d, int64_t n, int64_t m, int64_t ld,
                                        int32_t layout, uint32_t* out_d, int32_t* bad_d,
                                        void* stream);

/* Fused WL-GEMV, one vector (B = 1).  packed_d: WW_LAYOUT_COL4, 16-B aligned;
 * scales_d: per row n x 4 or per tensor 4 fp32; x_d: m complex64; y_d: n complex64
 * (x and y must not alias).  Asynchronous on `stream`. */
ww_status ww_wl_gemv(const ww_layer* L, const void* packed_d, const float* scales_d,
                     const float* x_d, float* y_d, void* stream);

/* Batched small-B variant, 1 <= B <= WW_MAX_BATCH: X_d is B rows of m complex64 with row
 * stride ldx (complex elements, >= m); Y_d is B rows of n complex64 with stride ldy
 * (>= n).  Every decoded code drives all the vectors of a launch (one pass over the
 * weights per launch); B > 4 runs as groups of 4 vectors, one launch each (the last group
 * may overlap the previous one), so ww_query_launch(L, B > 4) describes one group. */
ww_status ww_wl_gemv_batched(const ww_layer* L, const void* packed_d, const float* scales_d,
                             const float* X_d, int64_t ldx, float* Y_d, int64_t ldy, int32_t B,
                             void* stream);

/* Row sharding over `world` GPUs: the row-range parallelism of the paper's kernel
 * (contiguous per-thread row ranges) lifted to GPUs, and SPEC's partition_rows
 * (disjoint contiguous ranges covering all rows).  Errors: world < 1, rank not in
 * [0, world), n < 1 or m < 1 -> WW_ERR_INVALID_ARGUMENT (out untouched).  Pure host function.
 * Ceil blocks so an all-gather has equal counts:
 * rows_per_rank = ceil(n/world), n_padded = world*rows_per_rank, rank r owns rows
 * [r*rpr, min((r+1)*rpr, n)) (possibly empty).  Its COL4/PLANAR-row weights are the
 * contiguous byte range [packed_offset_bytes, +packed_bytes) of a COL4 buffer, its
 * per-row scales the floats [scale_offset_floats, +scale_count), and its outputs go to
 * complex offset y_offset_complex of the gathered vector (B = 1; for B > 1 the gathered
 * buffer is rank-major [world][B][rows_per_rank]). */
typedef struct {
    int32_t world, rank;
    int64_t n, rows_per_rank, n_padded, row_begin, row_end;
    int64_t packed_offset_bytes, packed_bytes, scale_offset_floats, scale_count,
        y_offset_complex;
} ww_shard;
ww_status ww_shard_plan(int64_t n, int64_t m, int32_t world, int32_t rank, ww_shard* out);

/* Launch configuration the GPU entry points use for (L, B): grid (one CTA per SM, each
 * owning a contiguous row range), block, dynamic shared memory, the number of x column
 * tiles and their width (16-column chunks), the SM count it was planned for, the parts
 * of a row and the path (0 = single x tile; 1 = column tiles with row waves, taken when x
 * or the CTA's row totals do not fit shared memory).  parts = 1: a row is one warp's work
 * unit, swept 32 chunks at a time (split_chunks = W = ceil(m/16)).  parts = 2 (B = 1, path
 * 0, J = ceil(W/32) >= 2, chosen when it shortens the busiest SM sub-partition's share by
 * >= 4 %): rows are cut after split_chunks = 32 ceil(J/2) chunks into halves dealt out to
 * the warps like rows, and a first half's lane accumulators are handed through shared
 * memory to the warp that sweeps the second half, so the row is still accumulated in
 * whole-row order (same bits).  A row's accumulation order is a function of (m, B) only,
 * so results never depend on n, the shard, the grid or the parts.  Pure host function
 * (the SM count comes from the current device, 148 without one). */
typedef struct {
    int32_t grid, block, smem_bytes, tiles, tile_chunks, num_sms, parts, split_chunks, path;
} ww_launch_info;
ww_status ww_query_launch(const ww_layer* L, int32_t B, ww_launch_info* out);

/* Unfused ablation (not the product path): the paper's unfused baseline
 * -- eight real ternary GEMVs per widely-linear layer, one per
 * (plane, component of x), each re-streaming its plane, then one combine.
 * ww_ternary_gemv_plane: acc_d[i] = sum_j t_ij * x_j.comp for plane `plane` (0..3 = U_re,
 * U_im, W_re, W_im) of a WW_LAYOUT_PLANAR buffer (4-B aligned) and component `comp` (0 = re,
 * 1 = im) of the complex64 vector x_d; acc_d: n fp32.  flags: WW_FLAG_PDL.
 * ww_wl_combine: y (complex64, n) from acc8_d = 8 x n fp32 partial sums ordered
 * [U_re.re, U_re.im, U_im.re, U_im.im, W_re.re, W_re.im, W_im.re, W_im.im], the layer's
 * scales and convention, scales applied once per row.  Both asynchronous on
 * `stream`; argument errors before any launch. */
ww_status ww_ternary_gemv_plane(int64_t n, int64_t m, const void* planar_d, int32_t plane,
                                const float* x_d, int32_t comp, float* acc_d, uint32_t flags,
                                void* stream);
ww_status ww_wl_combine(const ww_layer* L, const float* acc8_d, const float* scales_d, float* y_d,
                        void* stream);

/* ------------------------------------------------------------------------------------
 * Persistent stage-chained program (DESIGN.md §6 "program kernel"): one cooperative launch
 * runs `nstages` widely-linear layers (B = 1) in order, e.g. one decode step of the
 * config-4 stack.  Stage s may read what stage s-1 wrote (wait = 1): the dependency is a
 * readiness counter per rank instead of a kernel boundary (the fork/join removal of P:1022-
 * 1026 applied across layers), while every CTA's producer warp keeps streaming the next
 * stages' packed weights into shared memory.  Output rows are stored straight into the
 * gathered output of every rank (`y[g]`, peer-mapped device pointers at world > 1): the
 * all-gather of the row-sharded layer is fused into the GEMV
 * epilogue.  Fused ops for the decode block:
 *   prologue WW_PRO_RMSNORM: x <- x * gamma / sqrt(mean(x^2) + eps) over the real 2m-vector
 *     (re, im interleaved, gamma = 2m fp32), WW_PRO_MUL: x <- x (.) x2 (re*re, im*im);
 *   epilogue WW_EPI_RESIDUAL: y_i += residual_i, WW_EPI_SILU: rows i < silu_rows get
 *     (silu(re), silu(im)), silu(v) = v / (1 + exp(-v)).
 * Requirements: 16 | m, x / x2 / packed / scales 16-B aligned, y / residual 8-B aligned,
 * world <= WW_PROG_MAX_RANKS, the stage's x of at most WW_PROG_MAX_M columns.  Outputs of
 * a stage are its gathered rows [row0, row0 + n_local) in every y[g] (g < world).
 * `ranks_in_launch` > 1 runs several ranks' shards in ONE launch on one GPU (CTAs split
 * evenly between them; used to test the multi-rank protocol without several GPUs).
 * ------------------------------------------------------------------------------------ */
#define WW_PROG_MAX_RANKS 8
#define WW_PROG_MAX_M 11264 /* 22 x 512 columns: x (and x2) of a stage in shared memory */
#define WW_PRO_NONE 0
#define WW_PRO_RMSNORM 1
#define WW_PRO_MUL 2
#define WW_EPI_NONE 0
#define WW_EPI_RESIDUAL 1
#define WW_EPI_SILU 2

/* Per-stage kernel with the same fused decode-block ops (B = 1, x of one shared-memory tile,
 * 16 | m, TMA staging): WW_PRO_* on the staged x before the sweep, WW_EPI_* on each output
 * row.  residual is indexed by row0 + local row (the global row of a row-sharded stage);
 * silu_rows compares against the same global index.  ops == NULL is ww_wl_gemv.  Errors:
 * WW_ERR_MISALIGNED (16-B x / x2 / gamma, 8-B residual / y), WW_ERR_UNSUPPORTED (x and x2
 * beyond shared memory), WW_ERR_INVALID_ARGUMENT (missing operand, x / y overlap). */
typedef struct {
    int32_t prologue, epilogue; /* WW_PRO_*, WW_EPI_* */
    const float* x2;            /* WW_PRO_MUL: second complex64[m] operand */
    const float* gamma;         /* WW_PRO_RMSNORM: 2m fp32 */
    float eps;
    const float* residual;      /* WW_EPI_RESIDUAL: complex64 by global row */
    int64_t row0;               /* global index of local row 0 */
    int64_t silu_rows;          /* WW_EPI_SILU: global rows below get SiLU */
} ww_ops;
ww_status ww_wl_gemv_fused(const ww_layer* L, const void* packed_d, const float* scales_d,
                           const float* x_d, float* y_d, const ww_ops* ops, void* stream);

typedef struct {
    const void* packed;   /* this rank's WW_LAYOUT_COL4 rows [row0, row0 + n_local) */
    const float* scales;  /* their scales: n_local x 4 (per row) or 4 (per tensor) */
    int64_t n_local;      /* rows this rank computes (>= 0) */
    int64_t row0;         /* global index of its first row */
    int64_t m;            /* complex input columns */
    int32_t scale_mode;   /* ww_scale_mode */
    int32_t conv;         /* ww_convention */
    const float* x;       /* complex64[m] input on this rank */
    const float* x2;      /* WW_PRO_MUL: second complex64[m] operand, else NULL */
    float* y[WW_PROG_MAX_RANKS]; /* complex64 gathered output on rank g (g < world) */
    const float* residual;       /* WW_EPI_RESIDUAL: complex64 indexed by global row */
    const float* gamma;          /* WW_PRO_RMSNORM: 2m fp32 */
    float eps;                   /* WW_PRO_RMSNORM */
    int32_t prologue;            /* WW_PRO_* */
    int32_t epilogue;            /* WW_EPI_* */
    int32_t wait;                /* 1: x depends on earlier stages of the program */
    int64_t silu_rows;           /* WW_EPI_SILU: global rows below this get SiLU */
} ww_stage;

/* Host-side handle filled by ww_program_init (caller-owned POD; keep it with the
 * workspace).  Launch geometry: grid = ranks_in_launch x ctas_per_rank CTAs of `block`
 * threads (16 consumer warps + 1 producer warp), `smem_bytes` of shared memory, a weight
 * ring of `nslot` slots of `slot_bytes`. */
typedef struct {
    int32_t nstages, world, rank_base, ranks_in_launch;
    int32_t grid, block, smem_bytes, ctas_per_rank, nslot, slot_bytes, x_bytes, has_mul;
    void* workspace;                         /* device descriptors (caller-allocated) */
    uint32_t* sync[WW_PROG_MAX_RANKS];       /* device sync words of every rank */
} ww_program;

/* Device workspace bytes for nstages x ranks_in_launch stage descriptors (128-B aligned). */
size_t ww_program_workspace_bytes(int32_t nstages, int32_t ranks_in_launch);
/* Bytes of one rank's sync words; caller-allocated, 128-B aligned, ZERO-initialised once
 * (at world > 1 in memory every rank can reach: sync_d[g] is rank g's block as seen here). */
size_t ww_program_sync_bytes(void);
/* Validate the stages (stages[r * nstages + s] = stage s of rank rank_base + r), encode the
 * TMA maps and copy the descriptors into workspace_d (synchronous).  Errors before any
 * device work: WW_ERR_INVALID_ARGUMENT / WW_ERR_MISALIGNED / WW_ERR_UNSUPPORTED. */
ww_status ww_program_init(const ww_stage* stages, int32_t nstages, int32_t world,
                          int32_t rank_base, int32_t ranks_in_launch, uint32_t* const* sync_d,
                          void* workspace_d, ww_program* out);
/* Launch the program (asynchronous on `stream`; cooperative launch, all CTAs co-resident).
 * Every rank must launch the same program the same number of times. */
ww_status ww_program_run(const ww_program* prog, void* stream);

/* Batched WL-GEMV on the tensor cores (tcgen05.mma kind::i8) for the small-batch variant
 * (BASELINE config 5): with B vectors the layer is a dense contraction of the stacked ternary
 * planes (4n x m; L->layout must be WW_LAYOUT_TILE32, whose App. H words are decoded in-kernel
 * to int8 in shared memory by a byte-permute table) with the B x 2 real
 * components of x, each split into three signed 8-bit limbs of a 22-bit fixed-point value
 * (scale 2^-E per vector and component, E from max |x|); int32 accumulation is exact, the
 * limbs are recombined in fp64 and the scales applied once per row (Eq. 1 /
 * Eqs. 2-3).  Error: x's 22-bit grid relative to max |x| of its vector and component.
 * X: B rows of m complex64 (stride ldx), Y: B rows of n complex64 (stride ldy); 1 <= B <= 16,
 * m <= 11264 (each x component is staged in shared memory to split it).  A layer with fewer
 * 32-row tiles than SMs splits each tile's K range over up to 4 CTAs of one thread-block
 * cluster whose exact int32 partial sums meet in the first CTA's shared memory (DSMEM);
 * results do not depend on the split.
 * workspace_d: ww_tc_workspace_bytes(n, m, B) bytes, 128-B aligned, caller-owned (limbs and
 * exponents, rewritten every call).  Two launches on `stream` (limbs, then the MMA kernel). */
size_t ww_tc_workspace_bytes(int64_t n, int64_t m, int32_t B);
ww_status ww_wl_gemv_batched_tc(const ww_layer* L, const void* packed_d, const float* scales_d,
                                const float* X_d, int64_t ldx, float* Y_d, int64_t ldy, int32_t B,
                                void* workspace_d, void* stream);

/* WL-GEMV on the tensor cores with the ternary operand decoded into tensor memory (B = 1..4;
 * DESIGN.md §6 "wl_tcv_kernel").  The eight real sub-GEMVs of Eq. 1 (Eqs. 6-7,
 * P:931-946) are one exact integer contraction per 32-row tile: the App. H words
 * (WW_LAYOUT_TILE32, read once from HBM) are expanded in-kernel to int8 {-1, 0, +1} in tensor
 * memory, each real component of x is an offset 22-bit fixed-point value 2^22 + rint(x 2^E)
 * (E = 20 - ilogb(max |x|) per vector and component) split into three unsigned bytes, and
 * tcgen05.mma kind::i8 accumulates in int32 (exact); the scales are applied once per row
 * after accumulation with the EQ1 / ALG1 signs.  Error: x's grid 2^-E (about
 * max|x| 2^-21) and the final fp64 -> fp32 rounding; results are bitwise independent of the
 * grid and of the row shard.  x must be finite.
 * L->layout must be WW_LAYOUT_TILE32 (packed_d: ww_packed_bytes_layout(n, m, TILE32) bytes,
 * 16-B aligned); X: B rows of m complex64 (stride ldx >= m, 8-B aligned), Y: B rows of n
 * complex64 (stride ldy >= n); x and y must not overlap.  WW_FLAG_PDL as for ww_wl_gemv (the
 * weights are read before griddepcontrol.wait, x / scales / y / workspace after it).
 * workspace_d: ww_tcv_workspace_bytes(n, m, B) bytes, 16-B aligned, caller-owned, ZEROED
 * before its first use; every call leaves it zeroed again (split tiles reduce their int32
 * partial sums there), so launches sharing one workspace must be stream-ordered.
 * Errors: WW_ERR_UNSUPPORTED (layout, B > 4, x's slabs beyond shared memory), the usual
 * argument / alignment errors before any launch.  One launch on `stream`. */
size_t ww_tcv_workspace_bytes(int64_t n, int64_t m, int32_t B);
ww_status ww_wl_gemv_tc(const ww_layer* L, const void* packed_d, const float* scales_d, const float* X_d,
                        int64_t ldx, float* Y_d, int64_t ldy, int32_t B, void* workspace_d, void* stream);

/* WL-GEMV by ternary subset-sum lookup (B = 1; DESIGN.md §6 "wl_lut_kernel").  Eq. 1
 * (Eqs. 6-7) with every group of 4 codes of a plane taken as one
 * table entry: per launch each CTA builds, with adds and subtracts only (a code
 * selects +x, -x or nothing), the 81 sums sum_k c_k x_k, c in {-1,0,+1}^4, of each group of
 * 4 columns of x in shared memory; a weight byte (WW_LAYOUT_LUT81) indexes it.  The scales
 * are applied once per row after accumulation, EQ1 / ALG1 signs as ww_wl_gemv.
 * Columns are split over the CTAs of a thread-block cluster (1024 columns each) whose
 * per-row totals are summed in rank order through distributed shared memory: results are
 * deterministic and independent of the row shard.  Rounding order differs from ww_wl_gemv
 * (groups of 4 are summed first), same error bound.
 * packed_d: ww_lut81_packed_bytes(n, m) bytes, 16-B aligned; x_d: m complex64, y_d: n
 * complex64 (8-B aligned, must not overlap); scales as ww_wl_gemv.  WW_FLAG_PDL: the first
 * weight loads are issued before griddepcontrol.wait, x / scales / y touched after it.
 * Errors: WW_ERR_UNSUPPORTED (layout; m > 8192: cluster of more than 8 CTAs; more than 1536
 * rows per cluster), argument / alignment errors before any launch.  One launch on `stream`.
 * ww_lut81_from_planar / ww_lut81_to_planar: host conversion from / to the App. H planes
 * (WW_LAYOUT_PLANAR); WW_ERR_INVALID_ENCODING on a (1,1) slot, a byte > 80 or a nonzero
 * padding code (nothing defined is written past that point). */
size_t ww_lut81_packed_bytes(int64_t n, int64_t m);
ww_status ww_lut81_from_planar(int64_t n, int64_t m, const void* planar, void* out);
ww_status ww_lut81_to_planar(int64_t n, int64_t m, const void* lut, void* planar_out);
ww_status ww_wl_gemv_lut(const ww_layer* L, const void* packed_d, const float* scales_d,
                         const float* x_d, float* y_d, void* stream);

/* Keep [ptr, ptr + bytes) persisting in L2 for kernels launched on `stream` (and kernel nodes
 * captured from it): access-policy window, hit ratio 1, streaming misses; reserves up to
 * `bytes` of persisting L2 (device maximum).  For activations every CTA re-reads while the
 * packed weights stream past.  bytes == 0 clears the window.  WW_ERR_UNSUPPORTED without
 * persisting L2, WW_ERR_CUDA if the runtime refuses. */
ww_status ww_stream_keep_in_l2(void* stream, const void* ptr, size_t bytes);

const char* ww_status_string(ww_status s);
const char* ww_last_error(void); /* thread-local message of the last failing call */
int32_t ww_version(void);

#ifdef __cplusplus
}
#endif
#endif
