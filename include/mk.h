/*
 * mk.h — C ABI of the B200-native generalized sparse convolution library (libmk.so).
 *
 * Implements the data-parallel hot path of Choy, Gwak, Savarese, "4D Spatio-Temporal
 * ConvNets: Minkowski Convolutional Neural Networks" (arXiv 1904.08755).  Citations:
 * "P:n" = line n of the paper's text, "S:n" = line n of SPEC.md, "Rk" = the
 * reading k of an ambiguous passage, listed in DESIGN.md §3.
 *
 * Conventions shared by every call
 *  - Plain C types only.  Device pointers are prefixed d_, host pointers h_.  A stream is
 *    a cudaStream_t passed as void* (NULL = legacy default stream).  All device work is
 *    enqueued on that stream; the caller owns ordering with other streams.
 *  - Coordinates are int32 rows [n][D+1]: D spatial components, then the batch index
 *    (Eq. 1).  D is 1..7 on this implementation.  Batch indices are >= 0.
 *    A row is packed into one 128-bit key (reading R19): D <= 3 any int32 components;
 *    D = 4: t in [-2^15, 2^15), batch <= 65534; D = 5..7 (e.g. the 7D space-time-chroma
 *    lattice of the TS-CRF): axes 0-2 in [-2^19, 2^19), axes 3-5 in
 *    [-2^11, 2^11), axis 6 in [-2^15, 2^15), batch <= 65534 for D = 7.  Rows outside
 *    these ranges are COORD_RANGE errors.
 *  - Features are row-major [n][C] (row i = f_i^T, Eq. 1).  Weights are [K][C_out][C_in]
 *    row-major: the K matrices W_i of size N_out x N_in (R17).
 *  - Handles (mk_coords, mk_kmap) are immutable once created ("build then freeze",
 *    S:113/S:173): any number of streams may read them concurrently.  They own their
 *    device memory and release it (stream-ordered, on the stream they were created on)
 *    in *_destroy.  Feature/weight/gradient buffers are caller-owned; outputs are
 *    overwritten, never accumulated into.
 *  - Calls that must report a size (coords_quantize / create / stride / expand) wait once
 *    on the host until the size is known: the last block of the ranking kernel posts it into
 *    a host-mapped mailbox, so the call returns while the tail of that kernel may still run
 *    (all later work is ordered on the stream; the call does not drain it).  mk_kmap_build is asynchronous: the pair count is read back lazily, the
 *    first time mk_kmap_info is asked for n_pairs (or a call needs it: export, weight
 *    gradient), by waiting for the build's completion event only.  Every other call is
 *    asynchronous.
 *  - Every call returns mk_status.  On failure mk_last_error_message() (thread-local)
 *    describes it and mk_last_error_row() gives the first offending input row, or -1.
 *    No C++ exception crosses this boundary.  On failure no handle is returned and
 *    caller buffers may have been partially written.
 */
#ifndef MK_H
#define MK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MK_MAX_DIM 7        /* dimensions supported on the GPU path (D <= 7; see R19 for the
                               component ranges of D = 4 and D = 5..7 packed keys) */
#define MK_MAX_REGION 8     /* entries of mk_region.size / .dilation */

typedef enum {
  MK_OK = 0,
  MK_ERR_INVALID_ARGUMENT = 1,   /* null pointer, bad size, negative batch index, ...  */
  MK_ERR_DIMENSION_MISMATCH = 2, /* coordinate sets / regions of different D    */
  MK_ERR_SHAPE_MISMATCH = 3,     /* channel counts inconsistent with the map    */
  MK_ERR_NONFINITE_INPUT = 4,    /* NaN / Inf point coordinate                   */
  MK_ERR_COORD_RANGE = 5,        /* coordinate outside the representable domain (R19)   */
  MK_ERR_STRIDE = 6,             /* coordinate not a multiple of the tensor stride*/
  MK_ERR_UNSUPPORTED = 7,        /* D > 7, channels > 256, bf16 channels % 16 != 0, ... */
  MK_ERR_OUT_OF_MEMORY = 8,
  MK_ERR_CUDA = 9                /* a CUDA runtime error; message carries its text      */
} mk_status;

typedef enum { MK_F32 = 0, MK_BF16 = 1 } mk_dtype;

/* Kernel shapes N^D (P:154 hypercube V^D(K); Fig. 3 P:250-282 cross / hypercross / hybrid). */
typedef enum { MK_HYPERCUBE = 0, MK_HYPERCROSS = 1, MK_HYBRID = 2, MK_CUSTOM = 3 } mk_region_type;

/* A kernel region.  Per-axis index range R(K) = {-(K-1)/2 .. (K-1)/2} for odd K
 * (V^1(3) = {-1,0,1}) and {0 .. K-1} for even K (R3); each component is scaled by
 * dilation[d] ("dilated convolution").  Built-in shapes are enumerated in
 * lexicographic order, axis 0 most significant (R2):
 *   HYPERCUBE  = prod_d R(size[d])
 *   HYPERCROSS = {0} U { i e_d : i in R(size[d]) \ {0} }
 *   HYBRID     = (cube over the spatial axes at temporal offset 0) U
 *                { i e_t : i in R(size[t]) \ {0} },  t = temporal_axis (R4)
 *   CUSTOM     = offsets[n_offsets][D] (host), distinct, caller's order, taken literally.
 * dilation entries of 0 are read as 1; temporal_axis < 0 means D-1. */
typedef struct {
  int32_t type;                    /* mk_region_type */
  int32_t D;
  int32_t size[MK_MAX_REGION];
  int32_t dilation[MK_MAX_REGION];
  int32_t temporal_axis;
  const int32_t* offsets;          /* CUSTOM only: host [n_offsets][D] */
  int32_t n_offsets;
} mk_region;

typedef struct mk_context mk_context;
typedef struct mk_coords mk_coords;
typedef struct mk_kmap mk_kmap;

/* Optional device allocator (e.g. a framework caching allocator).  NULL callbacks select
 * cudaMallocAsync / cudaFreeAsync on the call's stream. */
typedef void* (*mk_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*mk_free_fn)(void* ptr, void* stream, void* user);

/* ---------------------------------------------------------------- context ---------- */
/* Binds the library to a CUDA device.  Fails with MK_ERR_UNSUPPORTED on devices older
 * than sm_100 (the kernels are compiled for sm_100a only).  With the default allocator (NULL
 * callbacks) it sets the device's default stream-ordered pool to keep freed memory and
 * reserves 8 GB in it once (MK_POOL_RESERVE_MB overrides, 0 disables), so a call never
 * maps new pool memory in steady state.  The context keeps one grow-only scratch buffer
 * (weight-gradient partial sums); it is freed by mk_context_destroy. */
mk_status mk_context_create(int device, mk_alloc_fn alloc, mk_free_fn free_fn, void* user,
                            mk_context** out);
void mk_context_destroy(mk_context* ctx);

/* ---------------------------------------------------------------- coordinates ------ */
/* Sparse tensor quantization, Alg. 1: C' = floor(C_p / v) per axis, computed
 * as IEEE fp32 division then floor (R6), unique by exact key (R5), rows numbered in
 * first-occurrence order of the input points (R8); the first point of each voxel is its
 * representative (R9: i_x of the reduction f).
 *   d_points      device float32 [n][D]          point coordinates
 *   d_batch       device int32 [n] or NULL (all 0) batch index per point, >= 0
 *   voxel         quantization step v_l > 0
 *   d_point_to_row  device int32 [n] or NULL: row of each point's voxel
 *   d_first_point   device int32 [n] (capacity n) or NULL: first point of each row
 * Errors: NONFINITE_INPUT / COORD_RANGE / INVALID_ARGUMENT (negative batch) with the first
 * offending point row; for D >= 4 COORD_RANGE also flags components or a batch index
 * outside the packed-key ranges above (R19).  n = 0 is valid and yields an empty set. */
mk_status mk_coords_quantize(mk_context* ctx, const float* d_points, const int32_t* d_batch,
                             int64_t n, int32_t D, float voxel, void* stream, mk_coords** out,
                             int32_t* d_point_to_row, int32_t* d_first_point);

/* mk_coords_quantize without the wait for the row count: returns the handle as soon as the
 * kernels are enqueued.  The count (and any input error: NONFINITE_INPUT, COORD_RANGE, ...)
 * is collected at its first use — mk_coords_info(n), export, stride / expand, or a
 * kernel-map build on the handle — which then waits for it (the ranking kernel posts it to a
 * host-mapped mailbox).  d_first_point needs room for n rows (only the first N are written).
 * Lets the host prepare the next call (e.g. mk_kmap_build) while the GPU quantizes. */
mk_status mk_coords_quantize_deferred(mk_context* ctx, const float* d_points, const int32_t* d_batch,
                                      int64_t n, int32_t D, float voxel, void* stream, mk_coords** out,
                                      int32_t* d_point_to_row, int32_t* d_first_point);

/* A coordinate set from integer rows (Eq. 1), duplicates merged, first occurrence wins.
 *   d_coords        device int32 [n][D+1], batch last
 *   h_tensor_stride host int32 [D] or NULL (all 1): every spatial component must be a
 *                   multiple of it ("minimum distance between coordinates")
 *   d_inverse       device int32 [n] or NULL: row of each input row
 * Errors: STRIDE, INVALID_ARGUMENT (negative batch), COORD_RANGE (D >= 4 packing) with
 * the first offending row. */
mk_status mk_coords_create(mk_context* ctx, const int32_t* d_coords, int64_t n, int32_t D,
                           const int32_t* h_tensor_stride, void* stream, mk_coords** out,
                           int32_t* d_inverse);

/* Size, dimension and per-axis tensor stride (h_tensor_stride host [D], may be NULL). */
mk_status mk_coords_info(const mk_coords* c, int64_t* n, int32_t* D, int32_t* h_tensor_stride);

/* Copies the rows to d_out (device int32 [n][D+1]). */
mk_status mk_coords_export(const mk_coords* c, int32_t* d_out, void* stream);

/* Label reduction of Alg. 1: d_row_labels[r] = the label shared by
 * every point of voxel r, or ignore_label when its points carry two or more distinct
 * labels (the reduction f of P:181; R10: ignore_label is the caller's IGNORE_LABEL).
 * d_point_to_row [n_points] and d_first_point [n_rows] are the outputs of
 * mk_coords_quantize; d_labels device int32 [n_points]; d_row_labels device int32 [n_rows]
 * (written).  Deterministic (no order-dependent step).  Asynchronous. */
mk_status mk_coords_labels(const int32_t* d_point_to_row, const int32_t* d_first_point,
                           const int32_t* d_labels, int64_t n_points, int64_t n_rows,
                           int32_t ignore_label, int32_t* d_row_labels, void* stream);

/* Exact membership: d_rows[i] = row of d_queries[i] ([q][D+1]) or -1. */
mk_status mk_coords_lookup(const mk_coords* c, const int32_t* d_queries, int64_t q,
                           int32_t* d_rows, void* stream);

/* Output coordinates of a strided convolution (rule R11 from S:84):
 * s_out = s_in * conv_stride per axis; rows u' = floor_div(u, s_out) * s_out (floor toward
 * -inf, R7), batch unchanged, first occurrence in input row order. h_conv_stride host [D]. */
mk_status mk_coords_stride(mk_context* ctx, const mk_coords* in, const int32_t* h_conv_stride,
                           void* stream, mk_coords** out);

/* Output coordinates of a generative transposed convolution (a transposed conv may
 * produce "arbitrary output coordinates"): the union over rows u of `in`
 * and offsets i of `region` of u + i * s_out, batch unchanged (R18), rows in first
 * occurrence of (row, offset) order.  h_out_stride host [D] (NULL = in's tensor stride)
 * must divide in's tensor stride (MK_ERR_STRIDE); it is the new set's tensor stride.
 * Typical use: upsampling a stride-2s set to stride s with the region {0,1}^D, then
 * mk_kmap_build(in, out, region, transposed = 1).  Waits once for the row count. */
mk_status mk_coords_expand(mk_context* ctx, const mk_coords* in, const mk_region* region,
                           const int32_t* h_out_stride, void* stream, mk_coords** out);

void mk_coords_destroy(mk_coords* c);

/* ---------------------------------------------------------------- kernel region ---- */
/* Enumerates N^D.  *K receives the count; h_offsets (host int32 [K][D]) may be NULL. */
mk_status mk_region_offsets(const mk_region* region, int32_t* K, int32_t* h_offsets);

/* ---------------------------------------------------------------- kernel map ------- */
/* Kernel map M = {(I_i, O_i)}_i for the generalized sparse convolution Eq. 3
 * (P:155-159): for every output u in C_out and offset i in N^D, the pair (row of u + i*s,
 * row of u) when u + i*s is in C_in; s = the input tensor stride (R14).  With transposed
 * != 0 the roles of input and output are reversed (R13): pairs (row of v - i*s,
 * row of v) for v in C_out with s = the OUTPUT (fine) tensor stride — the map of the
 * transposed convolution from a coarse set back to a fine one.  Batch indices are never
 * offset (R18).  Within each offset pairs are sorted by output row.  Requires
 * in and out of equal D (DIMENSION_MISMATCH) and region->D == D. */
mk_status mk_kmap_build(mk_context* ctx, const mk_coords* in, const mk_coords* out,
                        const mk_region* region, int32_t transposed, void* stream,
                        mk_kmap** out_map);

/* K, |M|, N_in, N_out.  Any pointer may be NULL.  Requesting n_pairs waits (once per map)
 * for the build to complete on the device (event wait, not a stream sync). */
mk_status mk_kmap_info(const mk_kmap* m, int32_t* K, int64_t* n_pairs, int64_t* n_in,
                       int64_t* n_out);

/* CSR export: d_ptr device int64 [K+1], d_in / d_out device int32 [n_pairs]. */
mk_status mk_kmap_export(const mk_kmap* m, int64_t* d_ptr, int32_t* d_in, int32_t* d_out,
                         void* stream);

void mk_kmap_destroy(mk_kmap* m);

/* ---------------------------------------------------------------- pooling ---------- */
/* Pooling over a kernel map.  The inputs of output row o are
 * the pairs (a, o) of every offset, in concatenated order (offset k ascending).
 *   MK_POOL_MAX  Alg. 3: F_out[o][c] = max_a F_in[a][c]; d_argmax [n_out][C] (device int32,
 *                written when non-NULL) = the first maximal input row (ties: lowest
 *                concatenated index), needed by the reverse mode.
 *   MK_POOL_AVG  Alg. 4: the mean over the inputs (F' / N).
 *   MK_POOL_SUM  Alg. 4 without the division ("sum pooling").
 * Features [n][C] row-major, fp32 or bf16 (computed in fp32; bf16 outputs rounded RNE).
 * Output rows with no input are 0 (argmax -1) — reading R23.  Strided pooling uses a map from
 * a set to its strided set (mk_coords_stride); unpooling uses a transposed map.
 * Asynchronous; deterministic (fixed reduction order, no atomics). */
typedef enum { MK_POOL_MAX = 0, MK_POOL_AVG = 1, MK_POOL_SUM = 2 } mk_pool_mode;

mk_status mk_pool_forward(mk_context* ctx, const mk_kmap* m, int32_t mode, const void* d_fin,
                          int32_t C, mk_dtype dt, void* d_fout, int32_t* d_argmax, void* stream);

/* Reverse mode: G_in[a] = sum over the outputs o of a (offset order) of G_out[o] (SUM),
 * G_out[o] / N_o (AVG), or G_out[o][c] where argmax[o][c] == a (MAX; d_argmax from the
 * forward call).  d_gin [n_in][C] is overwritten. */
mk_status mk_pool_backward(mk_context* ctx, const mk_kmap* m, int32_t mode, const void* d_gout,
                           int32_t C, mk_dtype dt, const int32_t* d_argmax, void* d_gin,
                           void* stream);

/* Global pooling (every input maps to the origin of its batch): d_fout [n_batch][C]
 * = sum (MK_POOL_SUM) or mean (MK_POOL_AVG) of the rows of `c` whose batch index is b; rows
 * with b >= n_batch are ignored; a batch without rows gives 0.  Deterministic (fixed-order
 * two-level reduction).  n_batch * C <= 51200.  Asynchronous. */
mk_status mk_global_pool(mk_context* ctx, const mk_coords* c, int32_t mode, const void* d_fin,
                         int32_t C, mk_dtype dt, int32_t n_batch, void* d_fout, void* stream);

/* ---------------------------------------------------------------- TS-CRF ----------- */
/* Mean-field inference of the trilateral stationary CRF (Alg. 5, Eq. 4) over a
 * map that connects a (typically 7D space-time-chroma, D = 7) coordinate set to itself
 * (e.g. mk_kmap_build(c, c, hypercross 3^7 = 15 offsets)):
 *   Q^0 = softmax(phi_u)  (R25);  for n = 1..n_iters:  Q^n = softmax(phi_u + conv(Q^(n-1); W))
 * d_phi_u device fp32 [n][C] unary logits; d_W device fp32 [K][C][C] the pairwise kernel
 * phi_p per offset (same layout as conv weights); d_q device fp32 [n][C] receives Q^N.
 * fp32 throughout (exact-FFMA convolution).  Asynchronous. */
mk_status mk_crf_infer(mk_context* ctx, const mk_kmap* m, const float* d_phi_u, const float* d_W,
                       int32_t C, int32_t n_iters, float* d_q, void* stream);

/* Learning through the mean-field iterations (Eq. 5): given dL/dQ^N (d_gq,
 * device fp32 [n][C]) for the Q^N of mk_crf_infer(phi_u, W, n_iters), writes
 *   d_gphi  [n][C]    dL/dphi_u = sum over n = 0..N of (dL/dQ^n) dQ^n/dphi_u,
 *   d_gW    [K][C][C] dL/dphi_p = sum over n = 1..N of (dL/dQ^n) dQ^n/dphi_p
 * (backpropagation through time; not touched when n_iters = 0).  The forward is recomputed
 * with every Q^n kept: (n_iters + 4) n C + K C^2 floats of stream-ordered workspace.  fp32;
 * deterministic (the weight gradient uses the fixed-order split-K reduction).  Asynchronous. */
mk_status mk_crf_backward(mk_context* ctx, const mk_kmap* m, const float* d_phi_u, const float* d_W,
                          int32_t C, int32_t n_iters, const float* d_gq, float* d_gphi, float* d_gW,
                          void* stream);

/* ---------------------------------------------------------------- convolution ------ */
/* Generalized sparse convolution, Alg. 2:
 *   F_out[o] = sum over pairs (a, o) of offset k of W_k F_in[a];  rows without any pair
 *   are 0 ("F^o <- 0"; R15).  No bias (R16).
 *   d_fin   [n_in][c_in] of in_dt;  d_w [K][c_out][c_in] of in_dt;  d_fout [n_out][c_out]
 *   of out_dt.  Accumulation is fp32.  MK_BF16 inputs run on the tcgen05 tensor cores.
 *   MK_F32 inputs run on the same tensor cores as six bf16 convolutions of three-way bf16
 *   splits of the operands (x = x1 + x2 + x3; the dropped products are below 2^-24 relative,
 *   fp32-level accuracy) when c_in and c_out are multiples of 16 and no epilogue is fused;
 *   otherwise, or with the environment variable MK_F32_MODE=exact, exact fp32 FFMA kernels.
 *   Both are deterministic.  Channel contract: 1 <= c_in, c_out <= 256 for
 *   MK_F32; multiples of 16 in 16..256 for MK_BF16 (every such pair is planned: wide
 *   outputs are split over column slices, wide weight-gradient tiles use fewer, larger CTAs);
 *   anything else returns MK_ERR_UNSUPPORTED.
 * Works on any map; mk_conv_transpose_forward additionally requires a transposed map. */
mk_status mk_conv_forward(mk_context* ctx, const mk_kmap* m, const void* d_fin, int32_t c_in,
                          const void* d_w, void* d_fout, int32_t c_out, mk_dtype in_dt,
                          mk_dtype out_dt, void* stream);

/* mk_conv_forward with a fused row-wise epilogue ("functions that do not require
 * spatial information (coordinates) such as ReLU ... apply directly to the features F";
 * batch normalisation is 1D normalisation of the rows of F), for chaining MinkowskiNet /
 * MinkUNet blocks without extra passes over F (R26):
 *   F_out[o][j] = act(conv[o][j] * scale[j] + shift[j] + residual[o][j]),
 *   act = max(0, .) when relu != 0, identity otherwise.
 * d_scale, d_shift: device fp32 [c_out] — BatchNorm in its inference (folded) form,
 *   scale = gamma / sqrt(var + eps), shift = beta - mean * scale; NULL means 1 / 0.
 * d_residual: device [n_out][c_out] of out_dt (the block's skip input), NULL means 0.
 * Applied in fp32 to the fp32 accumulator before the output conversion; rows without
 * pairs get act(shift + residual).  Works on any map (also transposed maps, as the
 * transposed forward).  Asynchronous. */
mk_status mk_conv_forward_fused(mk_context* ctx, const mk_kmap* m, const void* d_fin, int32_t c_in,
                                const void* d_w, void* d_fout, int32_t c_out, mk_dtype in_dt,
                                mk_dtype out_dt, const float* d_scale, const float* d_shift,
                                const void* d_residual, int32_t relu, void* stream);

/* Reverse mode of mk_conv_forward (not in the paper, which covers forward only):
 *   d_gin[a]  = sum over pairs (a, o) of offset k of W_k^T G_out[o]       (NULL: skip)
 *   d_gw[k]   = sum over pairs (a, o) of offset k of G_out[o] F_in[a]^T   (NULL: skip),
 *               float32 [K][c_out][c_in], reduced in a fixed order (deterministic).
 * d_gout [n_out][c_out], d_fin [n_in][c_in], d_w [K][c_out][c_in] and d_gin are of dt. */
mk_status mk_conv_backward(mk_context* ctx, const mk_kmap* m, const void* d_gout,
                           const void* d_fin, const void* d_w, int32_t c_in, int32_t c_out,
                           mk_dtype dt, void* d_gin, float* d_gw, void* stream);

/* Transposed convolution: the same operations on a map built with transposed=1
 * (fails with INVALID_ARGUMENT otherwise).  W is the transposed conv's own weights
 * [K][c_out][c_in]; passing W_k^T of a forward conv gives its adjoint. */
mk_status mk_conv_transpose_forward(mk_context* ctx, const mk_kmap* m, const void* d_fin,
                                    int32_t c_in, const void* d_w, void* d_fout, int32_t c_out,
                                    mk_dtype in_dt, mk_dtype out_dt, void* stream);
mk_status mk_conv_transpose_backward(mk_context* ctx, const mk_kmap* m, const void* d_gout,
                                     const void* d_fin, const void* d_w, int32_t c_in,
                                     int32_t c_out, mk_dtype dt, void* d_gin, float* d_gw,
                                     void* stream);

/* ---------------------------------------------------------------- diagnostics ------ */
const char* mk_last_error_message(void);
int64_t mk_last_error_row(void);
/* Number of library kernels launched by this process so far (bench "gpu_launches"). */
int64_t mk_kernel_launch_count(void);
/* The stable radix sort the map builder uses to order rows by neighbour bitmask, exposed
 * for testing: d_perm (device int32 [n]) receives the permutation that sorts the low `bits`
 * (1..32) bits of d_keys (device uint32 [n], not modified) stably; ctx's cooperative
 * one-kernel path unless MK_SORT_COOP=0.  Asynchronous. */
mk_status mk_debug_sort_perm(mk_context* ctx, const uint32_t* d_keys, int64_t n, int32_t bits, int32_t* d_perm,
                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MK_H */
