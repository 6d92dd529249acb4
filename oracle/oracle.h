/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the generalized sparse
 * convolution hot path of Choy et al., "4D Spatio-Temporal ConvNets: Minkowski
 * Convolutional Neural Networks" (arXiv 1904.08755).  Citations "P:n" are lines of
 * /root/reference/PAPER.md; "S:n" lines of SPEC.md; "Rk" readings in DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or constant with the
 * CUDA path (paper_1904_08755_b200/), and never includes anything from it.
 *
 * Conventions: coordinates are int32 rows [n][D+1], spatial axes first, batch index
 * last (Eq. 1).  Features are fp64 row-major [n][C].  Weights are fp64
 * [K][C_out][C_in] (W in R^{K^D x N_out x N_in}).  Kernel maps are CSR per
 * offset: ptr[K+1] (int64), in[|M|], out[|M|] (int32), output-ascending inside each
 * offset.
 *
 * Every function returns an orc_status (0 = OK).  err_row receives the first
 * offending input row where one exists, else -1.
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_INVALID_ARGUMENT = 1,
  ORC_DIMENSION_MISMATCH = 2,
  ORC_SHAPE_MISMATCH = 3,
  ORC_NONFINITE_INPUT = 4,
  ORC_COORD_RANGE = 5,
  ORC_STRIDE = 6,
  ORC_UNSUPPORTED = 7
};

enum { ORC_HYPERCUBE = 0, ORC_HYPERCROSS = 1, ORC_HYBRID = 2, ORC_CUSTOM = 3 };

/* O1 — Alg. 1: C' = floor(C_p / v), unique by exact key, first point wins. */
int orc_quantize(const float* points, const int32_t* batch, int64_t n, int32_t D, float voxel,
                 int32_t* coords_out, int32_t* point_to_row, int32_t* first_point,
                 int64_t* n_out, int64_t* err_row);

/* O2 — create a coordinate set from integer rows (Eq. 1), first occurrence wins. */
int orc_create(const int32_t* coords, int64_t n, int32_t D, const int32_t* tensor_stride,
               int32_t* coords_out, int32_t* inverse, int64_t* n_out, int64_t* err_row);

/* O3 — output coordinates of a strided conv (reading R11). */
int orc_stride(const int32_t* coords, int64_t n, int32_t D, const int32_t* tensor_stride,
               const int32_t* conv_stride, int32_t* coords_out, int64_t* n_out, int64_t* err_row);

/* f4 — output coordinates of a generative transposed convolution ("arbitrary output
 * coordinates"): C_out = union over rows u of C_in and offsets i of
 * {u + i * scale}, batch unchanged, first occurrence in (row, offset) order; coords_out
 * holds up to n * K rows. */
int orc_expand(const int32_t* coords, int64_t n, int32_t D, const int32_t* offsets, int32_t K,
               const int32_t* scale, int32_t* coords_out, int64_t* n_out, int64_t* err_row);

/* O4 — kernel offset set N^D.  offsets may be NULL (count only). */
int orc_region(int32_t type, int32_t D, const int32_t* size, const int32_t* dilation,
               int32_t temporal_axis, const int32_t* custom, int32_t n_custom,
               int32_t* offsets, int32_t* K);

/* O1' — label reduction of Alg. 1: the labels of the points of a voxel are
 * folded in input order with f((l_x,i_x),(l_y,i_y)) = (l_x,i_x) if l_x == l_y else
 * (IGNORE, i_x).  point_to_row is O1's inverse map (rows 0..n_rows-1). */
int orc_labels(const int32_t* point_to_row, const int32_t* labels, int64_t n_points, int64_t n_rows,
               int32_t ignore_label, int32_t* row_labels);

/* Exact membership query: row of each query coordinate, -1 when absent. */
int orc_lookup(const int32_t* coords, int64_t n, int32_t D, const int32_t* queries, int64_t q,
               int32_t* rows);

/* O5 — kernel map (Eq. 3; transposed P:202).  Pair (a, o) at offset k
 * iff C_in[a] = C_out[o] + sign * offsets[k] * scale with sign = +1 (conv) / -1
 * (transposed), batch unchanged.  First call with ptr only (in/out NULL) to size. */
int orc_kmap(const int32_t* c_in, int64_t n_in, const int32_t* c_out, int64_t n_out, int32_t D,
             const int32_t* offsets, int32_t K, const int32_t* scale, int32_t transposed,
             int64_t* ptr, int32_t* in_idx, int32_t* out_idx);

/* O6 — Alg. 2, fp64. */
void orc_conv_forward(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                      const double* f_in, int32_t c_in, const double* W, double* f_out,
                      int64_t n_out, int32_t c_out);
/* O6 restricted to selected output rows (same definition, evaluated row by row). */
void orc_conv_forward_rows(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx,
                           int32_t K, const double* f_in, int32_t c_in, const double* W,
                           int32_t c_out, const int32_t* rows, int64_t n_rows, double* f_rows);
/* O7 — input gradient: G_in[I_k] += W_k^T G_out[O_k]. */
void orc_conv_dgrad(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                    const double* g_out, int32_t c_out, const double* W, double* g_in,
                    int64_t n_in, int32_t c_in);
/* O8 — weight gradient: dW_k = sum over pairs G_out[o] (x) F_in[a]. */
void orc_conv_wgrad(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                    const double* g_out, int32_t c_out, const double* f_in, int32_t c_in,
                    double* dW);

/* f2 — pooling over a kernel map.  mode: 0 = max (Alg. 3), 1 = average
 * (Alg. 4: F' / N), 2 = sum (Alg. 4 without the division, "sum pooling").  For every output
 * o the inputs are the pairs (a, o) of all offsets, in concatenated order (offset k
 * ascending, "I and O ... concatenated"); max keeps the FIRST maximal input in that
 * order (ties) and reports it in argmax[o][c].  Outputs with no input are 0 (argmax
 * -1).  fp64. */
enum { ORC_POOL_MAX = 0, ORC_POOL_AVG = 1, ORC_POOL_SUM = 2 };
void orc_pool_forward(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                      const double* f_in, int32_t C, int64_t n_out, int32_t mode, double* f_out,
                      int32_t* argmax);
/* Reverse mode: max routes G_out[o][c] to argmax[o][c]; avg spreads G_out[o] / N_o over the
 * inputs of o; sum copies G_out[o] to them. */
void orc_pool_backward(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                       const double* g_out, int32_t C, int64_t n_out, int32_t mode, const int32_t* argmax,
                       double* g_in, int64_t n_in);
/* Global pooling ("maps all inputs to the origin"): one output per batch index b,
 * sum (mode 2) or average (mode 1) of the rows whose batch is b.  batch[r] in [0, n_batch). */
void orc_global_pool(const int32_t* batch, int64_t n, const double* f_in, int32_t C, int32_t n_batch,
                     int32_t mode, double* f_out);

/* f3 — mean-field inference of the TS-CRF (Alg. 5, Eq. 4): Q^0 = softmax(phi_u)
 * (reading R25: the normalised form of Alg. 5's exp(phi_u)); for n = 1..N:
 * Q~^n = generalized sparse conv of Q^(n-1) with the pairwise kernel phi_p = W [K][C][C]
 * over the 7D kernel map (Eq. 4's sum over j in N^7(x_i) of phi_p(x_i, x_j) Q_j), then
 * Q^n = softmax(phi_u + Q~^n) per node.  fp64. */
void orc_crf_infer(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                   const double* phi_u, int64_t n, int32_t C, const double* W, int32_t n_iters, double* q);

/* The reverse map ("the role of input and output coordinates is reversed"): every pair
 * (a, o) of offset k becomes (o, a), output-ascending within the offset.  Its forward conv
 * with W_k^T is the input gradient O7; reverse(kmap(fine -> coarse)) is the transposed map. */
int orc_kmap_reverse(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                     int64_t* rptr, int32_t* rin, int32_t* rout);

/* Threads of the optional OpenMP loops (n > 0 sets it; returns the count in effect).  The
 * parallel loops split only work whose writes are disjoint (pairs of one offset, rows of
 * dW_k, output rows), so every result is bit-identical for any thread count. */
int orc_set_threads(int32_t n);

#ifdef __cplusplus
}
#endif
#endif
