// conv.cuh — internal interface between the conv entry points (conv.cu) and the kernels
// (conv_simt.cu: fp32 FFMA; conv_umma.cu: bf16 tcgen05).
#pragma once
#include "mk_internal.cuh"

namespace mk {

// Read-only view of a dense neighbour table for an output-stationary gather-GEMM:
// at(k, r) = source row feeding row r at offset k (or -1).  With `mirror` set, the table
// is the forward nbr of a symmetric submanifold map read at the mirrored offset
// (nbrT[k] == nbr[mirror[k]]), so dgrad needs no second table.
struct NbrView {
  const int32_t* tab = nullptr;     // [K][n], n = rows padded to a multiple of 128 (padding -1)
  const int32_t* mirror = nullptr;  // [K] or null
  const uint32_t* mask = nullptr;   // [n/128][mw], already mirrored for dgrad views
  const int32_t* perm = nullptr;    // [n] output row of table position i, or null (identity)
  int64_t n = 0;
  int K = 0;
  int mw = 1;
  __device__ __forceinline__ int kk(int k) const { return mirror ? __ldg(mirror + k) : k; }
  __device__ __forceinline__ int32_t at(int k, int64_t r) const { return __ldg(tab + (int64_t)kk(k) * n + r); }
  __device__ __forceinline__ int64_t row_of(int64_t i) const { return perm ? (int64_t)__ldg(perm + i) : i; }
  __device__ __forceinline__ bool active(int64_t tile128, int k) const {
    return (__ldg(mask + tile128 * mw + (k >> 5)) >> (k & 31)) & 1u;
  }
};

// The forward view of a map (rows = outputs, entries = input rows) and its reverse view
// (rows = inputs, entries = output rows; nbrT, or nbr read at the mirrored offset when the
// map is a symmetric submanifold map).
inline NbrView forward_view(const mk_kmap* m) {
  NbrView v;
  v.tab = m->nbr;
  v.mask = m->tile_mask;
  v.perm = m->perm;
  v.n = m->nbr_stride;
  v.K = m->K;
  v.mw = m->mask_words;
  return v;
}

inline NbrView dgrad_view(const mk_kmap* m) {
  NbrView v;
  v.K = m->K;
  v.mw = m->mask_words;
  v.n = m->nbrT_stride;
  v.mask = m->tile_maskT;
  v.perm = m->permT;
  if (m->nbrT) {
    v.tab = m->nbrT;
  } else {  // symmetric submanifold map: nbrT[k] = nbr[mirror[k]]
    v.tab = m->nbr;
    v.mirror = m->d_mirror;
  }
  return v;
}

// Split-K plan for the weight gradient: the pairs of offset k are cut into chunks of at
// most `chunk` pairs; chunks[c] = (k, begin, end, c); chunk_begin[k] = first chunk of k.
struct WgradPlan {
  int4* chunks = nullptr;
  int32_t* chunk_begin = nullptr;
  float* part = nullptr;  // [n_chunks][c_out][c_in]
  int64_t n_chunks = 0;
};

// Fused forward epilogue (ReLU and batch normalisation act on the rows of F):
//   y[r][j] = act(acc[r][j] * scale[j] + shift[j] + residual[r][j]),  act = ReLU or identity.
// scale / shift fp32 [c_y] (null: 1 / 0); residual [n_rows][c_y] in the output dtype, indexed
// by output row (null: 0).  Default-constructed = plain conv.
struct Epilogue {
  const float* scale = nullptr;
  const float* shift = nullptr;
  const void* residual = nullptr;
  int relu = 0;
  __host__ __device__ bool active() const { return scale || shift || residual || relu; }
};
__device__ __forceinline__ float epi_apply(const Epilogue& ep, float v, int j, float res) {
  if (ep.scale) v *= __ldg(ep.scale + j);
  if (ep.shift) v += __ldg(ep.shift + j);
  v += res;
  return ep.relu ? fmaxf(v, 0.f) : v;
}

mk_status launch_conv_f32(const NbrView& nb, const float* x, int c_x, const float* W, int c_in_w, int c_out_w,
                          void* y, int c_y, mk_dtype out_dt, int64_t n_rows, bool trans, cudaStream_t s,
                          const Epilogue& ep = Epilogue());
mk_status launch_wgrad_f32(const mk_kmap* m, const WgradPlan& plan, const float* g, int c_out, const float* x,
                           int c_in, float* dW, cudaStream_t s);

// bf16 tensor-core path (conv_umma.cu)
mk_status launch_conv_bf16(mk_context* ctx, const NbrView& nb, const void* x, int64_t n_src, int c_x, const void* W,
                           int c_in_w, int c_out_w, void* y, int c_y, mk_dtype out_dt, int64_t n_rows, bool trans,
                           cudaStream_t s, const Epilogue& ep = Epilogue());
mk_status launch_wgrad_bf16(mk_context* ctx, const mk_kmap* m, const void* g, int c_out, const void* x, int c_in,
                            float* dW, cudaStream_t s);
// fp32 on the bf16 tensor cores by three-way operand splitting (conv_split.cu)
bool split_f32_enabled(int c_in, int c_out, int K, const Epilogue& ep);
mk_status launch_conv_f32_split(mk_context* ctx, const NbrView& nb, const float* x, int64_t n_src, int c_x,
                                const float* W, int c_in_w, int c_out_w, void* y, int c_y, mk_dtype out_dt,
                                int64_t n_rows, bool trans, cudaStream_t s);
mk_status launch_wgrad_f32_split(mk_context* ctx, const mk_kmap* m, const float* g, int c_out, const float* x,
                                 int c_in, float* dW, cudaStream_t s);
__global__ void k_reduce_partials(const int32_t* __restrict__ chunk_begin, const float* __restrict__ part,
                                  int64_t tile_elems, float* __restrict__ dW);

}  // namespace mk
