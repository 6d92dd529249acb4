// conv_simt.cu — exact-fp32 (FFMA) gather-GEMM kernels: the fp32 mode of mk_conv_* and
// the precision anchor of the tensor-core path.
//
//   k_conv_f32<TRANS>  output-stationary: a CTA owns 32 output rows and all output channels,
//                      loops over the non-empty offsets of its 128-row tile, gathers the
//                      neighbour rows into shared memory (zeros for absent neighbours) and
//                      accumulates W_k x (or W_k^T g for TRANS = dgrad) in registers.
//                      Row-complete outputs => no atomics, fixed summation order.
//   k_wgrad_f32        split-K over the pairs of one offset: each CTA reduces a chunk of
//                      pairs into a partial dW_k tile; k_reduce_partials sums the partials of
//                      every offset in chunk order (deterministic, blocked summation).
#include <cuda_bf16.h>

#include "conv.cuh"

namespace mk {
namespace {

constexpr int kRows = 32;    // output rows per CTA
constexpr int kCk = 32;      // channel chunk staged in shared memory
constexpr int kThreads = 256;

template <typename TOut>
__device__ __forceinline__ void store_out(TOut* p, float v);
template <>
__device__ __forceinline__ void store_out<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void store_out<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// out[r][j] = sum_k sum_c Wk(j, c) * in[nb(k, r)][c]
//   forward: j = co, c = ci, Wk(j,c) = W[k][co][ci], nb = nbr[k][o]
//   dgrad  : j = ci, c = co, Wk(j,c) = W[k][co][ci] (transposed access), nb = nbrT[k][a]
template <bool TRANS, typename TOut>
__global__ void __launch_bounds__(kThreads) k_conv_f32(NbrView nb, const float* __restrict__ x, int c_x,
                                                       const float* __restrict__ W, int c_in_w, int c_out_w,
                                                       TOut* __restrict__ y, int c_y, int64_t n_rows,
                                                       Epilogue ep) {
  __shared__ float s_x[kRows][kCk + 1];
  __shared__ float s_w[256][kCk + 1];  // [j][c chunk], c_y <= 256
  __shared__ int32_t s_nb[kRows];
  const int64_t row0 = (int64_t)blockIdx.x * kRows;
  const int r = threadIdx.x % kRows;     // lane -> row (conflict-free s_x reads with padding)
  const int jg = threadIdx.x / kRows;    // 8 groups of output channels
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.f;
  const int64_t tile128 = row0 / 128;
  for (int k = 0; k < nb.K; ++k) {
    if (!nb.active(tile128, k)) continue;
    __syncthreads();
    if (threadIdx.x < kRows) {
      const int64_t row = row0 + threadIdx.x;
      s_nb[threadIdx.x] = row < n_rows ? nb.at(k, row) : -1;
    }
    __syncthreads();
    bool any = false;
    for (int i = 0; i < kRows; ++i) any |= s_nb[i] >= 0;
    if (!any) continue;
    const float* Wk = W + (int64_t)k * c_out_w * c_in_w;
    for (int c0 = 0; c0 < c_x; c0 += kCk) {
      __syncthreads();
      for (int i = threadIdx.x; i < kRows * kCk; i += kThreads) {
        const int rr = i / kCk, cc = i % kCk;
        const int32_t a = s_nb[rr];
        s_x[rr][cc] = (a >= 0 && c0 + cc < c_x) ? x[(int64_t)a * c_x + c0 + cc] : 0.f;
      }
      for (int i = threadIdx.x; i < c_y * kCk; i += kThreads) {
        const int j = i / kCk, cc = i % kCk;
        float w = 0.f;
        if (c0 + cc < c_x) w = TRANS ? Wk[(int64_t)(c0 + cc) * c_in_w + j] : Wk[(int64_t)j * c_in_w + c0 + cc];
        s_w[j][cc] = w;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int j = jg + 8 * i;
        if (j < c_y) {
          float a = acc[i];
#pragma unroll 8
          for (int cc = 0; cc < kCk; ++cc) a = fmaf(s_w[j][cc], s_x[r][cc], a);
          acc[i] = a;
        }
      }
    }
  }
  const int64_t pos = row0 + r;
  if (pos < n_rows) {
    const int64_t row = nb.row_of(pos);  // tables are stored in the map's internal row order
    const TOut* res = (const TOut*)ep.residual;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int j = jg + 8 * i;
      if (j < c_y) {
        float v = acc[i];
        if (ep.active()) v = epi_apply(ep, v, j, res ? (float)res[row * c_y + j] : 0.f);
        store_out<TOut>(y + row * c_y + j, v);
      }
    }
  }
}

// Partial dW over one chunk of pairs of one offset: part[chunk][co][ci] (64x64 tile per CTA).
__global__ void __launch_bounds__(kThreads) k_wgrad_f32(const int4* __restrict__ chunks, const int32_t* __restrict__ in_idx,
                                                        const int32_t* __restrict__ out_idx, const float* __restrict__ g,
                                                        int c_out, const float* __restrict__ x, int c_in,
                                                        float* __restrict__ part) {
  __shared__ float s_g[32][64 + 1];
  __shared__ float s_x[32][64 + 1];
  const int4 ch = chunks[blockIdx.x];  // (k, begin, end, chunk id)
  const int co0 = blockIdx.y * 64, ci0 = blockIdx.z * 64;
  const int tco = threadIdx.x / 16, tci = threadIdx.x % 16;  // 16x16 threads, 4x4 outputs each
  float acc[4][4] = {};
  for (int p0 = ch.y; p0 < ch.z; p0 += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 64; i += kThreads) {
      const int pp = i / 64, c = i % 64;
      const int p = p0 + pp;
      float gv = 0.f, xv = 0.f;
      if (p < ch.z) {
        if (co0 + c < c_out) gv = g[(int64_t)out_idx[p] * c_out + co0 + c];
        if (ci0 + c < c_in) xv = x[(int64_t)in_idx[p] * c_in + ci0 + c];
      }
      s_g[pp][c] = gv;
      s_x[pp][c] = xv;
    }
    __syncthreads();
#pragma unroll 4
    for (int pp = 0; pp < 32; ++pp) {
      float gv[4], xv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        gv[i] = s_g[pp][tco + 16 * i];
        xv[i] = s_x[pp][tci + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(gv[i], xv[j], acc[i][j]);
    }
  }
  float* out = part + (int64_t)ch.w * c_out * c_in;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int co = co0 + tco + 16 * i, ci = ci0 + tci + 16 * j;
      if (co < c_out && ci < c_in) out[(int64_t)co * c_in + ci] = acc[i][j];
    }
}

}  // namespace

// dW[k] = sum of the partials of offset k's chunks, in chunk order.
__global__ void k_reduce_partials(const int32_t* __restrict__ chunk_begin, const float* __restrict__ part,
                                  int64_t tile_elems, float* __restrict__ dW) {
  const int k = blockIdx.y;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= tile_elems) return;
  float s = 0.f;
  for (int c = chunk_begin[k]; c < chunk_begin[k + 1]; ++c) s += part[(int64_t)c * tile_elems + e];
  dW[(int64_t)k * tile_elems + e] = s;
}

mk_status launch_conv_f32(const NbrView& nb, const float* x, int c_x, const float* W, int c_in_w, int c_out_w,
                          void* y, int c_y, mk_dtype out_dt, int64_t n_rows, bool trans, cudaStream_t s,
                          const Epilogue& ep) {
  if (c_y > 256) MK_FAIL(MK_ERR_UNSUPPORTED, "fp32 conv: more than 256 output channels");
  if (n_rows == 0) return MK_OK;
  const unsigned grid = (unsigned)ceil_div(n_rows, kRows);
  if (out_dt == MK_F32) {
    if (trans) k_conv_f32<true, float><<<grid, kThreads, 0, s>>>(nb, x, c_x, W, c_in_w, c_out_w, (float*)y, c_y, n_rows, ep);
    else k_conv_f32<false, float><<<grid, kThreads, 0, s>>>(nb, x, c_x, W, c_in_w, c_out_w, (float*)y, c_y, n_rows, ep);
  } else {
    if (trans)
      k_conv_f32<true, __nv_bfloat16><<<grid, kThreads, 0, s>>>(nb, x, c_x, W, c_in_w, c_out_w, (__nv_bfloat16*)y, c_y, n_rows, ep);
    else
      k_conv_f32<false, __nv_bfloat16><<<grid, kThreads, 0, s>>>(nb, x, c_x, W, c_in_w, c_out_w, (__nv_bfloat16*)y, c_y, n_rows, ep);
  }
  MK_LAUNCH_CHECK();
  return MK_OK;
}

// Small channel counts (c_out, c_in <= 32, e.g. the TS-CRF's classes): the whole C_out x C_in
// partial in one CTA, one output element per thread (up to 4), pairs staged 64 at a time.
constexpr int kSmallPairs = 64;
__global__ void __launch_bounds__(256) k_wgrad_f32_small(const int4* __restrict__ chunks,
                                                         const int32_t* __restrict__ in_idx,
                                                         const int32_t* __restrict__ out_idx,
                                                         const float* __restrict__ g, int c_out,
                                                         const float* __restrict__ x, int c_in,
                                                         float* __restrict__ part) {
  __shared__ float s_g[kSmallPairs][33];
  __shared__ float s_x[kSmallPairs][33];
  const int4 ch = chunks[blockIdx.x];  // (k, begin, end, chunk id)
  const int te = c_out * c_in;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int p0 = ch.y; p0 < ch.z; p0 += kSmallPairs) {
    __syncthreads();
    for (int i = threadIdx.x; i < kSmallPairs * 32; i += blockDim.x) {
      const int pp = i >> 5, c = i & 31;
      const int p = p0 + pp;
      const bool in = p < ch.z;
      s_g[pp][c] = in && c < c_out ? g[(int64_t)out_idx[p] * c_out + c] : 0.f;
      s_x[pp][c] = in && c < c_in ? x[(int64_t)in_idx[p] * c_in + c] : 0.f;
    }
    __syncthreads();
    const int np = min(kSmallPairs, ch.z - p0);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = threadIdx.x + r * 256;
      if (e >= te) break;
      const int co = e / c_in, ci = e - co * c_in;
      float a = acc[r];
      for (int pp = 0; pp < np; ++pp) a = fmaf(s_g[pp][co], s_x[pp][ci], a);
      acc[r] = a;
    }
  }
  float* out = part + (int64_t)ch.w * te;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int e = threadIdx.x + r * 256;
    if (e < te) out[e] = acc[r];
  }
}

mk_status launch_wgrad_f32(const mk_kmap* m, const WgradPlan& plan, const float* g, int c_out, const float* x,
                           int c_in, float* dW, cudaStream_t s) {
  if (plan.n_chunks > 0 && c_out <= 32 && c_in <= 32) {
    k_wgrad_f32_small<<<(unsigned)plan.n_chunks, 256, 0, s>>>(plan.chunks, m->in_idx, m->out_idx, g, c_out, x, c_in,
                                                              plan.part);
    MK_LAUNCH_CHECK();
  } else if (plan.n_chunks > 0) {
    dim3 grid((unsigned)plan.n_chunks, (unsigned)ceil_div(c_out, 64), (unsigned)ceil_div(c_in, 64));
    k_wgrad_f32<<<grid, kThreads, 0, s>>>(plan.chunks, m->in_idx, m->out_idx, g, c_out, x, c_in, plan.part);
    MK_LAUNCH_CHECK();
  }
  const int64_t te = (int64_t)c_out * c_in;
  dim3 rg((unsigned)ceil_div(te, 256), (unsigned)m->K);
  k_reduce_partials<<<rg, 256, 0, s>>>(plan.chunk_begin, plan.part, te, dW);
  MK_LAUNCH_CHECK();
  return MK_OK;
}

}  // namespace mk
