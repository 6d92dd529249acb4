// pool.cu — pooling over a kernel map:
//   max pooling (Alg. 3)   F_out[o][c] = max over the inputs a of o of F_in[a][c], with the
//                          argmax (first maximal input in concatenated order: offset k
//                          ascending — ties as S:262) for the reverse mode;
//   average pooling (Alg. 4)  F' / N with N = number of inputs of o;
//   sum pooling (Alg. 4 without the division).
// The paper sorts (I, O) by output and reduces with a custom kernel / cuSPARSE csrmm.  Here
// the map's dense neighbour table already groups the inputs of every output row, so one
// warp reduces one output row over its K table entries (32 channels per lane pass) — a
// gather-reduce bound by L2 traffic.  The reverse mode walks the map's reverse view (the
// outputs of every input row) and sums in offset order: no atomics, deterministic.
// Outputs with no input are written as 0 (argmax -1).
#include <cuda_bf16.h>

#include "conv.cuh"

namespace mk {
namespace {

constexpr int kThreads = 256;
constexpr int kRowsPerBlock = kThreads / 32;

__device__ __forceinline__ float ld_feat(const void* p, int64_t i, int bf16) {
  return bf16 ? __bfloat162float(((const __nv_bfloat16*)p)[i]) : ((const float*)p)[i];
}
__device__ __forceinline__ void st_feat(void* p, int64_t i, float v, int bf16) {
  if (bf16) ((__nv_bfloat16*)p)[i] = __float2bfloat16_rn(v);
  else ((float*)p)[i] = v;
}

// One warp per table position i (output row perm[i]).  The K <= 32 neighbour indices of
// the row are loaded once (lane k holds entry k) and broadcast with shuffles, so the value
// loads of all offsets are independent; lanes cover 32 channels per pass.
__global__ void __launch_bounds__(kThreads) k_pool_fwd(NbrView nb, int64_t n_rows, const void* __restrict__ x,
                                                       int C, int bf16, int mode, void* __restrict__ y,
                                                       int32_t* __restrict__ argmax) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  if (i >= n_rows) return;
  const int64_t o = nb.row_of(i);
  const int kw = min(nb.K, 32);
  for (int c0 = 0; c0 < C; c0 += 32) {  // warp-uniform trip count: the shuffles see every lane
    const int c = c0 + lane;
    const bool valid = c < C;
    float acc = 0.f;
    int32_t best = -1, cnt = 0;
    for (int k0 = 0; k0 < nb.K; k0 += kw) {
      const int32_t mine = k0 + lane < nb.K ? nb.at(k0 + lane, i) : -1;
#pragma unroll 8
      for (int kk = 0; kk < kw && k0 + kk < nb.K; ++kk) {
        const int32_t a = __shfl_sync(0xffffffffu, mine, kk);
        if (a < 0 || !valid) continue;
        const float v = ld_feat(x, (int64_t)a * C + c, bf16);
        if (mode == MK_POOL_MAX) {
          if (best < 0 || v > acc) {  // strictly greater: the first maximal input wins
            acc = v;
            best = a;
          }
        } else {
          acc += v;
        }
        ++cnt;
      }
    }
    if (!valid) continue;
    if (mode == MK_POOL_AVG && cnt > 0) acc /= (float)cnt;
    st_feat(y, o * C + c, acc, bf16);
    if (mode == MK_POOL_MAX && argmax) argmax[o * C + c] = best;
  }
}

// Number of inputs of every output row (average pooling's N), from the forward table.
__global__ void k_pool_counts(NbrView nb, int64_t n_rows, int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = 0;
    for (int k = 0; k < nb.K; ++k) c += nb.at(k, i) >= 0;
    cnt[nb.row_of(i)] = c;
  }
}

// One warp per position i of the reverse view (input row a = permT[i]); the outputs o of a
// are visited in offset order (indices loaded once per lane, broadcast with shuffles).
__global__ void __launch_bounds__(kThreads) k_pool_bwd(NbrView nt, int64_t n_rows, const void* __restrict__ g,
                                                       int C, int bf16, int mode, const int32_t* __restrict__ argmax,
                                                       const int32_t* __restrict__ cnt, void* __restrict__ gx) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  if (i >= n_rows) return;
  const int64_t a = nt.row_of(i);
  const int kw = min(nt.K, 32);
  for (int c0 = 0; c0 < C; c0 += 32) {  // warp-uniform trip count: the shuffles see every lane
    const int c = c0 + lane;
    const bool valid = c < C;
    float acc = 0.f;
    for (int k0 = 0; k0 < nt.K; k0 += kw) {
      const int32_t mine = k0 + lane < nt.K ? nt.at(k0 + lane, i) : -1;
#pragma unroll 8
      for (int kk = 0; kk < kw && k0 + kk < nt.K; ++kk) {
        const int32_t o = __shfl_sync(0xffffffffu, mine, kk);
        if (o < 0 || !valid) continue;
        const int64_t e = (int64_t)o * C + c;
        if (mode == MK_POOL_MAX) {
          if (__ldg(argmax + e) == (int32_t)a) acc += ld_feat(g, e, bf16);
        } else if (mode == MK_POOL_AVG) {
          acc += ld_feat(g, e, bf16) / (float)__ldg(cnt + o);
        } else {
          acc += ld_feat(g, e, bf16);
        }
      }
    }
    if (valid) st_feat(gx, a * C + c, acc, bf16);
  }
}

// Vectorised variants (C a multiple of 8 for bf16 / 4 for fp32, 16-byte aligned rows): one
// thread per (table position, 16-byte channel chunk), value loads of 4 offsets in flight,
// 16-byte loads and stores, argmax as 8 / 4 int32 per chunk.  configs[1] stride-2 2^3
// pooling, bf16 64 ch, cold L2: max fwd 38 us (warp-per-row scalar kernel: 33), max bwd 51
// (72), avg fwd 29 (31); warm L2 max fwd 16.5 us.
template <typename T>
struct Vec16;
template <>
struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void load(const void* p, float (&v)[8]) {
    const uint4 u = __ldg((const uint4*)p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[2 * e] = __uint_as_float(w[e] << 16);
      v[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
  }
  __device__ static void store(void* p, const float (&v)[8]) {
    uint32_t h[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __nv_bfloat162 t = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
      h[e] = *(const uint32_t*)&t;
    }
    *(uint4*)p = make_uint4(h[0], h[1], h[2], h[3]);
  }
};
template <>
struct Vec16<float> {
  static constexpr int N = 4;
  __device__ static void load(const void* p, float (&v)[4]) {
    const float4 f = __ldg((const float4*)p);
    v[0] = f.x, v[1] = f.y, v[2] = f.z, v[3] = f.w;
  }
  __device__ static void store(void* p, const float (&v)[4]) { *(float4*)p = make_float4(v[0], v[1], v[2], v[3]); }
};

template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_pool_fwd_vec(NbrView nb, int64_t n_rows, const T* __restrict__ x, int C,
                                                      T* __restrict__ y, int32_t* __restrict__ argmax) {
  constexpr int mode = MODE;
  constexpr int U = 4;  // value loads in flight per thread
  constexpr int V = Vec16<T>::N;
  const int L = C / V;  // chunks per row
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_rows * L; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / L;
    const int ch = (int)(t - i * L);
    const int64_t o = nb.row_of(i);
    float acc[V];
    int32_t best[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.f, best[e] = -1;
    int cnt = 0;
    for (int k0 = 0; k0 < nb.K; k0 += U) {
      int32_t a[U];
#pragma unroll
      for (int j = 0; j < U; ++j) a[j] = k0 + j < nb.K ? nb.at(k0 + j, i) : -1;
      float v[U][V];
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (a[j] >= 0) Vec16<T>::load(x + (int64_t)a[j] * C + ch * V, v[j]);
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (a[j] < 0) continue;
        ++cnt;
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if (mode == MK_POOL_MAX) {
            if (best[e] < 0 || v[j][e] > acc[e]) {  // strictly greater: the first maximal input wins
              acc[e] = v[j][e];
              best[e] = a[j];
            }
          } else {
            acc[e] += v[j][e];
          }
        }
      }
    }
    if (mode == MK_POOL_AVG && cnt > 0) {
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] /= (float)cnt;
    }
    Vec16<T>::store(y + o * C + ch * V, acc);
    if (mode == MK_POOL_MAX && argmax) {
      int4* am = (int4*)(argmax + o * C + ch * V);
#pragma unroll
      for (int e = 0; e < V; e += 4) am[e / 4] = make_int4(best[e], best[e + 1], best[e + 2], best[e + 3]);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_pool_bwd_vec(NbrView nt, int64_t n_rows, const T* __restrict__ g, int C,
                                                      int mode, const int32_t* __restrict__ argmax,
                                                      const int32_t* __restrict__ cnt, T* __restrict__ gx) {
  constexpr int V = Vec16<T>::N;
  const int L = C / V;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_rows * L; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / L;
    const int ch = (int)(t - i * L);
    const int64_t a = nt.row_of(i);
    float acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.f;
    for (int k0 = 0; k0 < nt.K; k0 += 8) {
      int32_t o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = k0 + j < nt.K ? nt.at(k0 + j, i) : -1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // in offset order (fixed summation order)
        if (o[j] < 0) continue;
        const int64_t e0 = (int64_t)o[j] * C + ch * V;
        float v[V];
        Vec16<T>::load(g + e0, v);
        if (mode == MK_POOL_MAX) {
#pragma unroll
          for (int e = 0; e < V; e += 4) {
            const int4 am = __ldg((const int4*)(argmax + e0 + e));
            acc[e] += am.x == (int32_t)a ? v[e] : 0.f;
            acc[e + 1] += am.y == (int32_t)a ? v[e + 1] : 0.f;
            acc[e + 2] += am.z == (int32_t)a ? v[e + 2] : 0.f;
            acc[e + 3] += am.w == (int32_t)a ? v[e + 3] : 0.f;
          }
        } else if (mode == MK_POOL_AVG) {
          const float c = (float)__ldg(cnt + o[j]);
#pragma unroll
          for (int e = 0; e < V; ++e) acc[e] += v[e] / c;
        } else {
#pragma unroll
          for (int e = 0; e < V; ++e) acc[e] += v[e];
        }
      }
    }
    Vec16<T>::store(gx + a * C + ch * V, acc);
  }
}

bool vec_ok(int C, bool bf16, const void* p0, const void* p1) {
  const int V = bf16 ? 8 : 4;
  return C % V == 0 && ((uintptr_t)p0 & 15) == 0 && ((uintptr_t)p1 & 15) == 0;
}

mk_status check_pool(const mk_kmap* m, int32_t mode, int32_t C, mk_dtype dt) {
  if (!m) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "pool: null map");
  if (mode != MK_POOL_MAX && mode != MK_POOL_AVG && mode != MK_POOL_SUM)
    MK_FAIL(MK_ERR_INVALID_ARGUMENT, "pool: unknown mode");
  if (C < 1) MK_FAIL(MK_ERR_SHAPE_MISMATCH, "pool: channel count must be >= 1");
  if (dt != MK_F32 && dt != MK_BF16) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "pool: unknown dtype");
  return MK_OK;
}

}  // namespace
}  // namespace mk

using namespace mk;

extern "C" {

mk_status mk_pool_forward(mk_context* ctx, const mk_kmap* m, int32_t mode, const void* d_fin, int32_t C, mk_dtype dt,
                          void* d_fout, int32_t* d_argmax, void* stream) {
  clear_error();
  mk_status st = check_pool(m, mode, C, dt);
  if (st != MK_OK) return st;
  if (!ctx) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_pool_forward: null context");
  if (m->n_out == 0) return MK_OK;
  if (!d_fout || (m->n_in > 0 && !d_fin)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_pool_forward: null features");
  const NbrView v = forward_view(m);
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* am = mode == MK_POOL_MAX ? d_argmax : nullptr;
  if (vec_ok(C, dt == MK_BF16, d_fin, d_fout) && ((uintptr_t)am & 15) == 0) {
    const int64_t work = m->n_out * (C / (dt == MK_BF16 ? 8 : 4));
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(work, 256), 16 * ctx->num_sms);
    const bool b = dt == MK_BF16;
    const auto* xb = (const __nv_bfloat16*)d_fin;
    const auto* xf = (const float*)d_fin;
    auto* yb = (__nv_bfloat16*)d_fout;
    auto* yf = (float*)d_fout;
    if (mode == MK_POOL_MAX) {
      if (b) k_pool_fwd_vec<__nv_bfloat16, MK_POOL_MAX><<<grid, 256, 0, s>>>(v, m->n_out, xb, C, yb, am);
      else k_pool_fwd_vec<float, MK_POOL_MAX><<<grid, 256, 0, s>>>(v, m->n_out, xf, C, yf, am);
    } else if (mode == MK_POOL_AVG) {
      if (b) k_pool_fwd_vec<__nv_bfloat16, MK_POOL_AVG><<<grid, 256, 0, s>>>(v, m->n_out, xb, C, yb, am);
      else k_pool_fwd_vec<float, MK_POOL_AVG><<<grid, 256, 0, s>>>(v, m->n_out, xf, C, yf, am);
    } else {
      if (b) k_pool_fwd_vec<__nv_bfloat16, MK_POOL_SUM><<<grid, 256, 0, s>>>(v, m->n_out, xb, C, yb, am);
      else k_pool_fwd_vec<float, MK_POOL_SUM><<<grid, 256, 0, s>>>(v, m->n_out, xf, C, yf, am);
    }
  } else {
    const unsigned grid = (unsigned)ceil_div(m->n_out, kRowsPerBlock);
    k_pool_fwd<<<grid, kThreads, 0, s>>>(v, m->n_out, d_fin, C, dt == MK_BF16, mode, d_fout, am);
  }
  MK_LAUNCH_CHECK();
  return MK_OK;
}

mk_status mk_pool_backward(mk_context* ctx, const mk_kmap* m, int32_t mode, const void* d_gout, int32_t C,
                           mk_dtype dt, const int32_t* d_argmax, void* d_gin, void* stream) {
  clear_error();
  mk_status st = check_pool(m, mode, C, dt);
  if (st != MK_OK) return st;
  if (!ctx) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_pool_backward: null context");
  if (m->n_in == 0) return MK_OK;
  if (!d_gin || (m->n_out > 0 && !d_gout)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_pool_backward: null gradients");
  if (mode == MK_POOL_MAX && m->n_out > 0 && !d_argmax)
    MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_pool_backward: max pooling needs the forward argmax");
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* cnt = nullptr;
  if (mode == MK_POOL_AVG && m->n_out > 0) {
    cnt = (int32_t*)dev_alloc(ctx->alloc, sizeof(int32_t) * m->n_out, s);
    if (!cnt) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "mk_pool_backward: workspace allocation failed");
    k_pool_counts<<<(unsigned)std::min<int64_t>(ceil_div(m->n_out, 256), 4 * ctx->num_sms), 256, 0, s>>>(
        forward_view(m), m->n_out, cnt);
    g_launches++;
  }
  const NbrView v = dgrad_view(m);
  if (vec_ok(C, dt == MK_BF16, d_gout, d_gin) && ((uintptr_t)d_argmax & 15) == 0) {
    const int64_t work = m->n_in * (C / (dt == MK_BF16 ? 8 : 4));
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(work, 256), 16 * ctx->num_sms);
    if (dt == MK_BF16)
      k_pool_bwd_vec<__nv_bfloat16><<<grid, 256, 0, s>>>(v, m->n_in, (const __nv_bfloat16*)d_gout, C, mode, d_argmax,
                                                          cnt, (__nv_bfloat16*)d_gin);
    else
      k_pool_bwd_vec<float><<<grid, 256, 0, s>>>(v, m->n_in, (const float*)d_gout, C, mode, d_argmax, cnt,
                                                  (float*)d_gin);
  } else {
    const unsigned grid = (unsigned)ceil_div(m->n_in, kRowsPerBlock);
    k_pool_bwd<<<grid, kThreads, 0, s>>>(v, m->n_in, d_gout, C, dt == MK_BF16, mode, d_argmax, cnt, d_gin);
  }
  g_launches++;
  const cudaError_t e = cudaGetLastError();
  if (cnt) dev_free(ctx->alloc, cnt, s);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("mk_pool_backward: ") + cudaGetErrorString(e));
  return MK_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ global pooling
// Global pooling ("the kernel map that maps all inputs to the origin"): one output
// row per batch index b, the sum (or mean) of the rows whose batch is b.  Deterministic
// two-level reduction: CTA j owns a contiguous range of rows and sums them in row order into
// a shared [n_batch][C] accumulator (thread = channel, so every element has one writer),
// then writes its partial; the partials are summed in CTA order.
namespace mk {
namespace {

constexpr int kGpCtas = 296;

__global__ void __launch_bounds__(256) k_global_partial(const int4* __restrict__ keys, int64_t n, int D,
                                                        const void* __restrict__ x, int C, int bf16, int n_batch,
                                                        float* __restrict__ part, int32_t* __restrict__ pcnt) {
  extern __shared__ float s_acc[];  // [n_batch][C], then counts [n_batch]
  int32_t* s_cnt = (int32_t*)(s_acc + (int64_t)n_batch * C);
  for (int i = threadIdx.x; i < n_batch * C; i += blockDim.x) s_acc[i] = 0.f;
  for (int i = threadIdx.x; i < n_batch; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
  for (int64_t r = r0; r < r1; ++r) {
    const int b = key_batch(__ldg(keys + r), D);
    if (b < 0 || b >= n_batch) continue;  // (uniform across the block)
    for (int c = threadIdx.x; c < C; c += blockDim.x) s_acc[b * C + c] += ld_feat(x, r * C + c, bf16);
    if (threadIdx.x == 0) ++s_cnt[b];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_batch * C; i += blockDim.x) part[(int64_t)blockIdx.x * n_batch * C + i] = s_acc[i];
  for (int i = threadIdx.x; i < n_batch; i += blockDim.x) pcnt[(int64_t)blockIdx.x * n_batch + i] = s_cnt[i];
}

__global__ void k_global_reduce(const float* __restrict__ part, const int32_t* __restrict__ pcnt, int n_cta,
                                int n_batch, int C, int avg, int bf16, void* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n_batch * C) return;
  const int b = (int)(i / C);
  float s = 0.f;
  int64_t cnt = 0;
  for (int j = 0; j < n_cta; ++j) {
    s += part[(int64_t)j * n_batch * C + i];
    cnt += pcnt[(int64_t)j * n_batch + b];
  }
  if (avg && cnt > 0) s /= (float)cnt;
  st_feat(y, i, s, bf16);
}

}  // namespace
}  // namespace mk

extern "C" mk_status mk_global_pool(mk_context* ctx, const mk_coords* c, int32_t mode, const void* d_fin, int32_t C,
                                    mk_dtype dt, int32_t n_batch, void* d_fout, void* stream) {
  using namespace mk;
  clear_error();
  if (!ctx || !c) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_global_pool: null argument");
  if (mode != MK_POOL_AVG && mode != MK_POOL_SUM) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_global_pool: mode must be AVG or SUM");
  if (C < 1 || n_batch < 0) MK_FAIL(MK_ERR_SHAPE_MISMATCH, "mk_global_pool: bad sizes");
  if (dt != MK_F32 && dt != MK_BF16) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_global_pool: unknown dtype");
  if (n_batch == 0) return MK_OK;
  {
    const mk_status rs = coords_resolve(c);
    if (rs != MK_OK) return rs;
  }
  if (!d_fout || (c->n > 0 && !d_fin)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_global_pool: null features");
  const size_t smem = sizeof(float) * (size_t)n_batch * C + sizeof(int32_t) * n_batch;
  if (smem > 200 * 1024) MK_FAIL(MK_ERR_UNSUPPORTED, "mk_global_pool: n_batch * C above 51200");
  cudaStream_t s = (cudaStream_t)stream;
  const int n_cta = kGpCtas;
  char* ws = (char*)dev_alloc(ctx->alloc, sizeof(float) * (size_t)n_cta * n_batch * C + sizeof(int32_t) * n_cta * n_batch, s);
  if (!ws) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "mk_global_pool: workspace allocation failed");
  float* part = (float*)ws;
  int32_t* pcnt = (int32_t*)(part + (size_t)n_cta * n_batch * C);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_global_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_global_partial<<<n_cta, 256, smem, s>>>(c->keys, c->n, c->D, d_fin, C, dt == MK_BF16, n_batch, part, pcnt);
  k_global_reduce<<<(unsigned)ceil_div((int64_t)n_batch * C, 256), 256, 0, s>>>(part, pcnt, n_cta, n_batch, C,
                                                                               mode == MK_POOL_AVG, dt == MK_BF16, d_fout);
  g_launches += 2;
  const cudaError_t e = cudaGetLastError();
  dev_free(ctx->alloc, ws, s);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("mk_global_pool: ") + cudaGetErrorString(e));
  return MK_OK;
}
