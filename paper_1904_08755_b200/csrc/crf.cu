// crf.cu — mean-field inference of the trilateral stationary CRF (TS-CRF, SURVEY §8(f) f3;
// Alg. 5 and Eq. 4) on a 7D space-time-chroma kernel map:
//   Q^0 = softmax(phi_u)                                   (reading R25)
//   for n = 1..N:  Q~^n = generalized sparse conv(Q^(n-1); phi_p)   (the pairwise sum of
//                  Eq. 4 is a 7D sparse convolution because phi_p is stationary)
//                  Q^n  = softmax(phi_u + Q~^n)
// C <= 32 classes: one fused kernel per step (gather of the neighbours' Q rows, the C x C
// products from shared-memory W, softmax across the node's lane group); larger C: the
// exact-FFMA fp32 conv of conv_simt.cu followed by a warp-per-node softmax.
#include "conv.cuh"

namespace mk {
namespace {

// out[i] = softmax(phi[i] + add[i]) over C classes; one warp per row, warp-uniform loops.
__global__ void __launch_bounds__(256) k_crf_softmax(const float* __restrict__ phi, const float* __restrict__ add,
                                                     int64_t n, int C, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  const float* a = phi + i * C;
  const float* b = add ? add + i * C : nullptr;
  float m = -INFINITY;
  for (int c0 = 0; c0 < C; c0 += 32) {
    const int c = c0 + lane;
    if (c < C) m = fmaxf(m, a[c] + (b ? b[c] : 0.f));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float z = 0.f;
  for (int c0 = 0; c0 < C; c0 += 32) {
    const int c = c0 + lane;
    if (c < C) z += expf(a[c] + (b ? b[c] : 0.f) - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  const float inv = 1.f / z;
  for (int c0 = 0; c0 < C; c0 += 32) {
    const int c = c0 + lane;
    if (c < C) out[i * C + c] = expf(a[c] + (b ? b[c] : 0.f) - m) * inv;
  }
}

// One fused mean-field step for C <= 32 classes: Q_out[o] = softmax(phi[o] + sum_k W_k Q_in[a_k])
// over the pairs (a_k, o) of the map (Eq. 4).  A group of Cp = pow2(C) lanes owns one node
// (32 / Cp nodes per warp); lane j computes class j: the neighbour indices are broadcast
// within the group, the neighbour's Q row is spread over the group and broadcast one class
// at a time.  W lives in shared memory.  Fixed summation order (k, then c): deterministic.
// SOFTMAX = false: the convolution alone (out = sum_k W_k Q_in[a_k], or with trans = 1 the
// transposed weights W_k^T: the input gradient of Eq. 5's backward pass on the reverse view).
template <bool SOFTMAX>
__global__ void __launch_bounds__(256) k_crf_step(NbrView nb, int64_t n_rows, const float* __restrict__ phi,
                                                  const float* __restrict__ q_in, const float* __restrict__ W, int C,
                                                  int Cp, float* __restrict__ q_out, int trans) {
  extern __shared__ float s_w[];  // [K][c][j] = W[k][j][c] (lanes j read consecutive words)
  for (int i = threadIdx.x; i < nb.K * C * C; i += blockDim.x) {
    const int k = i / (C * C), r = i - k * C * C, jj = r / C, c = r - jj * C;
    if (trans) s_w[(k * C + jj) * C + c] = W[i];  // W^T[k][c][jj] = W[k][jj][c]
    else s_w[(k * C + c) * C + jj] = W[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, j = lane & (Cp - 1);
  const int per_warp = 32 / Cp;
  float* s_q = s_w + nb.K * C * C + (threadIdx.x & ~(Cp - 1)) * Cp;  // [Cp offsets][Cp classes]
  const int gsh = lane & ~(Cp - 1);
  const unsigned lowmask = Cp == 32 ? 0xffffffffu : ((1u << Cp) - 1u);
  // grid-stride over node groups (W is staged once per block)
  const int64_t n_groups = (n_rows + per_warp - 1) / per_warp;
  for (int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gw < n_groups;
       gw += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t pos = gw * per_warp + (lane / Cp);
    const bool valid = pos < n_rows;
    float acc = 0.f;
    // The neighbours' Q rows of the node are staged in shared memory first (independent
    // loads), then lane j forms sum_k sum_c W_k[j][c] Q_k[c] from broadcast reads.
    for (int k0 = 0; k0 < nb.K; k0 += Cp) {
      const int32_t mine = valid && k0 + j < nb.K ? nb.at(k0 + j, pos) : -1;
      const unsigned present = (__ballot_sync(0xffffffffu, mine >= 0) >> gsh) & lowmask;
#pragma unroll 8
      for (int kk = 0; kk < Cp; ++kk) {
        const int32_t a = __shfl_sync(0xffffffffu, mine, kk, Cp);
        s_q[kk * Cp + j] = (a >= 0 && j < C) ? __ldg(q_in + (int64_t)a * C + j) : 0.f;
      }
      __syncwarp();
      for (unsigned pr = present; pr; pr &= pr - 1) {
        const int kk = __ffs(pr) - 1;
        const float* wk = s_w + (k0 + kk) * C * C + min(j, C - 1);
        const float* qk = s_q + kk * Cp;
        float t = 0.f;
        for (int c = 0; c < C; ++c) t = fmaf(wk[c * C], qk[c], t);
        acc += t;
      }
      __syncwarp();
    }
    const int64_t o = valid ? nb.row_of(pos) : 0;
    if (!SOFTMAX) {
      if (valid && j < C) q_out[o * C + j] = acc;
      continue;
    }
    // softmax over the group's C classes
    const float v = (valid && j < C) ? __ldg(phi + o * C + j) + acc : -INFINITY;
    float m = v;
    for (int w = Cp / 2; w > 0; w >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, w, Cp));
    const float e = (valid && j < C) ? expf(v - m) : 0.f;
    float z = e;
    for (int w = Cp / 2; w > 0; w >>= 1) z += __shfl_xor_sync(0xffffffffu, z, w, Cp);
    if (valid && j < C) q_out[o * C + j] = e / z;
  }
}

}  // namespace
}  // namespace mk

using namespace mk;

extern "C" mk_status mk_crf_infer(mk_context* ctx, const mk_kmap* m, const float* d_phi_u, const float* d_W,
                                  int32_t C, int32_t n_iters, float* d_q, void* stream) {
  clear_error();
  if (!ctx || !m) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_crf_infer: null argument");
  if (m->n_in != m->n_out || m->transposed)
    MK_FAIL(MK_ERR_SHAPE_MISMATCH, "mk_crf_infer: the map must connect a coordinate set to itself");
  if (C < 1 || n_iters < 0) MK_FAIL(MK_ERR_SHAPE_MISMATCH, "mk_crf_infer: bad sizes");
  const int64_t n = m->n_out;
  if (n == 0) return MK_OK;
  if (!d_phi_u || !d_q || (n_iters > 0 && !d_W)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_crf_infer: null buffers");
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)ceil_div(n, 8);
  k_crf_softmax<<<grid, 256, 0, s>>>(d_phi_u, nullptr, n, C, d_q);  // Q^0
  MK_LAUNCH_CHECK();
  if (n_iters == 0) return MK_OK;
  float* qt = (float*)dev_alloc(ctx->alloc, sizeof(float) * n * C, s);
  if (!qt) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "mk_crf_infer: workspace allocation failed");
  const NbrView v = forward_view(m);
  mk_status st = MK_OK;
  if (C <= 32 && (v.K * C * C + 256 * 32) * (int)sizeof(float) <= 48 * 1024) {
    // fused steps (conv + softmax in one kernel); ping-pong between d_q and the workspace
    int Cp = 1;
    while (Cp < C) Cp <<= 1;
    const int64_t groups = ceil_div(n, 32 / Cp);
    const unsigned g2 = (unsigned)std::min<int64_t>(ceil_div(groups, 8), 6 * ctx->num_sms);
    float* bufs[2] = {d_q, qt};
    for (int it = 0; it < n_iters; ++it) {
      const float* src = bufs[it & 1];
      float* dst = bufs[(it + 1) & 1];
      k_crf_step<true><<<g2, 256, sizeof(float) * (v.K * C * C + 256 * Cp), s>>>(v, n, d_phi_u, src, d_W, C, Cp, dst,
                                                                                 0);
      g_launches++;
    }
    cudaError_t e2 = cudaSuccess;
    if (n_iters & 1) e2 = cudaMemcpyAsync(d_q, qt, sizeof(float) * n * C, cudaMemcpyDeviceToDevice, s);
    const cudaError_t e = e2 == cudaSuccess ? cudaGetLastError() : e2;
    dev_free(ctx->alloc, qt, s);
    if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("mk_crf_infer: ") + cudaGetErrorString(e));
    return MK_OK;
  }
  for (int it = 0; it < n_iters && st == MK_OK; ++it) {
    st = launch_conv_f32(v, d_q, C, d_W, C, C, qt, C, MK_F32, n, false, s);  // Q~^n
    if (st == MK_OK) {
      k_crf_softmax<<<grid, 256, 0, s>>>(d_phi_u, qt, n, C, d_q);              // Q^n
      g_launches++;
    }
  }
  const cudaError_t e = cudaGetLastError();
  dev_free(ctx->alloc, qt, s);
  if (st != MK_OK) return st;
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("mk_crf_infer: ") + cudaGetErrorString(e));
  return MK_OK;
}

// ------------------------------------------------------------------ learning (Eq. 5)
namespace mk {
namespace {

// Reverse of a row softmax: da[i][c] = q[i][c] * (g[i][c] - sum_j q[i][j] g[i][j]);
// also accumulates da into acc (dL/dphi_u collects every iteration's da, Eq. 5).
__global__ void __launch_bounds__(256) k_crf_softmax_bwd(const float* __restrict__ q, const float* __restrict__ g,
                                                         int64_t n, int C, float* __restrict__ da,
                                                         float* __restrict__ acc, int first) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  float dot = 0.f;
  for (int c0 = 0; c0 < C; c0 += 32) {
    const int c = c0 + lane;
    if (c < C) dot += q[i * C + c] * g[i * C + c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  for (int c0 = 0; c0 < C; c0 += 32) {
    const int c = c0 + lane;
    if (c >= C) continue;
    const float d = q[i * C + c] * (g[i * C + c] - dot);
    if (da) da[i * C + c] = d;
    acc[i * C + c] = first ? d : acc[i * C + c] + d;
  }
}

__global__ void k_axpy(const float* __restrict__ x, int64_t n, float* __restrict__ y, int first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = first ? x[i] : y[i] + x[i];
}

}  // namespace
}  // namespace mk

// Backpropagation through the N mean-field iterations (Eq. 5).  The forward is
// recomputed with every Q^n kept (fp32, (N + 1) n C floats of workspace); then, from
// n = N down to 1: dA^n = softmax'(Q^n) dQ^n, dphi_u += dA^n, dW += G-weighted wgrad of the
// iteration's conv (dA^n against Q^(n-1)), dQ^(n-1) = dgrad of the conv; finally
// dphi_u += softmax'(Q^0) dQ^0 (Q^0 = softmax(phi_u), reading R25).
extern "C" mk_status mk_crf_backward(mk_context* ctx, const mk_kmap* m, const float* d_phi_u, const float* d_W,
                                     int32_t C, int32_t n_iters, const float* d_gq, float* d_gphi, float* d_gW,
                                     void* stream) {
  using namespace mk;
  clear_error();
  if (!ctx || !m) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_crf_backward: null argument");
  if (m->n_in != m->n_out || m->transposed)
    MK_FAIL(MK_ERR_SHAPE_MISMATCH, "mk_crf_backward: the map must connect a coordinate set to itself");
  if (C < 1 || n_iters < 0) MK_FAIL(MK_ERR_SHAPE_MISMATCH, "mk_crf_backward: bad sizes");
  const int64_t n = m->n_out, wn = (int64_t)m->K * C * C;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_iters > 0 && (!d_W || !d_gW)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_crf_backward: null weights");
  if (n == 0) {
    if (n_iters > 0) MK_CUDA_TRY(cudaMemsetAsync(d_gW, 0, sizeof(float) * wn, s));
    return MK_OK;
  }
  if (!d_phi_u || !d_gq || !d_gphi) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_crf_backward: null buffers");
  const int64_t nc = n * C;
  // workspace: Q^0..Q^N, the conv output / dA, two dQ buffers, one dW partial
  float* ws = (float*)dev_alloc(ctx->alloc, sizeof(float) * ((n_iters + 1) * nc + 3 * nc + wn), s);
  if (!ws) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "mk_crf_backward: workspace allocation failed");
  float* Q = ws;
  float* tmp = Q + (n_iters + 1) * nc;
  float* dq[2] = {tmp + nc, tmp + 2 * nc};
  float* gw_tmp = tmp + 3 * nc;
  const unsigned grid = (unsigned)ceil_div(n, 8);
  const NbrView v = forward_view(m);
  mk_status st = MK_OK;
  k_crf_softmax<<<grid, 256, 0, s>>>(d_phi_u, nullptr, n, C, Q);  // Q^0
  g_launches++;
  // C <= 32: the fused group-per-node kernels of mk_crf_infer (conv + softmax forward,
  // transposed-weight conv backward); larger C: the generic FFMA conv
  const size_t fsmem = sizeof(float) * ((size_t)v.K * C * C + 256 * 32);
  const bool fused = C <= 32 && fsmem <= 48 * 1024;
  int Cp = 1;
  while (Cp < C) Cp <<= 1;
  const unsigned g2 = (unsigned)std::min<int64_t>(ceil_div(ceil_div(n, 32 / Cp), 8), 6 * ctx->num_sms);
  for (int it = 0; it < n_iters && st == MK_OK; ++it) {
    if (fused) {
      k_crf_step<true><<<g2, 256, fsmem, s>>>(v, n, d_phi_u, Q + it * nc, d_W, C, Cp, Q + (it + 1) * nc, 0);
      g_launches++;
      continue;
    }
    st = launch_conv_f32(v, Q + it * nc, C, d_W, C, C, tmp, C, MK_F32, n, false, s);
    if (st == MK_OK) {
      k_crf_softmax<<<grid, 256, 0, s>>>(d_phi_u, tmp, n, C, Q + (it + 1) * nc);
      g_launches++;
    }
  }
  cudaError_t e = cudaMemcpyAsync(dq[0], d_gq, sizeof(float) * nc, cudaMemcpyDeviceToDevice, s);
  const unsigned wgrid = (unsigned)std::min<int64_t>(ceil_div(wn, 256), 4 * ctx->num_sms);
  for (int it = n_iters; it >= 1 && st == MK_OK && e == cudaSuccess; --it) {
    float* g_cur = dq[(n_iters - it) & 1];
    float* g_prev = dq[(n_iters - it + 1) & 1];
    k_crf_softmax_bwd<<<grid, 256, 0, s>>>(Q + it * nc, g_cur, n, C, tmp, d_gphi, it == n_iters);
    g_launches++;
    // dQ^(it-1) = conv dgrad of dA; dW_it = wgrad(dA, Q^(it-1))
    if (fused) {
      k_crf_step<false><<<g2, 256, fsmem, s>>>(dgrad_view(m), n, nullptr, tmp, d_W, C, Cp, g_prev, 1);
      g_launches++;
      st = mk_conv_backward(ctx, m, tmp, Q + (it - 1) * nc, d_W, C, C, MK_F32, nullptr, gw_tmp, stream);
    } else {
      st = mk_conv_backward(ctx, m, tmp, Q + (it - 1) * nc, d_W, C, C, MK_F32, g_prev, gw_tmp, stream);
    }
    if (st == MK_OK) {
      k_axpy<<<wgrid, 256, 0, s>>>(gw_tmp, wn, d_gW, it == n_iters);
      g_launches++;
    }
  }
  if (st == MK_OK && e == cudaSuccess) {
    k_crf_softmax_bwd<<<grid, 256, 0, s>>>(Q, dq[n_iters & 1], n, C, nullptr, d_gphi, n_iters == 0);
    g_launches++;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  dev_free(ctx->alloc, ws, s);
  if (st != MK_OK) return st;
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("mk_crf_backward: ") + cudaGetErrorString(e));
  return MK_OK;
}
