// crf.cu — mean-field inference of the trilateral stationary CRF (TS-CRF, SURVEY §8(f) f3;
// Alg. 5 and Eq. 4) on a 7D space-time-chroma kernel map:
//   Q^0 = softmax(phi_u)                                   (reading R25)
//   for n = 1..N:  Q~^n = generalized sparse conv(Q^(n-1); phi_p)   (the pairwise sum of
//                  Eq. 4 is a 7D sparse convolution because phi_p is stationary)
//                  Q^n  = softmax(phi_u + Q~^n)
// The convolution is the exact-FFMA fp32 kernel of conv_simt.cu (channels = classes: tiny
// dense products, memory bound); the softmax is one warp per node.
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
