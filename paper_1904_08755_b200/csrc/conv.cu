// conv.cu — entry points of the generalized sparse convolution (Alg. 2), its
// reverse mode, and the transposed convolution.  Validation and dispatch only:
// bf16 -> tcgen05 tensor cores (conv_umma.cu); fp32 -> the same tensor cores on three-way
// bf16 splits of the operands (conv_split.cu) when the channel counts suit them, else (and
// with MK_F32_MODE=exact) exact FFMA kernels (conv_simt.cu).
#include <algorithm>

#include "conv.cuh"

namespace mk {
namespace {

mk_status check_common(mk_context* ctx, const mk_kmap* m, int32_t c_in, int32_t c_out, mk_dtype dt) {
  if (!ctx || !m) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "conv: null context or map");
  if (c_in < 1 || c_out < 1) MK_FAIL(MK_ERR_SHAPE_MISMATCH, "conv: channel counts must be >= 1");
  if (dt != MK_F32 && dt != MK_BF16) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "conv: unknown dtype");
  if (c_in > 256 || c_out > 256) MK_FAIL(MK_ERR_UNSUPPORTED, "conv: channel counts above 256");
  if (dt == MK_BF16 && (c_in % 16 != 0 || c_out % 16 != 0))
    MK_FAIL(MK_ERR_UNSUPPORTED, "conv: bf16 tensor-core path needs channel counts that are multiples of 16");
  return MK_OK;
}

mk_status forward_impl(mk_context* ctx, const mk_kmap* m, const void* d_fin, int32_t c_in, const void* d_w,
                       void* d_fout, int32_t c_out, mk_dtype in_dt, mk_dtype out_dt, cudaStream_t s,
                       const Epilogue& ep = Epilogue()) {
  mk_status st = check_common(ctx, m, c_in, c_out, in_dt);
  if (st != MK_OK) return st;
  if (out_dt != MK_F32 && out_dt != MK_BF16) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "conv: unknown output dtype");
  if (m->n_out > 0 && !d_fout) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "conv: null output");
  if (m->n_in > 0 && m->n_out > 0 && (!d_fin || !d_w)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "conv: null input or weights");
  if (m->n_out == 0) return MK_OK;
  const NbrView v = forward_view(m);
  if (in_dt == MK_F32 && split_f32_enabled(c_in, c_out, m->K, ep))
    return launch_conv_f32_split(ctx, v, (const float*)d_fin, m->n_in, c_in, (const float*)d_w, c_in, c_out, d_fout,
                                 c_out, out_dt, m->n_out, false, s);
  if (in_dt == MK_F32)
    return launch_conv_f32(v, (const float*)d_fin, c_in, (const float*)d_w, c_in, c_out, d_fout, c_out, out_dt,
                           m->n_out, false, s, ep);
  return launch_conv_bf16(ctx, v, d_fin, m->n_in, c_in, d_w, c_in, c_out, d_fout, c_out, out_dt, m->n_out, false, s,
                          ep);
}

mk_status backward_impl(mk_context* ctx, const mk_kmap* m, const void* d_gout, const void* d_fin, const void* d_w,
                        int32_t c_in, int32_t c_out, mk_dtype dt, void* d_gin, float* d_gw, cudaStream_t s) {
  mk_status st = check_common(ctx, m, c_in, c_out, dt);
  if (st != MK_OK) return st;
  if (m->n_out > 0 && m->n_in > 0 && !d_gout) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "conv backward: null grad_out");
  if (d_gin && m->n_in > 0) {
    if (m->n_out > 0 && !d_w) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "conv backward: null weights");
    const NbrView v = dgrad_view(m);
    if (dt == MK_F32 && split_f32_enabled(c_in, c_out, m->K, Epilogue()))
      st = launch_conv_f32_split(ctx, v, (const float*)d_gout, m->n_out, c_out, (const float*)d_w, c_in, c_out, d_gin,
                                 c_in, MK_F32, m->n_in, true, s);
    else if (dt == MK_F32)
      st = launch_conv_f32(v, (const float*)d_gout, c_out, (const float*)d_w, c_in, c_out, d_gin, c_in, MK_F32,
                           m->n_in, true, s);
    else
      st = launch_conv_bf16(ctx, v, d_gout, m->n_out, c_out, d_w, c_in, c_out, d_gin, c_in, MK_BF16, m->n_in, true, s);
    if (st != MK_OK) return st;
  }
  if (d_gw) {
    if (m->n_out > 0 && m->n_in > 0 && !d_fin) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "conv backward: null input features");
    if (dt == MK_F32 && split_f32_enabled(c_in, c_out, m->K, Epilogue())) {
      st = launch_wgrad_f32_split(ctx, m, (const float*)d_gout, c_out, (const float*)d_fin, c_in, d_gw, s);
    } else if (dt == MK_F32) {
      st = kmap_host(m);  // per-offset pair counts on the host (waits for the build only)
      if (st != MK_OK) return st;
      // split-K plan: chunks of <= P pairs per offset, P = 4096 or smaller so that the grid has
      // about 4 chunks per SM (small maps / few channels: a 7D CRF map has 600k pairs of 16 ch)
      int64_t P = 4096;
      while (P > 256 && m->h_ptr[m->K] / P < 4 * (int64_t)ctx->num_sms) P >>= 1;
      std::vector<int4> chunks;
      std::vector<int32_t> begin(m->K + 1, 0);
      for (int k = 0; k < m->K; ++k) {
        begin[k] = (int32_t)chunks.size();
        for (int64_t b = m->h_ptr[k]; b < m->h_ptr[k + 1]; b += P)
          chunks.push_back(make_int4(k, (int)b, (int)std::min(b + P, m->h_ptr[k + 1]), (int)chunks.size()));
      }
      begin[m->K] = (int32_t)chunks.size();
      WgradPlan plan;
      plan.n_chunks = (int64_t)chunks.size();
      const size_t part_bytes = sizeof(float) * std::max<int64_t>(1, plan.n_chunks) * c_out * c_in;
      char* ws = (char*)dev_alloc(ctx->alloc, part_bytes + sizeof(int4) * (chunks.size() + 1) + 256 +
                                                sizeof(int32_t) * (m->K + 1), s);
      if (!ws) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "conv backward: workspace allocation failed");
      plan.part = (float*)ws;
      plan.chunks = (int4*)(ws + ((part_bytes + 255) & ~size_t(255)));
      plan.chunk_begin = (int32_t*)(plan.chunks + chunks.size() + 1);
      cudaError_t e = cudaSuccess;
      if (!chunks.empty())
        e = cudaMemcpyAsync(plan.chunks, chunks.data(), sizeof(int4) * chunks.size(), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(plan.chunk_begin, begin.data(), sizeof(int32_t) * (m->K + 1), cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) {
        dev_free(ctx->alloc, ws, s);
        MK_FAIL(MK_ERR_CUDA, std::string("conv backward: ") + cudaGetErrorString(e));
      }
      st = launch_wgrad_f32(m, plan, (const float*)d_gout, c_out, (const float*)d_fin, c_in, d_gw, s);
      // pageable H2D copies above are staged synchronously, so host vectors may go out of scope
      dev_free(ctx->alloc, ws, s);
    } else {
      st = launch_wgrad_bf16(ctx, m, d_gout, c_out, d_fin, c_in, d_gw, s);
    }
  }
  return st;
}

}  // namespace
}  // namespace mk

using namespace mk;

extern "C" {

mk_status mk_conv_forward(mk_context* ctx, const mk_kmap* m, const void* d_fin, int32_t c_in, const void* d_w,
                          void* d_fout, int32_t c_out, mk_dtype in_dt, mk_dtype out_dt, void* stream) {
  clear_error();
  return forward_impl(ctx, m, d_fin, c_in, d_w, d_fout, c_out, in_dt, out_dt, (cudaStream_t)stream);
}

mk_status mk_conv_forward_fused(mk_context* ctx, const mk_kmap* m, const void* d_fin, int32_t c_in, const void* d_w,
                                void* d_fout, int32_t c_out, mk_dtype in_dt, mk_dtype out_dt, const float* d_scale,
                                const float* d_shift, const void* d_residual, int32_t relu, void* stream) {
  clear_error();
  Epilogue ep;
  ep.scale = d_scale;
  ep.shift = d_shift;
  ep.residual = d_residual;
  ep.relu = relu ? 1 : 0;
  return forward_impl(ctx, m, d_fin, c_in, d_w, d_fout, c_out, in_dt, out_dt, (cudaStream_t)stream, ep);
}

mk_status mk_conv_backward(mk_context* ctx, const mk_kmap* m, const void* d_gout, const void* d_fin,
                           const void* d_w, int32_t c_in, int32_t c_out, mk_dtype dt, void* d_gin, float* d_gw,
                           void* stream) {
  clear_error();
  HostTimer ht("conv_backward");
  const mk_status st = backward_impl(ctx, m, d_gout, d_fin, d_w, c_in, c_out, dt, d_gin, d_gw, (cudaStream_t)stream);
  ht.mark("impl");
  return st;
}

mk_status mk_conv_transpose_forward(mk_context* ctx, const mk_kmap* m, const void* d_fin, int32_t c_in,
                                    const void* d_w, void* d_fout, int32_t c_out, mk_dtype in_dt, mk_dtype out_dt,
                                    void* stream) {
  clear_error();
  if (m && !m->transposed) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_conv_transpose_forward: map is not transposed");
  return forward_impl(ctx, m, d_fin, c_in, d_w, d_fout, c_out, in_dt, out_dt, (cudaStream_t)stream);
}

mk_status mk_conv_transpose_backward(mk_context* ctx, const mk_kmap* m, const void* d_gout, const void* d_fin,
                                     const void* d_w, int32_t c_in, int32_t c_out, mk_dtype dt, void* d_gin,
                                     float* d_gw, void* stream) {
  clear_error();
  if (m && !m->transposed) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_conv_transpose_backward: map is not transposed");
  return backward_impl(ctx, m, d_gout, d_fin, d_w, c_in, c_out, dt, d_gin, d_gw, (cudaStream_t)stream);
}

}  // extern "C"
