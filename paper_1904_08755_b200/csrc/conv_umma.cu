// conv_umma.cu — bf16 tcgen05 gather-GEMM kernels (placeholder until the tensor-core path lands).
#include "conv.cuh"

namespace mk {
mk_status launch_conv_bf16(mk_context*, const NbrView&, const void*, int, const void*, int, int, void*, int, mk_dtype,
                           int64_t, bool, cudaStream_t) {
  MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 tensor-core conv not built yet");
}
mk_status launch_wgrad_bf16(mk_context*, const mk_kmap*, const void*, int, const void*, int, float*, cudaStream_t) {
  MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 tensor-core wgrad not built yet");
}
}  // namespace mk
