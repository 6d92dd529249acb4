// ubench_umma_layout.cu — tcgen05.mma (kind::f16, M = 128, K = 16) throughput by operand
// layout: K-major SW128 / SW64 (the forward kernel at C = 64 / C = 96) and MN-major SW64 /
// SW128 panels (the weight gradient).  One CTA per SM, one thread issues UMMAs into 4
// rotating accumulators (no dependency between consecutive UMMAs), issued by warp 0 under
// elect.sync, a commit + wait every 8 or every 512 UMMAs.
// Development tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1904_08755_b200/csrc ubench_umma_layout.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace mk::sm100;

struct Case {
  const char* name;
  int mn_major;   // 0: K-major (rows = M or N, row bytes = rb along K); 1: MN-major panels
  int rb;         // row bytes of the swizzle atom (128 / 64 / 32)
  int N;
};

__global__ void __launch_bounds__(128, 1) k_umma(Case c, int iters, int per, long long* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {  // the whole warp runs the loop; elect.sync picks the issuing lane
    const uint32_t a = smem_u32(sm), b = a + 32768;
    const uint32_t code = c.rb == 128 ? 2u : c.rb == 64 ? 4u : 6u;
    uint64_t ad, bd;
    uint32_t kstep;
    if (!c.mn_major) {  // K-major: SBO = 8 rows x rb, K step = 32 bytes
      ad = smem_desc(a, 16, 8 * c.rb, code);
      bd = smem_desc(b, 16, 8 * c.rb, code);
      kstep = 2;
    } else {  // MN-major: panels of rb / 2 elements x 64 K rows; LBO = panel stride, SBO = 8 K rows
      const uint32_t panel = 64 * c.rb;
      ad = smem_desc(a, panel, 8 * c.rb, code);
      bd = smem_desc(b, panel, 8 * c.rb, code);
      kstep = (16 * c.rb) >> 4;
    }
    const uint32_t idesc = idesc_bf16(128, (uint32_t)c.N, (uint32_t)c.mn_major, (uint32_t)c.mn_major);
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          umma_f16(tbase + (uint32_t)((q & 3) * c.N), ad + (q & 3) * kstep, bd + (q & 3) * kstep, idesc, it > 0 || q >= 4);
      }
      __syncwarp();
      if ((it + 1) % per == 0 || it + 1 == iters) {  // commit + wait every `per` batches of 8
        if (elect_one()) umma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const Case cases[] = {{"K-major SW128", 0, 128, 96}, {"K-major SW64 ", 0, 64, 96}, {"K-major SW32 ", 0, 32, 96},
                        {"MN-major SW64 ", 1, 64, 96}, {"MN-major SW128", 1, 128, 96}, {"MN-major SW128 N=128", 1, 128, 128},
                        {"K-major SW128 N=64", 0, 128, 64}, {"MN-major SW64 N=64", 1, 64, 64}};
  const int iters = 2000;
  for (int per : {1, 64}) {
    printf("-- commit + wait every %d x 8 UMMAs\n", per);
    for (const Case& c : cases) {
      k_umma<<<148, 128, 100 * 1024>>>(c, iters, per, d);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> h(148);
      cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
      double m = 0;
      for (auto v : h) m += v;
      m /= 148.0 * iters * 8;
      printf("%-22s N=%3d: %6.1f cycles per UMMA (%s)\n", c.name, c.N, m, cudaGetErrorString(e));
    }
  }
  return 0;
}
