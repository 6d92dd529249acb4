#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
__global__ void k(int* p, int n, long a, long b, long c, long d, long e, long f) { if (threadIdx.x == 1000) p[0] = n + a + b + c + d + e + f; }
int main() {
  int* p; cudaMalloc(&p, 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaStreamSynchronize(s);
      auto t0 = std::chrono::steady_clock::now();
      const int N = 2000;
      for (int i = 0; i < N; ++i) {
        if (mode == 0) k<<<1177, 256, 0, s>>>(p, i, 1, 2, 3, 4, 5, 6);
        else {
          cudaLaunchConfig_t cfg = {}; cfg.gridDim = 1177; cfg.blockDim = 256; cfg.stream = s;
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at; cfg.numAttrs = mode == 2 ? 1 : 0;
          cudaLaunchKernelEx(&cfg, k, p, i, 1L, 2L, 3L, 4L, 5L, 6L);
        }
        if (i % 64 == 63) cudaStreamSynchronize(s);  // keep the queue short
      }
      auto t1 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(s);
      if (rep) printf("mode %d (%s): %.2f us per launch (incl. periodic syncs)\n", mode, mode == 0 ? "<<<>>>" : mode == 1 ? "LaunchKernelEx" : "LaunchKernelEx+PDL", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    }
  }
  // pure host API cost: single launch after an idle stream
  for (int mode = 0; mode < 3; ++mode) {
    double tot = 0; const int N = 200;
    for (int i = 0; i < N; ++i) {
      cudaStreamSynchronize(s);
      auto t0 = std::chrono::steady_clock::now();
      if (mode == 0) k<<<1177, 256, 0, s>>>(p, i, 1, 2, 3, 4, 5, 6);
      else {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = 1177; cfg.blockDim = 256; cfg.stream = s;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = mode == 2 ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k, p, i, 1L, 2L, 3L, 4L, 5L, 6L);
      }
      tot += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    }
    printf("idle-stream single launch mode %d: %.2f us\n", mode, tot / N);
  }
  return 0;
}
