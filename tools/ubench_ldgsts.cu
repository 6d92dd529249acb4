// ubench_ldgsts.cu — random 128-byte row gathers by warps issuing 16 KB cp.async stages with
// the row indices already in registers: bandwidth vs issuing warps per SM, and the cost of
// the zero-fill (src-size) form (mode bit 4), the SW128 destination swizzle (mode bit 2) and
// a cp.async.mbarrier.arrive.noinc per stage.  Each warp gathers 16 KB stages (128 random 128-byte rows of a 19 MB table) into
// its own ring of D+1 smem slots, keeping D stages in flight (wait_group D), optionally
// with one noinc arrival per stage on a per-warp mbarrier.  Development tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1904_08755_b200/csrc ubench_ldgsts.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace mk::sm100;

// mode bits: 1 = indices from shared memory (LDS.128, 4 per lane group) instead of registers,
// 2 = swizzled destination, 4 = zero-fill form (src-size operand), 8 = runtime row stride
__global__ void k_g(const uint4* __restrict__ tab, const int* __restrict__ idx, int stages_per_warp, int D, int noinc,
                    int mode, int stride16, long long* issue_cycles, uint4* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[32];
  __shared__ __align__(16) int sidx[16][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) mbar_init(&bar[warp], 32);
  fence_mbar_init();
  __syncthreads();
  const int slots = D + 1;
  const uint32_t base = smem_u32(sm) + warp * slots * 16384;
  long long t_issue = 0;
  uint32_t ph = 0;
  const int gw = blockIdx.x * nw + warp;
  const int q4 = lane >> 3, jj = lane & 7;
  for (int st = 0; st < stages_per_warp; ++st) {
    const uint32_t dst = base + (st % slots) * 16384;
    const int* ix = idx + ((size_t)gw * stages_per_warp + st) * 128;
    int rows[32];
    if (mode & 1) {
      reinterpret_cast<int4*>(sidx[warp])[lane] = __ldg(reinterpret_cast<const int4*>(ix) + lane);
      __syncwarp();
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) rows[i] = __ldg(ix + i * 4 + lane / 8);
      if (rows[0] == -7) out[1] = make_uint4(0, 0, 0, 0);
    }
    long long t0 = clock64();
    if (mode & 1) {
#pragma unroll 2
      for (int i = 0; i < 32; i += 4) {
        const int4 a4 = *(const int4*)(&sidx[warp][q4 * 32 + i]);
        const int av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = q4 * 32 + i + e;
          const uint32_t d = (mode & 2) ? dst + swz(r, jj, 128) : dst + r * 128 + jj * 16;
          const uint4* src = (mode & 8) ? tab + (int64_t)max(av[e], 0) * stride16 + jj : tab + (size_t)av[e] * 8 + jj;
          if (mode & 4) cp_async16(d, src, av[e] >= 0 ? 16u : 0u);
          else cp_async16(d, src, 16u);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int r = i * 4 + lane / 8;
        const uint32_t d = (mode & 2) ? dst + swz(r, jj, 128) : dst + r * 128 + jj * 16;
        if (mode & 4) cp_async16(d, tab + (size_t)rows[i] * 8 + jj, rows[i] >= 0 ? 16u : 0u);
        else cp_async16(d, tab + (size_t)rows[i] * 8 + jj, 16u);
      }
    }
    if (noinc) cp_async_arrive_noinc(&bar[warp]);
    cp_async_commit();
    t_issue += clock64() - t0;
    cp_async_wait_n(D);
    if (noinc && st >= D) {  // the arrival of stage st - D
      mbar_wait(&bar[warp], ph);
      ph ^= 1;
    }
  }
  cp_async_wait_n(0);
  __syncthreads();
  if (lane == 0) issue_cycles[blockIdx.x * nw + warp] = t_issue;
  if (((uint32_t*)sm)[threadIdx.x] == 0x12345678) out[0] = make_uint4(1, 1, 1, 1);
}

int main() {
  const int n_rows = 150000, sm = 148;
  uint4* tab;
  cudaMalloc(&tab, (size_t)n_rows * 128);
  cudaMemset(tab, 1, (size_t)n_rows * 128);
  const int max_idx = 148 * 32 * 64 * 128;
  std::vector<int> h(max_idx);
  srand(1);
  for (auto& v : h) v = rand() % n_rows;
  int* idx;
  cudaMalloc(&idx, sizeof(int) * max_idx);
  cudaMemcpy(idx, h.data(), sizeof(int) * max_idx, cudaMemcpyHostToDevice);
  long long* ic;
  cudaMalloc(&ic, 148 * 32 * 8);
  uint4* out;
  cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k_g, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case {
    int W, D, mode;
  };
  const Case cases[] = {{4, 0, 0}, {8, 0, 0}, {12, 0, 0}, {4, 1, 0}, {4, 1, 4}, {4, 1, 2}, {4, 1, 6}};
  for (const Case& cs : cases) {
    const int W = cs.W, D = cs.D, mode = cs.mode;
    for (int noinc = 0; noinc < 2; ++noinc) {
      const int spw = 1400000 / 128 / (sm * W);  // ~1.4M rows in total (a configs[1] conv)
      const int smem = (D + 1) * W * 16384;
      k_g<<<sm, W * 32, smem>>>(tab, idx, spw, D, noinc, mode, 8, ic, out);
      cudaEventRecord(e0);
      k_g<<<sm, W * 32, smem>>>(tab, idx, spw, D, noinc, mode, 8, ic, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> hc(sm * W);
      cudaMemcpy(hc.data(), ic, 8 * sm * W, cudaMemcpyDeviceToHost);
      double mi = 0;
      for (auto v : hc) mi += v;
      mi /= hc.size() * spw;
      const double bytes = (double)sm * W * spw * 16384;
      printf("warps/SM=%2d depth=%d mode=%d noinc=%d: %7.1f us %6.2f TB/s  issue %6.0f cycles/stage (%s)\n", W, D,
             mode, noinc, ms * 1e3, bytes / (ms * 1e-3) / 1e12, mi, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
