// ubench_rowseg.cu — random-row gather bandwidth (cp.async 16 B, L2-resident table) as a
// function of the table's row pitch S and the bytes G gathered per row (one contiguous
// segment at offset OFF of the row), with the lanes of a warp instruction taking consecutive
// 16-byte chunks of the stage's (row, chunk) list.  Question it answers: is the gather rate
// bound by bytes, by 16-byte requests (instructions), or by the 128-byte lines each
// instruction touches?  (The conv kernels gather 64-byte chunks of 192-byte rows at C = 96.)
// Every warp keeps D + 1 stages of ~16 KB in flight-or-landing (wait_group D).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1904_08755_b200/csrc ubench_rowseg.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace mk::sm100;

constexpr int kStage = 6144;  // bytes per stage (32 rows of 192 B, 48 of 128 B, 96 of 64 B)

__global__ void k_g(const uint8_t* __restrict__ tab, const int* __restrict__ idx, int stages_per_warp, int D, int S,
                    int G, int OFF, long long* issue_cycles, uint4* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int slots = D + 1;
  int (*sidx)[2][256] = (int (*)[2][256])(sm + nw * slots * kStage);  // [warps][2][256] row indices
  const uint32_t base = smem_u32(sm) + warp * slots * kStage;
  const int cpr = G / 16;              // 16-byte chunks per row
  const int NR = kStage / G;           // rows per stage
  const int nch = NR * cpr;            // chunks per stage
  long long t_issue = 0;
  const int gw = blockIdx.x * nw + warp;
  auto load_idx = [&](int st, int b) {
    const int* ix = idx + ((size_t)gw * stages_per_warp + st) * 256;
    for (int i = lane; i < NR; i += 32) sidx[warp][b][i] = __ldg(ix + i);
  };
  load_idx(0, 0);
  __syncwarp();
  for (int st = 0; st < stages_per_warp; ++st) {
    const uint32_t dst = base + (st % slots) * kStage;
    const int b = st & 1;
    // next stage's indices (plain loads; they land while this stage's copies are issued)
    int nx[8];
    const int* ixn = idx + ((size_t)gw * stages_per_warp + st + 1) * 256;
#pragma unroll
    for (int j = 0; j < 8; ++j) nx[j] = (st + 1 < stages_per_warp && lane + 32 * j < NR) ? __ldg(ixn + lane + 32 * j) : 0;
    const long long t0 = clock64();
    int q = lane;
    int row = q / cpr, c = q - row * cpr;
    const int drow = 32 / cpr, dc = 32 - drow * cpr;
    for (; q < nch; q += 32) {
      const int r = sidx[warp][b][row];
      cp_async16(dst + q * 16, tab + (size_t)r * S + OFF + c * 16, 16u);
      row += drow;
      c += dc;
      if (c >= cpr) {
        c -= cpr;
        ++row;
      }
    }
    cp_async_commit();
    t_issue += clock64() - t0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (lane + 32 * j < NR) sidx[warp][b ^ 1][lane + 32 * j] = nx[j];
    cp_async_wait_n(D);
    __syncwarp();
  }
  cp_async_wait_n(0);
  __syncthreads();
  if (lane == 0) issue_cycles[blockIdx.x * nw + warp] = t_issue;
  if (((uint32_t*)sm)[threadIdx.x] == 0x12345678) out[0] = make_uint4(1, 1, 1, 1);
}

int main() {
  const int sm = 148;
  const size_t tab_bytes = 40u << 20;  // 40 MB: L2-resident
  uint8_t* tab;
  cudaMalloc(&tab, tab_bytes);
  cudaMemset(tab, 1, tab_bytes);
  const int max_stages = 6000000 / 24 + 2 * 148 * 32;  // stages of all warps, any case (>= 24 rows each)
  std::vector<int> h((size_t)max_stages * 256);
  int* idx;
  cudaMalloc(&idx, sizeof(int) * h.size());
  long long* ic;
  cudaMalloc(&ic, 148 * 32 * 8);
  uint4* out;
  cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k_g, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case {
    int S, G, OFF;
  };
  // (pitch, gathered bytes, offset): C = 96 chunks of 32 ch (64 B at 0 / 64 / 128), whole
  // 192-byte rows, C = 64 rows (128 B), C = 128 rows (256 B), 64-byte chunks of 128-byte rows
  const Case cases[] = {{192, 64, 0}, {192, 64, 64}, {192, 192, 0}, {128, 128, 0}, {256, 256, 0}, {128, 64, 0},
                        {256, 128, 0}, {192, 128, 0}};
  for (const Case& cs : cases) {
    const int n_rows = (int)(tab_bytes / cs.S);
    srand(1);
    for (auto& v : h) v = rand() % n_rows;
    cudaMemcpy(idx, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice);
    for (int W : {8, 16, 24}) {
      for (int D : {0, 1}) {
        if ((D + 1) * W * kStage + W * 2048 > 200 * 1024) continue;
        const int spw = 6000000 / (kStage / cs.G) / (sm * W);  // ~6 M rows in total
        const int smem = (D + 1) * W * kStage + W * 2 * 256 * 4;
        k_g<<<sm, W * 32, smem>>>(tab, idx, spw, D, cs.S, cs.G, cs.OFF, ic, out);
        cudaEventRecord(e0);
        k_g<<<sm, W * 32, smem>>>(tab, idx, spw, D, cs.S, cs.G, cs.OFF, ic, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> hc(sm * W);
        cudaMemcpy(hc.data(), ic, 8 * sm * W, cudaMemcpyDeviceToHost);
        double mi = 0;
        for (auto v : hc) mi += v;
        mi /= hc.size() * spw;
        const double rows = (double)sm * W * spw * (kStage / cs.G);
        const double bytes = rows * cs.G;
        // 128-byte lines touched per row by the segment [OFF + r*S, +G)
        double lines = 0;
        for (int r = 0; r < 8; ++r) {
          const long a = (long)r * cs.S + cs.OFF, e = a + cs.G - 1;
          lines += (e / 128 - a / 128 + 1) / 8.0;
        }
        printf("S=%3d G=%3d off=%3d warps/SM=%2d D=%d: %7.1f us %6.2f TB/s %6.2f Grows/s %6.2f Glines/s  issue %6.0f cyc/stage (%s)\n",
               cs.S, cs.G, cs.OFF, W, D, ms * 1e3, bytes / (ms * 1e-3) / 1e12, rows / (ms * 1e-3) / 1e9,
               rows * lines / (ms * 1e-3) / 1e9, mi, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
