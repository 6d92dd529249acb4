// ubench_gather.cu — B200 micro-benchmark of random 128-byte row gathers (the conv
// kernels' access pattern): LDG.128 to registers, cp.async to shared memory, and TMA
// tile::gather4, at several in-flight depths.  Development tool (not part of libmk).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1904_08755_b200/csrc ubench_gather.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace mk::sm100;

// each warp gathers rows idx[base..]: 8 lanes per 128-byte row, 4 rows per instruction
template <int U>
__global__ void k_ldg(const uint4* __restrict__ tab, const int* __restrict__ idx, int n_idx, uint4* out) {
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int b = wid * 4 * U; b < n_idx; b += nw * 4 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = b + u * 4 + lane / 8;
      v[u] = r < n_idx ? __ldg(tab + (size_t)__ldg(idx + r) * 8 + (lane & 7)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc.x ^= v[u].x, acc.y ^= v[u].y, acc.z ^= v[u].z, acc.w ^= v[u].w;
  }
  if (acc.x == 0x12345678) out[0] = acc;
}

// 128 threads per CTA; a stage = 128 rows (16 KB); `lag` groups in flight per thread
__global__ void k_cpasync(const uint4* __restrict__ tab, const int* __restrict__ idx, int n_idx, int lag,
                          uint4* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int t = threadIdx.x;
  const int S = 8;
  int g = 0;
  for (int b = blockIdx.x * 128; b < n_idx; b += gridDim.x * 128, ++g) {
    const uint32_t st = smem_u32(sm + (g % S) * 16384);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = i * 16 + t / 8;
      const int row = b + r < n_idx ? __ldg(idx + b + r) : 0;
      cp_async16(st + r * 128 + (t & 7) * 16, tab + (size_t)row * 8 + (t & 7), 16);
    }
    cp_async_commit();
    cp_async_wait_n(lag);
  }
  cp_async_wait_n(0);
  __syncthreads();
  if (((uint32_t*)sm)[t] == 0x12345678) out[0] = make_uint4(1, 1, 1, 1);
}

// cp.async, warp-per-stage: each warp gathers whole 128-row stages into its own slot,
// waits for them (wait_group 0) and moves on — the conv kernel's producer pattern.
__global__ void k_cpasync_warp(const uint4* __restrict__ tab, const int* __restrict__ idx, int n_idx, uint4* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t st = smem_u32(sm + (warp % 12) * 16384);
  for (int b = (blockIdx.x * nw + warp) * 128; b < n_idx; b += gridDim.x * nw * 128) {
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const int r = i * 4 + lane / 8;
      const int row = b + r < n_idx ? __ldg(idx + b + r) : 0;
      cp_async16(st + r * 128 + (lane & 7) * 16, tab + (size_t)row * 8 + (lane & 7), 16);
    }
    cp_async_commit();
    cp_async_wait_n(0);
  }
  __syncthreads();
  if (((uint32_t*)sm)[threadIdx.x] == 0x12345678) out[0] = make_uint4(1, 1, 1, 1);
}

// LDG -> STS register staging, warp-per-stage
__global__ void k_ldgsts_warp(const uint4* __restrict__ tab, const int* __restrict__ idx, int n_idx, uint4* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint4* st = (uint4*)(sm + (warp % 12) * 16384);
  for (int b = (blockIdx.x * nw + warp) * 128; b < n_idx; b += gridDim.x * nw * 128) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      uint4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = (h * 8 + i) * 4 + lane / 8;
        const int row = b + r < n_idx ? __ldg(idx + b + r) : 0;
        v[i] = __ldg(tab + (size_t)row * 8 + (lane & 7));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) st[((h * 8 + i) * 4 + lane / 8) * 8 + (lane & 7)] = v[i];
    }
    __syncwarp();
  }
  __syncthreads();
  if (((uint32_t*)sm)[threadIdx.x] == 0x12345678) out[0] = make_uint4(1, 1, 1, 1);
}

// TMA gather4 where `lanes` lanes of every warp issue (warp-per-stage, mbarrier per warp)
__global__ void k_tma_lanes(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, int n_idx, int lanes,
                            uint4* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) mbar_init(&bar[warp], 1);
  fence_mbar_init();
  __syncthreads();
  const uint32_t st = smem_u32(sm + (warp % 12) * 16384);
  uint32_t ph = 0;
  for (int b = (blockIdx.x * nw + warp) * 128; b < n_idx; b += gridDim.x * nw * 128) {
    if (lane == 0) mbar_arrive_expect_tx(&bar[warp], 128 * 128);
    __syncwarp();
    if (lane < lanes) {
      for (int q = lane; q < 32; q += lanes) {
        const int r0 = b + q * 4;
        int4 rr;
        rr.x = r0 < n_idx ? __ldg(idx + r0) : -1;
        rr.y = r0 + 1 < n_idx ? __ldg(idx + r0 + 1) : -1;
        rr.z = r0 + 2 < n_idx ? __ldg(idx + r0 + 2) : -1;
        rr.w = r0 + 3 < n_idx ? __ldg(idx + r0 + 3) : -1;
        tma_gather4(st + q * 512, &tm, 0, rr, &bar[warp]);
      }
    }
    mbar_wait(&bar[warp], ph);
    ph ^= 1;
  }
  __syncthreads();
  if (((uint32_t*)sm)[threadIdx.x] == 0x12345678) out[0] = make_uint4(1, 1, 1, 1);
}

// TMA gather4: `nthr` issuing threads (one per warp) each gather 128/nthr rows of a stage
__global__ void k_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, int n_idx, int nthr,
                      int depth, uint4* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = (uint64_t*)(sm + 8 * 16384);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) mbar_init(bar + s, nthr);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp < nthr && lane == 0) {
    int g = 0;
    const int rows = 128 / nthr;
    for (int b = blockIdx.x * 128; b < n_idx; b += gridDim.x * 128, ++g) {
      const int s = g % 8;
      if (g >= depth) mbar_wait(bar + ((g - depth) % 8), ((g - depth) / 8) & 1);
      mbar_arrive_expect_tx(bar + s, rows * 128);
      for (int q = 0; q < rows; q += 4) {
        const int r0 = b + warp * rows + q;
        int4 rr;
        rr.x = r0 < n_idx ? idx[r0] : -1;
        rr.y = r0 + 1 < n_idx ? idx[r0 + 1] : -1;
        rr.z = r0 + 2 < n_idx ? idx[r0 + 2] : -1;
        rr.w = r0 + 3 < n_idx ? idx[r0 + 3] : -1;
        tma_gather4(smem_u32(sm + s * 16384 + (warp * rows + q) * 128), &tm, 0, rr, bar + s);
      }
    }
    for (int h = (g > depth ? g - depth : 0); h < g; ++h) mbar_wait(bar + (h % 8), (h / 8) & 1);
  }
  __syncthreads();
  if (((uint32_t*)sm)[threadIdx.x] == 0x12345678) out[0] = make_uint4(1, 1, 1, 1);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int N = 150000, M = 1400000;
  uint4* tab;
  int* idx;
  uint4* out;
  cudaMalloc(&tab, (size_t)N * 128);
  cudaMemset(tab, 1, (size_t)N * 128);
  cudaMalloc(&idx, M * 4);
  cudaMalloc(&out, 64);
  std::vector<int> h(M);
  srand(1);
  for (int i = 0; i < M; ++i) h[i] = (int)(((unsigned long long)rand() * 2654435761ull) % N);
  cudaMemcpy(idx, h.data(), M * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)M * 128;
  auto timeit = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-34s %8.1f us  %7.2f TB/s  (%s)\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  };
  char nm[64];
  for (int blocks : {148, 592})
    for (int u : {4}) {
      snprintf(nm, 64, "ldg U=%d grid=%d x256", u, blocks);
      if (u == 1) timeit(nm, [&] { k_ldg<1><<<blocks, 256>>>(tab, idx, M, out); });
      if (u == 4) timeit(nm, [&] { k_ldg<4><<<blocks, 256>>>(tab, idx, M, out); });
      if (u == 8) timeit(nm, [&] { k_ldg<8><<<blocks, 256>>>(tab, idx, M, out); });
    }
  cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  for (int blocks : {148})
    for (int lag : {3}) {
      snprintf(nm, 64, "cp.async lag=%d grid=%d x128", lag, blocks);
      timeit(nm, [&] { k_cpasync<<<blocks, 128, 8 * 16384>>>(tab, idx, M, lag, out); });
    }
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, (cuuint64_t)N}, str[1] = {128};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  ((EncFn)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tab, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int big = 12 * 16384;
  cudaFuncSetAttribute(k_cpasync_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_ldgsts_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_tma_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  for (int warps : {4, 8, 12, 16, 24, 32}) {
    snprintf(nm, 64, "cp.async warp-stage warps=%d", warps);
    timeit(nm, [&] { k_cpasync_warp<<<148, warps * 32, big>>>(tab, idx, M, out); });
    snprintf(nm, 64, "ldg->sts warp-stage warps=%d", warps);
    timeit(nm, [&] { k_ldgsts_warp<<<148, warps * 32, big>>>(tab, idx, M, out); });
    for (int lanes : {1, 4, 32}) {
      snprintf(nm, 64, "tma gather4 warps=%d lanes=%d", warps, lanes);
      timeit(nm, [&] { k_tma_lanes<<<148, warps * 32, big>>>(tm, idx, M, lanes, out); });
    }
  }
  return 0;
}
