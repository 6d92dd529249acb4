// ubench_umma.cu — cost of issuing tcgen05.mma (kind::f16, M=128, K=16) from one thread for
// several N, with a commit + mbarrier round trip every `per` MMAs.  Development tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1904_08755_b200/csrc ubench_umma.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace mk::sm100;

__global__ void __launch_bounds__(128, 1) k_umma(int N, int iters, int per, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(&tslot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(128, N, 0, 0);
    const uint32_t a = smem_u32(sm), b = a + 16384;
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      for (int q = 0; q < per; ++q) {
        const uint64_t ad = smem_desc(a + (q & 3) * 32, 16, 1024, 2);
        const uint64_t bd = smem_desc(b + (q & 3) * 32, 16, 1024, 2);
        umma_f16(tbase, ad, bd, idesc, (it | q) ? 1u : 0u);
      }
      umma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

// same, but the commit does not wait (fire-and-forget pipeline, wait only at the end)
__global__ void __launch_bounds__(128, 1) k_umma_nowait(int N, int iters, int per, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(&tslot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(128, N, 0, 0);
    const uint32_t a = smem_u32(sm), b = a + 16384;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (it >= 8) mbar_wait(&bar[it & 7], ((it >> 3) - 1) & 1);
      for (int q = 0; q < per; ++q) {
        const uint64_t ad = smem_desc(a + (q & 3) * 32, 16, 1024, 2);
        const uint64_t bd = smem_desc(b + (q & 3) * 32, 16, 1024, 2);
        umma_f16(tbase, ad, bd, idesc, (it | q) ? 1u : 0u);
      }
      umma_commit(&bar[it & 7]);
    }
    for (int it = iters > 8 ? iters - 8 : 0; it < iters; ++it) mbar_wait(&bar[it & 7], (it >> 3) & 1);
    long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

// step = [wait on an already-complete mbarrier] [tcgen05 fence] 4 MMAs, commit every 4 steps
__global__ void __launch_bounds__(128, 1) k_steps(int N, int steps, int fence, int waitbar, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[3];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive(&bar[1]);  // phase 0 of bar[1] complete: waits on it return at once
    const uint32_t idesc = idesc_bf16(128, N, 0, 0);
    const uint64_t dhi = smem_desc(0, 16, 1024, 2);
    const uint32_t a0 = smem_u32(sm) >> 4, b0 = a0 + 1024;
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int st = 0; st < steps; ++st) {
      if (waitbar) mbar_wait(&bar[1], 0);
      if (fence) tc_fence_after();
      const uint32_t d = tbase + (st & 7) * 64;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) umma_f16(d, dhi | (uint64_t)(a0 + kk * 2), dhi | (uint64_t)(b0 + kk * 2), idesc, 1u);
      if ((st & 3) == 3) {
        umma_commit(&bar[0]);
      }
    }
    umma_commit(&bar[2]);  // tracks every prior MMA
    mbar_wait(&bar[2], 0);
    (void)ph;
    long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// variant: mode 0 = lane-0 branch, runtime descriptors (current kernels)
//          mode 1 = whole warp computes, elect.sync issues, runtime descriptors
//          mode 2 = lane-0 branch, descriptors fixed before the loop (no per-MMA arithmetic)
__global__ void __launch_bounds__(128, 1) k_issue(int steps, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const uint32_t idesc = idesc_bf16(128, 64, 0, 0);
  const uint64_t dhi = smem_desc(0, 16, 1024, 2);
  const uint32_t a0 = smem_u32(sm) >> 4;
  long long t0 = clock64();
  if (warp == 0) {
    if (mode == 1) {
      uint32_t s = 0;
      for (int st = 0; st < steps; ++st) {
        const uint32_t alo = a0 + s * 1024, blo = a0 + 512 + s * 512;
        uint32_t pred;
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
        if (pred) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16(tbase + (st & 7) * 64, dhi | (uint64_t)(alo + kk * 2), dhi | (uint64_t)(blo + kk * 2), idesc, 1u);
          if ((st & 15) == 15) umma_commit(&bar[0]);
        }
        __syncwarp();
        if (++s == 4) s = 0;
      }
    } else if (lane == 0) {
      if (mode == 0) {
        uint32_t s = 0;
        for (int st = 0; st < steps; ++st) {
          const uint32_t alo = a0 + s * 1024, blo = a0 + 512 + s * 512;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16(tbase + (st & 7) * 64, dhi | (uint64_t)(alo + kk * 2), dhi | (uint64_t)(blo + kk * 2), idesc, 1u);
          if ((st & 15) == 15) umma_commit(&bar[0]);
          if (++s == 4) s = 0;
        }
      } else {
        const uint64_t ad0 = dhi | a0, bd0 = dhi | (a0 + 512);
        for (int st = 0; st < steps; ++st) {
          umma_f16(tbase, ad0, bd0, idesc, 1u);
          umma_f16(tbase, ad0 + 2, bd0 + 2, idesc, 1u);
          umma_f16(tbase, ad0 + 4, bd0 + 4, idesc, 1u);
          umma_f16(tbase, ad0 + 6, bd0 + 6, idesc, 1u);
          if ((st & 15) == 15) umma_commit(&bar[0]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      umma_commit(&bar[1]);
      mbar_wait(&bar[1], 0);
      out[blockIdx.x] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// time the commit instruction itself: issue 16 MMAs, then commit, measuring each part
__global__ void __launch_bounds__(128, 1) k_commit(int rounds, int nmma, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(&tslot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(128, 64, 0, 0);
    const uint64_t ad0 = smem_desc(smem_u32(sm), 16, 1024, 2), bd0 = smem_desc(smem_u32(sm) + 8192, 16, 1024, 2);
    long long t_mma = 0, t_commit = 0;
    for (int r = 0; r < rounds; ++r) {
      long long a = clock64();
      for (int q = 0; q < nmma; ++q) umma_f16(tbase + (q & 3) * 64, ad0 + (q & 3) * 2, bd0 + (q & 3) * 2, idesc, 1u);
      long long b = clock64();
      umma_commit(&bar[r & 3]);
      long long c = clock64();
      t_mma += b - a;
      t_commit += c - b;
      if (r >= 3) mbar_wait(&bar[(r - 3) & 3], ((r - 3) >> 2) & 1);
    }
    out[blockIdx.x * 2] = t_mma / rounds;
    out[blockIdx.x * 2 + 1] = t_commit / rounds;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// several CTAs per SM, each: 4 UMMAs (M=128, N=64, K=16) + commit per step, waiting only for
// the commit 8 steps back.  Do commits from different CTAs drain each other's MMAs?
__global__ void __launch_bounds__(128) k_multi(int steps, int commit_every, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32768 / 4; i += 128) ((uint32_t*)sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(&tslot, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(128, 64, 0, 0);
    const uint64_t dhi = smem_desc(0, 16, 1024, 2);
    const uint32_t a0 = smem_u32(sm) >> 4, b0 = a0 + 1024;
    long long t0 = clock64();
    int nc = 0;
    for (int st = 0; st < steps; ++st) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) umma_f16(tbase, dhi | (uint64_t)(a0 + kk * 2), dhi | (uint64_t)(b0 + kk * 2), idesc, 1u);
      if ((st + 1) % commit_every == 0) {
        if (nc >= 8) mbar_wait(&bar[nc & 7], ((nc >> 3) - 1) & 1);
        umma_commit(&bar[nc & 7]);
        ++nc;
      }
    }
    for (int j = nc > 8 ? nc - 8 : 0; j < nc; ++j) mbar_wait(&bar[j & 7], (j >> 3) & 1);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 128);
}

int main() {
  {
    long long* dm;
    cudaMalloc(&dm, 148 * 4 * 8);
    std::vector<long long> hm(148 * 4);
    cudaFuncSetAttribute(k_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
    for (int per_sm : {1, 2, 3}) {
      for (int ce : {1, 2, 4}) {
        const int steps = 2048;
        const int smem = (227 * 1024) / per_sm - 4096;  // forces per_sm CTAs per SM at most
        cudaFuncSetAttribute(k_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_multi<<<148 * per_sm, 128, smem>>>(steps, ce, dm);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double mmas_per_sm = (double)per_sm * steps * 4;
        printf("CTAs/SM=%d commit every %d steps: %8.1f us  %6.1f cycles per UMMA per SM (%s)\n", per_sm, ce, ms * 1e3,
               ms * 1e-3 * 1.965e9 / mmas_per_sm, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  long long* d;
  cudaMalloc(&d, 148 * 8);
  long long h[148];
  cudaFuncSetAttribute(k_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_umma_nowait, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int nowait = 0; nowait < 2; ++nowait)
    for (int N : {64, 128, 256})
      for (int per : {1, 4, 16}) {
        const int iters = 2048 / per;
        if (nowait) k_umma_nowait<<<148, 128, 65536>>>(N, iters, per, d);
        else k_umma<<<148, 128, 65536>>>(N, iters, per, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mean = 0;
        for (int i = 0; i < 148; ++i) mean += h[i];
        mean /= 148;
        printf("%s N=%3d per=%2d: %7.1f cycles per MMA  (%s)\n", nowait ? "pipelined" : "wait-each", N, per,
               mean / (iters * per), cudaGetErrorString(cudaGetLastError()));
      }
  {
    long long* d2;
    cudaMalloc(&d2, 148 * 16);
    long long h2[296];
    cudaFuncSetAttribute(k_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int nmma : {1, 4, 16, 64}) {
      k_commit<<<148, 128, 65536>>>(64, nmma, d2);
      cudaDeviceSynchronize();
      cudaMemcpy(h2, d2, sizeof(h2), cudaMemcpyDeviceToHost);
      printf("commit probe nmma=%2d: issue %6lld cycles, commit instruction %6lld cycles (%s)\n", nmma, h2[0], h2[1],
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int mode = 0; mode < 3; ++mode) {
    const int steps = 1024;
    k_issue<<<148, 128, 65536>>>(steps, mode, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i];
    mean /= 148;
    printf("issue mode=%d: %7.1f cycles per 4-MMA step, commit every 16 steps (%s)\n", mode, mean / steps,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_steps, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int fence = 0; fence < 2; ++fence)
    for (int wb = 0; wb < 2; ++wb) {
      const int steps = 512;
      k_steps<<<148, 128, 65536>>>(64, steps, fence, wb, d);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double mean = 0;
      for (int i = 0; i < 148; ++i) mean += h[i];
      mean /= 148;
      printf("steps N=64 fence=%d waitbar=%d: %7.1f cycles per 4-MMA step (%s)\n", fence, wb, mean / steps,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
