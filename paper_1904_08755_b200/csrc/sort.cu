// sort.cu — stable LSD radix sort of (uint32 key, int32 value) pairs, 8-bit digits.
//
// Used by the kernel-map builder to order output rows by their neighbour bitmask (the set
// of offsets k with a pair): rows with equal or similar masks land in the same 128-row
// tile, so the tensor-core conv skips (tile, k) units that have no pair at all.
// Per pass: k_radix_hist (per-block digit counts) -> k_radix_offsets (one CTA per digit
// scans the digit's block counts) -> k_radix_scatter (stable: elements are ranked in index
// order with a warp match + per-warp digit prefix).  Blocks are 256 threads x 4 elements.
#include "mk_internal.cuh"

namespace mk {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 4;
constexpr int kTile = kThreads * kItems;
constexpr int kWarps = kThreads / 32;

// Per-block digit counts, layout [digit][block].
__global__ void __launch_bounds__(kThreads) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                         int64_t nblocks, uint32_t* __restrict__ cnt_out) {
  __shared__ uint32_t cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int64_t e = base + i * kThreads + threadIdx.x;
    if (e < n) atomicAdd(&cnt[(keys[e] >> shift) & 255u], 1u);
  }
  __syncthreads();
  cnt_out[(int64_t)threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// One CTA per digit: exclusive scan of the digit's per-block counts (in place) and the
// digit total.
__global__ void __launch_bounds__(kThreads) k_radix_offsets(uint32_t* __restrict__ cnt, int64_t nblocks,
                                                            uint32_t* __restrict__ totals) {
  __shared__ uint32_t s_w[kWarps];
  __shared__ uint32_t s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* c = cnt + (int64_t)blockIdx.x * nblocks;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nblocks; b0 += kThreads) {
    const int64_t i = b0 + threadIdx.x;
    const uint32_t v = i < nblocks ? c[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t wb = 0;
    for (int w = 0; w < warp; ++w) wb += s_w[w];
    const uint32_t excl = s_carry + wb + x - v;
    if (i < nblocks) c[i] = excl;
    __syncthreads();
    if (threadIdx.x == kThreads - 1) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = s_carry;
}

// Stable scatter: output offset of (digit, block) = exclusive scan of the digit totals +
// the scanned per-block count (k_radix_offsets).
__global__ void __launch_bounds__(kThreads) k_radix_scatter(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
                                                            uint32_t* __restrict__ kout, int32_t* __restrict__ vout,
                                                            int64_t n, int shift, int64_t nblocks,
                                                            const uint32_t* __restrict__ cnt,
                                                            const uint32_t* __restrict__ totals) {
  __shared__ uint32_t wcnt[kWarps][256];
  __shared__ uint32_t wpre[kWarps][256];
  __shared__ uint32_t run[256];
  __shared__ uint32_t s_w[kWarps];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int w = 0; w < kWarps; ++w) wcnt[w][t] = 0;
  {
    // exclusive scan of the 256 digit totals + this block's offset within the digit
    const uint32_t v = totals[t];
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t wb = 0;
    for (int w = 0; w < warp; ++w) wb += s_w[w];
    run[t] = wb + x - v + cnt[(int64_t)t * nblocks + blockIdx.x];
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll 1
  for (int i = 0; i < kItems; ++i) {
    const int64_t e = base + i * kThreads + t;
    const bool valid = e < n;
    const uint32_t key = valid ? kin[e] : 0u;
    const int32_t val = valid ? (vin ? vin[e] : (int32_t)e) : 0;
    const uint32_t d = valid ? (key >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    {  // thread t = digit: prefix over warps in index order
      uint32_t r = run[t];
      for (int w = 0; w < kWarps; ++w) {
        wpre[w][t] = r;
        r += wcnt[w][t];
        wcnt[w][t] = 0;
      }
      run[t] = r;
    }
    __syncthreads();
    if (valid) {
      const uint32_t pos = wpre[warp][d] + rank;
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
  }
}

}  // namespace

// Sorts keys[0..n) (only the low `bits` bits are significant) stably, carrying the element
// index as value; writes the permutation to perm[0..n).  `keys` is clobbered.
mk_status radix_sort_perm(const Alloc& a, uint32_t* keys, int64_t n, int bits, int32_t* perm, cudaStream_t s) {
  if (n <= 0) return MK_OK;
  const int64_t nblocks = ceil_div(n, kTile);
  const int passes = (bits + 7) / 8;
  uint32_t* k2 = (uint32_t*)dev_alloc(a, sizeof(uint32_t) * n, s);
  int32_t* v2 = (int32_t*)dev_alloc(a, sizeof(int32_t) * n, s);
  int32_t* v1 = (int32_t*)dev_alloc(a, sizeof(int32_t) * n, s);
  uint32_t* cnt = (uint32_t*)dev_alloc(a, sizeof(uint32_t) * (256 * nblocks + 256 * passes), s);
  if (!k2 || !v2 || !v1 || !cnt) {
    dev_free(a, k2, s);
    dev_free(a, v2, s);
    dev_free(a, v1, s);
    dev_free(a, cnt, s);
    MK_FAIL(MK_ERR_OUT_OF_MEMORY, "radix sort: allocation failed");
  }
  uint32_t* totals = cnt + 256 * nblocks;  // [passes][256]
  cudaError_t e = cudaSuccess;
  uint32_t* kin = keys;
  uint32_t* kout = k2;
  int32_t* vin = nullptr;  // first pass: values are the element indices
  int32_t* vout = passes == 1 ? perm : v1;
  for (int p = 0; p < passes && e == cudaSuccess; ++p) {
    const int shift = 8 * p;
    k_radix_hist<<<(unsigned)nblocks, kThreads, 0, s>>>(kin, n, shift, nblocks, cnt);
    k_radix_offsets<<<256, kThreads, 0, s>>>(cnt, nblocks, totals + 256 * p);
    k_radix_scatter<<<(unsigned)nblocks, kThreads, 0, s>>>(kin, vin, kout, vout, n, shift, nblocks, cnt,
                                                           totals + 256 * p);
    g_launches += 3;
    std::swap(kin, kout);
    vin = vout;
    // ping-pong values, the last pass writes perm
    vout = (p + 2 == passes) ? perm : (vout == v1 ? v2 : v1);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  dev_free(a, k2, s);
  dev_free(a, v2, s);
  dev_free(a, v1, s);
  dev_free(a, cnt, s);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("radix sort: ") + cudaGetErrorString(e));
  return MK_OK;
}

}  // namespace mk
