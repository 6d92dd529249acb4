// sort.cu — stable LSD radix sort of (uint32 key, int32 value) pairs, 8- or 9-bit digits.
//
// Used by the kernel-map builder to order output rows by their neighbour bitmask (the set
// of offsets k with a pair): rows with equal or similar masks land in the same 128-row
// tile, so the tensor-core conv skips (tile, k) units that have no pair at all.
// Per pass: k_radix_hist (per-block digit counts) -> k_radix_offsets (one CTA per digit
// scans the digit's block counts) -> k_radix_scatter (stable: elements are ranked in index
// order with a warp match + per-warp digit prefix).  Blocks are 256 threads x 4 elements.
// A 27-bit mask (3x3x3) takes 3 passes of 9 bits.  (A single-pass "onesweep" variant with
// per-digit decoupled look-back was measured slower here: 18 us per pass at 150k keys,
// the per-digit look-back chains are serial.)
#include "mk_internal.cuh"

namespace mk {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 4;
constexpr int kTile = kThreads * kItems;
constexpr int kWarps = kThreads / 32;

// Per-block digit counts, layout [digit][block].
template <int RB>
__global__ void __launch_bounds__(kThreads) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                         int64_t nblocks, uint32_t* __restrict__ cnt_out) {
  pdl_enter();
  constexpr int DIG = 1 << RB;
  __shared__ uint32_t cnt[DIG];
  for (int d = threadIdx.x; d < DIG; d += kThreads) cnt[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int64_t e = base + i * kThreads + threadIdx.x;
    if (e < n) atomicAdd(&cnt[(__ldg(keys + e) >> shift) & (DIG - 1u)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < DIG; d += kThreads) cnt_out[(int64_t)d * nblocks + blockIdx.x] = cnt[d];
}

// One CTA per digit: exclusive scan of the digit's per-block counts (in place) and the
// digit total.
__global__ void __launch_bounds__(kThreads) k_radix_offsets(uint32_t* __restrict__ cnt, int64_t nblocks,
                                                            uint32_t* __restrict__ totals) {
  pdl_enter();
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
// the scanned per-block count (k_radix_offsets).  Thread t owns digits t*DPT .. t*DPT+DPT-1.
template <int RB>
__global__ void __launch_bounds__(kThreads) k_radix_scatter(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
                                                            uint32_t* __restrict__ kout, int32_t* __restrict__ vout,
                                                            int64_t n, int shift, int64_t nblocks,
                                                            const uint32_t* __restrict__ cnt,
                                                            const uint32_t* __restrict__ totals) {
  pdl_enter();
  constexpr int DIG = 1 << RB;
  constexpr int DPT = DIG / kThreads;  // digits per thread (1 or 2)
  __shared__ uint32_t wcnt[kWarps][DIG];
  __shared__ uint32_t wpre[kWarps][DIG];
  __shared__ uint32_t run[DIG];
  __shared__ uint32_t s_w[kWarps];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int w = 0; w < kWarps; ++w)
#pragma unroll
    for (int j = 0; j < DPT; ++j) wcnt[w][t * DPT + j] = 0;
  {
    uint32_t v[DPT], sum = 0;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      v[j] = totals[t * DPT + j];
      sum += v[j];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t wb = 0;
    for (int w = 0; w < warp; ++w) wb += s_w[w];
    uint32_t e = wb + x - sum;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      run[t * DPT + j] = e + cnt[(int64_t)(t * DPT + j) * nblocks + blockIdx.x];
      e += v[j];
    }
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
    const uint32_t d = valid ? (key >> shift) & (DIG - 1u) : (uint32_t)DIG;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < DPT; ++j) {  // thread = digit: prefix over warps in index order
      const int dd = t * DPT + j;
      uint32_t r = run[dd];
      for (int w = 0; w < kWarps; ++w) {
        wpre[w][dd] = r;
        r += wcnt[w][dd];
        wcnt[w][dd] = 0;
      }
      run[dd] = r;
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

template <int RB>
void launch_pass(const uint32_t* kin, const int32_t* vin, uint32_t* kout, int32_t* vout, int64_t n, int shift,
                 int64_t nblocks, uint32_t* cnt, uint32_t* totals, cudaStream_t s) {
  // plain launches: with PDL the three passes measured ~4 us slower each (configs[1])
  k_radix_hist<RB><<<(unsigned)nblocks, kThreads, 0, s>>>(kin, n, shift, nblocks, cnt);
  k_radix_offsets<<<1 << RB, kThreads, 0, s>>>(cnt, nblocks, totals);
  k_radix_scatter<RB><<<(unsigned)nblocks, kThreads, 0, s>>>(kin, vin, kout, vout, n, shift, nblocks, cnt, totals);
  g_launches += 3;
}

}  // namespace

// Sorts keys[0..n) (only the low `bits` bits are significant) stably, carrying the element
// index as value; writes the permutation to perm[0..n).  `keys` is clobbered.
mk_status radix_sort_perm(const Alloc& a, uint32_t* keys, int64_t n, int bits, int32_t* perm, cudaStream_t s) {
  if (n <= 0) return MK_OK;
  bits = std::max(1, std::min(bits, 32));
  const int64_t nblocks = ceil_div(n, kTile);
  const int passes = (bits + 8) / 9;            // digits of at most 9 bits
  const int rb = (bits + passes - 1) / passes;  // bits per digit (<= 9)
  const int dig = rb <= 8 ? 256 : 512;
  // one scratch block: keys / values ping-pong, per-block counts, digit totals
  const size_t b_kv = ((sizeof(uint32_t) * n + 255) / 256) * 256;
  char* ws = (char*)dev_alloc(a, 3 * b_kv + sizeof(uint32_t) * ((size_t)dig * nblocks + (size_t)dig * passes), s);
  if (!ws) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "radix sort: allocation failed");
  uint32_t* k2 = (uint32_t*)ws;
  int32_t* v1 = (int32_t*)(ws + b_kv);
  int32_t* v2 = (int32_t*)(ws + 2 * b_kv);
  uint32_t* cnt = (uint32_t*)(ws + 3 * b_kv);
  uint32_t* totals = cnt + (size_t)dig * nblocks;  // [passes][dig]
  uint32_t* kin = keys;
  uint32_t* kout = k2;
  int32_t* vin = nullptr;  // first pass: values are the element indices
  int32_t* vout = passes == 1 ? perm : v1;
  for (int p = 0; p < passes; ++p) {
    const int shift = rb * p;
    if (dig == 256)
      launch_pass<8>(kin, vin, kout, vout, n, shift, nblocks, cnt, totals + dig * p, s);
    else
      launch_pass<9>(kin, vin, kout, vout, n, shift, nblocks, cnt, totals + dig * p, s);
    std::swap(kin, kout);
    vin = vout;
    // ping-pong values, the last pass writes perm
    vout = (p + 2 == passes) ? perm : (vout == v1 ? v2 : v1);
  }
  const cudaError_t e = cudaGetLastError();
  dev_free(a, ws, s);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("radix sort: ") + cudaGetErrorString(e));
  return MK_OK;
}

}  // namespace mk
