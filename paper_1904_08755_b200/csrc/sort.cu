// sort.cu — stable LSD radix sort of (uint32 key, int32 value) pairs, 8- or 9-bit digits.
//
// Used by the kernel-map builder to order output rows by their neighbour bitmask (the set
// of offsets k with a pair): rows with equal or similar masks land in the same 128-row
// tile, so the tensor-core conv skips (tile, k) units that have no pair at all.
// A 27-bit mask (3x3x3) takes 3 passes of 9 bits.
// Default: all passes in ONE cooperative kernel (k_radix_sort_coop, one CTA per SM, grid
// barriers between phases, next-pass digit counts accumulated during the scatter).
// Fallback (no barrier slot, or MK_SORT_COOP=0): three kernels per pass, k_radix_hist
// (per-block digit counts) -> k_radix_offsets (one CTA per digit scans the digit's block
// counts) -> k_radix_scatter (stable: elements are ranked in index order with a warp match +
// per-warp digit prefix), 256 threads x 4 elements per block.  configs[1] (150k keys):
// 55 us for the nine launches, 34 us for the cooperative kernel.  (A single-pass "onesweep"
// variant with per-digit decoupled look-back was slower still: 18 us per pass, the
// per-digit look-back chains are serial.)
#include <cstdlib>

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


// ---------------------------------------------------------------- one-kernel variant
// All passes in one cooperative launch of G <= #SM CTAs (one per SM, all co-resident), the
// phases separated by grid barriers instead of kernel boundaries (each boundary of the
// three-kernel scheme costs a launch and a drain, ~4 us per kernel at 150k keys).  CTA c
// owns the contiguous tile [c T, (c+1) T) of the current order.  cnt_p[d][c] = number of
// keys of digit d (pass p) in tile c:
//   pass 0 H  per-tile digit counts -> cnt_0; zero this CTA's column of cnt_1.. | barrier
//   O  one warp per digit: exclusive scan of cnt_p[d][0..G) in place, totals[d] | barrier
//   S  stable scatter: run[d] = prefix of totals + cnt_p[d][c]; chunks of kCT keys ranked
//      in index order (warp match + per-warp digit prefix), as k_radix_scatter; each key
//      also counts its next-pass digit into cnt_{p+1}[d'][pos / T] (global atomics), so
//      later passes need no H phase                                              | barrier
constexpr int kCT = 512;
#ifndef MK_SORT_MINB
#define MK_SORT_MINB 1
#endif
constexpr int kCW = kCT / 32;
constexpr int kCR = 4;  // chunks of a tile held in registers (tiles up to 2048 keys)

#ifdef MK_SORT_PROF  // development: phase timestamps of CTA 0 / CTA G-1, printed at the end
#define SORT_MARK(i)                                                             \
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_prof[i]));
#else
#define SORT_MARK(i)
#endif

// Grid barrier over the G CTAs (co-resident: cooperative launch).  bar[0] counts arrivals
// and only grows during the kernel: barrier i of the kernel completes when it reaches
// (i + 1) G, so each CTA does one fire-and-forget release add and polls with acquire loads.
// bar[1] counts CTAs that passed their last barrier; the last one resets both words to 0
// for the next launch that uses this slot (stream-ordered after this one).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}
__device__ __forceinline__ void grid_barrier_done(unsigned* bar, unsigned G) {
  if (threadIdx.x == 0 && atomicAdd(bar + 1, 1u) == G - 1u) {
    bar[0] = 0;
    bar[1] = 0;
  }
}

template <int RB>
__global__ void __launch_bounds__(kCT, MK_SORT_MINB) k_radix_sort_coop(uint32_t* __restrict__ keys, uint32_t* __restrict__ k2,
                                                            int32_t* __restrict__ v1, int32_t* __restrict__ v2,
                                                            int32_t* __restrict__ perm, int64_t n, int passes,
                                                            int rb, uint32_t* __restrict__ cnt,
                                                            uint32_t* __restrict__ totals, unsigned* bar) {
  pdl_wait();
  constexpr int DIG = 1 << RB;
  extern __shared__ uint32_t sm_sort[];
  uint32_t* wcnt = sm_sort;                  // [kCW][DIG]
  uint32_t* wpre = wcnt + kCW * DIG;         // [kCW][DIG]
  uint32_t* run = wpre + kCW * DIG;          // [DIG]
  __shared__ uint32_t s_w[kCW];
#ifdef MK_SORT_PROF
  __shared__ unsigned long long s_prof[16];
#endif
  SORT_MARK(0)
  const unsigned G = gridDim.x, c = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t T = (n + G - 1) / G, tb = min(n, (int64_t)c * T), te = min(n, tb + T);
  const uint32_t dmask = (1u << rb) - 1u;
  const int dig = 1 << rb;  // digits in use (<= DIG)
  const int64_t cstride = (int64_t)DIG * G;  // one pass's count matrix
  uint32_t* kin = keys;
  uint32_t* kout = k2;
  int32_t* vin = nullptr;
  int32_t* vout = passes == 1 ? perm : v1;
  uint32_t kr[kCR];
  int32_t vr[kCR];
  auto fetch = [&](int64_t e, uint32_t* k, int32_t* v) {
    *k = kin[e];
    *v = vin ? vin[e] : (int32_t)e;
  };
  // ---- pass 0 H: digit counts of this tile (keys kept in registers for S)
  for (int d = t; d < DIG; d += kCT) run[d] = 0;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kCR; ++i) {
    const int64_t e = tb + (int64_t)i * kCT + t;
    if (e < te) {
      fetch(e, &kr[i], &vr[i]);
      atomicAdd(&run[kr[i] & dmask], 1u);
    }
  }
  for (int64_t e = tb + (int64_t)kCR * kCT + t; e < te; e += kCT) atomicAdd(&run[kin[e] & dmask], 1u);
  __syncthreads();
  for (int d = t; d < dig; d += kCT) {
    cnt[(int64_t)d * G + c] = run[d];
    for (int q = 1; q < passes; ++q) cnt[q * cstride + (int64_t)d * G + c] = 0;
  }
  SORT_MARK(1)
  unsigned nbar = 0;  // barriers passed
  grid_barrier(bar, ++nbar * G);
  SORT_MARK(2)
  for (int p = 0; p < passes; ++p) {
    const int shift = rb * p;
    uint32_t* cp = cnt + p * cstride;
    uint32_t* cn = cnt + (p + 1) * cstride;  // next pass (unused in the last)
    const bool last = p + 1 == passes;
    if (p > 0) {  // this pass's keys were written by other CTAs (complete after the barrier)
#pragma unroll
      for (int i = 0; i < kCR; ++i) {
        const int64_t e = tb + (int64_t)i * kCT + t;
        if (e < te) fetch(e, &kr[i], &vr[i]);
      }
    }
    // ---- O: one warp per digit scans the digit's G tile counts
    for (int d = (int)c * kCW + warp; d < dig; d += (int)G * kCW) {
      uint32_t* row = cp + (int64_t)d * G;
      uint32_t carry = 0;
      for (int i0 = 0; i0 < (int)G; i0 += 32) {
        const int i = i0 + lane;
        const uint32_t v = i < (int)G ? row[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (i < (int)G) row[i] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) totals[d] = carry;
    }
    SORT_MARK(3 + 4 * p)
    grid_barrier(bar, ++nbar * G);
    SORT_MARK(4 + 4 * p)
    // ---- S: digit bases, then the stable scatter of this tile
    {
      const uint32_t v = t < dig ? totals[t] : 0u;  // kCT >= DIG: one digit per thread
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
      if (t < DIG) run[t] = t < dig ? wb + x - v + cp[(int64_t)t * G + c] : 0u;
      for (int i = t; i < kCW * DIG; i += kCT) wcnt[i] = 0;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    auto chunk = [&](int64_t e, uint32_t key, int32_t val) {
      const bool valid = e < te;
      const uint32_t d = valid ? (key >> shift) & dmask : (uint32_t)DIG;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const uint32_t rank = __popc(peers & lt);
      if (valid && rank == 0) wcnt[warp * DIG + d] = __popc(peers);
      __syncthreads();
      if (t < DIG) {  // thread = digit: prefix over warps in index order
        uint32_t r = run[t];
        for (int w = 0; w < kCW; ++w) {
          wpre[w * DIG + t] = r;
          r += wcnt[w * DIG + t];
          wcnt[w * DIG + t] = 0;
        }
        run[t] = r;
      }
      __syncthreads();
      uint32_t pos = 0;
      if (valid) {
        pos = wpre[warp * DIG + d] + rank;
        kout[pos] = key;
        vout[pos] = val;
      }
      if (!last) {  // next-pass count, one atomic per distinct (digit, tile) of the warp
        const uint32_t slot = valid ? ((key >> (shift + rb)) & dmask) * G + (uint32_t)(pos / T) : 0xffffffffu;
        const unsigned same = __match_any_sync(0xffffffffu, slot);
        if (valid && (__ffs(same) - 1) == lane) atomicAdd(&cn[slot], (unsigned)__popc(same));
      }
      __syncthreads();
    };
#pragma unroll
    for (int i = 0; i < kCR; ++i) {
      const int64_t b0 = tb + (int64_t)i * kCT;
      if (b0 < te) chunk(b0 + t, kr[i], vr[i]);  // block-uniform condition
    }
    {  // the rest of the tile, one chunk ahead: the next chunk's key and value are in flight
       // while this chunk is ranked (just-in-time loads left every chunk waiting on memory)
      int64_t b0 = tb + (int64_t)kCR * kCT;
      uint32_t key = 0;
      int32_t val = 0;
      if (b0 + t < te) fetch(b0 + t, &key, &val);
      for (; b0 < te; b0 += kCT) {
        const int64_t e = b0 + t, en = e + kCT;
        uint32_t kn = 0;
        int32_t vn = 0;
        if (en < te) fetch(en, &kn, &vn);
        chunk(e, key, val);
        key = kn;
        val = vn;
      }
    }
    SORT_MARK(5 + 4 * p)
    if (!last) grid_barrier(bar, ++nbar * G);
    SORT_MARK(6 + 4 * p)
    uint32_t* tk = kin;
    kin = kout;
    kout = tk;
    vin = vout;
    vout = (p + 2 == passes) ? perm : (vout == v1 ? v2 : v1);
  }
  grid_barrier_done(bar, G);
#ifdef MK_SORT_PROF
  if (threadIdx.x == 0 && (c == 0 || c == G - 1))
    printf("sort cta %u: H %.2f b %.2f | O %.2f b %.2f S %.2f b %.2f | O %.2f b %.2f S %.2f b %.2f | O %.2f b %.2f S %.2f\n",
           c, (s_prof[1] - s_prof[0]) * 1e-3, (s_prof[2] - s_prof[1]) * 1e-3, (s_prof[3] - s_prof[2]) * 1e-3,
           (s_prof[4] - s_prof[3]) * 1e-3, (s_prof[5] - s_prof[4]) * 1e-3, (s_prof[6] - s_prof[5]) * 1e-3,
           (s_prof[7] - s_prof[6]) * 1e-3, (s_prof[8] - s_prof[7]) * 1e-3, (s_prof[9] - s_prof[8]) * 1e-3,
           (s_prof[10] - s_prof[9]) * 1e-3, (s_prof[11] - s_prof[10]) * 1e-3, (s_prof[12] - s_prof[11]) * 1e-3,
           (s_prof[13] - s_prof[12]) * 1e-3);
#endif
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
mk_status radix_sort_perm(const Alloc& a, uint32_t* keys, int64_t n, int bits, int32_t* perm, cudaStream_t s,
                          unsigned* bar, int num_sms) {
  if (n <= 0) return MK_OK;
  bits = std::max(1, std::min(bits, 32));
  const int64_t nblocks = ceil_div(n, kTile);
  const int passes = (bits + 8) / 9;            // digits of at most 9 bits
  const int rb = (bits + passes - 1) / passes;  // bits per digit (<= 9)
  const int dig = rb <= 8 ? 256 : 512;
  // one scratch block: keys / values ping-pong, per-block counts, digit totals
  const size_t b_kv = ((sizeof(uint32_t) * n + 255) / 256) * 256;
  // count matrix: [dig][nblocks] (three-kernel passes) or [passes][dig][G <= num_sms] (coop)
  const int64_t ncols = std::max<int64_t>(nblocks, (int64_t)passes * num_sms);
  char* ws = (char*)dev_alloc(a, 3 * b_kv + sizeof(uint32_t) * ((size_t)dig * ncols + (size_t)dig * passes), s);
  if (!ws) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "radix sort: allocation failed");
  uint32_t* k2 = (uint32_t*)ws;
  int32_t* v1 = (int32_t*)(ws + b_kv);
  int32_t* v2 = (int32_t*)(ws + 2 * b_kv);
  uint32_t* cnt = (uint32_t*)(ws + 3 * b_kv);
  uint32_t* totals = cnt + (size_t)dig * ncols;  // [passes][dig]
  static const bool no_coop = [] {
    const char* v = std::getenv("MK_SORT_COOP");
    return v && v[0] == '0';
  }();
  if (bar && !no_coop && n <= INT32_MAX) {
    static const int g_cap = [] {
      const char* v = std::getenv("MK_SORT_G");  // development: CTA count cap
      return v ? std::atoi(v) : 0;
    }();
    // Large sorts run beside the pair-list emit on the other stream (the map builder forks
    // them) and this kernel takes a whole SM's registers per CTA: two thirds of the SMs leave
    // room for the emit (configs[4] map phase 993 -> 939 us; small maps keep every SM).
    const int g_def = n >= (1 << 20) ? std::max(1, num_sms * 2 / 3) : num_sms;
    const int G = (int)std::max<int64_t>(
        1, std::min<int64_t>(g_cap > 0 ? std::min(g_cap, num_sms) : g_def, ceil_div(n, kCT)));
    const size_t smem = sizeof(uint32_t) * (2 * kCW * dig + dig);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kCT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (dig == 256) {
      static bool once = (cudaFuncSetAttribute(k_radix_sort_coop<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(sizeof(uint32_t) * (2 * kCW * 256 + 256))), true);
      (void)once;
      e = cudaLaunchKernelEx(&cfg, k_radix_sort_coop<8>, keys, k2, v1, v2, perm, n, passes, rb, cnt, totals, bar);
    } else {
      static bool once = (cudaFuncSetAttribute(k_radix_sort_coop<9>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(sizeof(uint32_t) * (2 * kCW * 512 + 512))), true);
      (void)once;
      e = cudaLaunchKernelEx(&cfg, k_radix_sort_coop<9>, keys, k2, v1, v2, perm, n, passes, rb, cnt, totals, bar);
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    dev_free(a, ws, s);
    if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("radix sort: ") + cudaGetErrorString(e));
    return MK_OK;
  }
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

extern "C" mk_status mk_debug_sort_perm(mk_context* ctx, const uint32_t* d_keys, int64_t n, int32_t bits,
                                        int32_t* d_perm, void* stream) {
  using namespace mk;
  clear_error();
  if (!ctx || n < 0 || (n > 0 && (!d_keys || !d_perm)) || bits < 1 || bits > 32)
    MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_debug_sort_perm: bad argument");
  if (n == 0) return MK_OK;
  if (n > INT32_MAX) MK_FAIL(MK_ERR_UNSUPPORTED, "mk_debug_sort_perm: more than 2^31 keys");
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t* k = (uint32_t*)dev_alloc(ctx->alloc, sizeof(uint32_t) * n, s);  // the sort clobbers its keys
  if (!k) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "mk_debug_sort_perm: allocation failed");
  const cudaError_t e = cudaMemcpyAsync(k, d_keys, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) {
    dev_free(ctx->alloc, k, s);
    MK_FAIL(MK_ERR_CUDA, std::string("mk_debug_sort_perm: ") + cudaGetErrorString(e));
  }
  const mk_status st = radix_sort_perm(ctx->alloc, k, n, bits, d_perm, s, ctx->barrier_slot(), ctx->num_sms);
  dev_free(ctx->alloc, k, s);
  return st;
}
