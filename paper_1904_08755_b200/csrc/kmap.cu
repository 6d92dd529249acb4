// kmap.cu — kernel-map builder (Eq. 3; transposed P:202).
//
// For every output row o (key u) and offset k (vector i_k) the builder probes u + sign*i_k*s
// in the input table.  Work is organised in tiles of 128 output rows — the row tile of the
// convolution kernels — so the same pass produces:
//   nbr[k][o]             dense neighbour table (-1 = absent) read by the conv kernels;
//   tile_cnt[k][tile]     pairs per (offset, tile) -> per-offset CSR offsets by a scan;
//   tile_mask[tile][w]    bit k set when (tile, k) has at least one pair (lets the conv
//                         kernels skip empty (tile, offset) MMAs).
// Kernels:
//   k_probe   one CTA per tile, 256 threads = 128 rows x 2 offset lanes; 16-byte key loads,
//             warp-ballot/popc counting into shared memory.
//   k_scan    one CTA per offset: exclusive scan of tile counts (pairs of an offset are laid
//             out tile after tile, i.e. in output-row order).
//   k_emit    ballot/popc compaction of nbr into the CSR pair lists; when the map is not
//             symmetric it also scatters the transposed table nbrT[k][a] = o used by dgrad.
// One host sync per build (the total pair count is needed to size the pair lists).
#include <algorithm>
#include <climits>
#include <cstring>
#include <deque>
#include <map>

#include <cstdlib>

#include "mk_internal.cuh"

namespace mk {
namespace {

constexpr int kTileRows = 128;
constexpr int kThreads = 256;
constexpr int kRM = 32;       // row-major staging width: entries per row (K <= 32)
constexpr int kRMPitch = 33;  // smem pitch of a staged row (bank-conflict free)

// u + sign * off * scale, per spatial axis, batch unchanged (R18).  False when the
// shifted coordinate cannot exist (outside int32 or the packed-key domain).
struct Scale {  // offset scale per axis (the fine tensor stride, R14)
  int32_t s[kMaxD];
};

__device__ __forceinline__ bool shift_key(int4 u, int D, const int32_t* off, int sign, const Scale& scale, int4* q) {
  int64_t c[kMaxD] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int d = 0; d < kMaxD; ++d) {  // fully unrolled: c[] stays in registers
    if (d < D) {
      const int64_t v = (int64_t)key_axis(u, D, d) + (int64_t)sign * off[d] * scale.s[d];
      if (v < INT32_MIN || v > INT32_MAX) return false;
      c[d] = v;
    }
  }
  return pack_key(c, D, key_batch(u, D), q);
}

// Probing.  One CTA per tile of 128 output rows, 256 threads; thread t owns row t % 128
// and its offsets k = t / 128 + 2i.  A query u + sign*i_k*s reads the key's whole 64-byte
// bucket (three keys and their rows: four independent 16-byte loads, one round trip) and
// kPB queries are in flight per thread; a query continues to the next bucket only when all
// three slots hold other keys (rare).  (A 4-lane cooperative variant — lane j loads word j
// of the bucket, a ballot resolves — was measured at 172 us on configs[1]: every lane of a
// group recomputes the query key and hash, so it is instruction bound.)
// Results are staged in shared memory per chunk of <= 32 offsets, then:
//   RM (K <= 32): written as a row-major block [row][32] (coalesced; k_permute_rm turns it
//                 into the permuted k-major table), plus per-row neighbour bitmasks;
//   otherwise:    written k-major [K][n_pad] (coalesced per offset).
// Per (offset, tile) pair counts and the tile's active-offset mask come from warp ballots
// over the staged block.
// Queries in flight per thread and CTAs per SM: the probe is latency bound, so occupancy
// pays more than per-thread ILP (configs[1] kmap phase: PB 4 / 2 CTAs 153 us, PB 4 / 3 CTAs
// 145 us, PB 2 / 4 CTAs 134 us, PB 2 / 5 CTAs 136 us; round 2, configs[4] map phase: PB 2 /
// 4 CTAs 1107 us, PB 1 / 6 CTAs 1006 us, PB 1 / 8 CTAs 1041 us, PB 4 / 3 CTAs 1250 us, with
// configs[1] within 3 us of the best).
#ifndef MK_PROBE_PB
#define MK_PROBE_PB 1
#endif
#ifndef MK_PROBE_MINB
#define MK_PROBE_MINB 6
#endif
constexpr int kPB = MK_PROBE_PB;

template <bool RM>
__global__ void __launch_bounds__(kThreads, MK_PROBE_MINB) k_probe(const int4* __restrict__ okeys, int64_t n_out, int64_t n_pad,
                                                    const TableRef tref,
                                                    const int32_t* __restrict__ offs, int K, int D, int sign,
                                                    Scale scale4, int32_t* __restrict__ nbr,
                                                    int32_t* __restrict__ tile_cnt, int64_t ntiles,
                                                    uint32_t* __restrict__ tile_mask, int mw,
                                                    uint32_t* __restrict__ rowmask) {
  pdl_enter();
  extern __shared__ int32_t sm[];
  int4* s_doff = (int4*)sm;                  // [K] offset deltas of a packed key (fast path)
  int32_t* s_off = sm + 4 * K;               // [K*D]
  int32_t* s_cnt = s_off + K * D;            // [32] counts of the current chunk
  int32_t* s_tab = s_cnt + kRM;              // [128][33]
  __shared__ int s_slow;                     // some offset delta does not fit the fast path
  if (threadIdx.x == 0) s_slow = 0;
  for (int i = threadIdx.x; i < K * D; i += kThreads) s_off[i] = offs[i];
  __syncthreads();
  // Fast path: key(u + sign*i_k*s) = key(u) + delta_k as one int4 add, valid whenever the row's
  // components are small enough that no component can leave its range (|u| < 2^30 and
  // |delta| < 2^30; D = 4 packs t in 16 bits: |t| < 2^14 and |dt| < 2^14).
  for (int k = threadIdx.x; k < K; k += kThreads) {
    int64_t d[4] = {0, 0, 0, 0};
    bool fits = D <= 4;  // packed D = 5..7 keys always take the exact slow path
#pragma unroll
    for (int a = 0; a < 4; ++a)
      if (a < D) {
        d[a] = (int64_t)sign * s_off[k * D + a] * scale4.s[a];
        fits &= (d[a] > -(1ll << 30) && d[a] < (1ll << 30)) && (a < 3 || (d[a] > -(1 << 14) && d[a] < (1 << 14)));
      }
    if (!fits) atomicOr(&s_slow, 1);
    s_doff[k] = make_int4((int32_t)d[0], (int32_t)d[1], (int32_t)d[2], D == 4 ? (int32_t)((uint32_t)d[3] << 16) : 0);
  }
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = threadIdx.x & (kTileRows - 1), kl = threadIdx.x >> 7;
  const int64_t o = tile * kTileRows + r;
  const bool valid = o < n_out;
  const int4 u = valid ? __ldg(okeys + o) : make_int4(0, 0, 0, 0);
  // the region of the input table that holds the row's batch (offsets never change the
  // batch, R18): one lookup per row instead of per query
  const int4* __restrict__ buckets = tref.buckets;
  uint32_t rbase = 0, rsize = 0;
  const bool in_tab = valid && tref.region(u, &rbase, &rsize);
  auto small = [](int32_t v, int32_t lim) { return v > -lim && v < lim; };
  // block-uniform: one row outside the fast-path range sends the whole tile down the slow path
  const bool fast = __syncthreads_and(!s_slow && D <= 4 && small(u.x, 1 << 30) && small(u.y, 1 << 30) &&
                                      small(u.z, 1 << 30) && (D < 4 || small(key_axis(u, D, 3), 1 << 14)));
  for (int kc = 0; kc < K; kc += kRM) {
    const int kn = min(kRM, K - kc);
    for (int kb = kl; kb < kn; kb += 2 * kPB) {
      int4 q[kPB], k0[kPB], v[kPB];
      uint32_t hb[kPB];
      bool ok[kPB];
#pragma unroll
      for (int b = 0; b < kPB; ++b) {
        const int k = kb + 2 * b;
        if (fast) {
          const int4 dq = s_doff[kc + (k < kn ? k : 0)];
          q[b] = make_int4(u.x + dq.x, u.y + dq.y, u.z + dq.z, u.w + dq.w);
          ok[b] = valid && k < kn;
        } else {
          ok[b] = valid && k < kn && shift_key(u, D, s_off + (kc + k) * D, sign, scale4, &q[b]);
        }
        // unconditional loads of the first sector (bucket 0 for masked queries): no
        // divergent regions, all kPB loads of the thread are issued back to back
        ok[b] = ok[b] && in_tab;
        hb[b] = ok[b] ? rbase + hash_bucket(hash_key(q[b]), rsize) : 0u;
        load_sector(buckets + (size_t)hb[b] * 4u, &k0[b], &v[b]);
      }
#pragma unroll
      for (int b = 0; b < kPB; ++b) {
        const int k = kb + 2 * b;
        if (k < kn) {
          int32_t a = -1;
          if (ok[b]) {
            if (key_eq(k0[b], q[b])) {
              a = v[b].x;
            } else if (k0[b].w != kEmptyWord && v[b].y >= 0) {  // slot 1 occupied (rare)
              a = bucket_rest(buckets + (size_t)hb[b] * 4u, q[b], k0[b], v[b]);
              if (a == -2) a = probe_next(buckets, rbase, rsize, q[b], hb[b]);  // bucket full of other keys
            }
          }
          s_tab[r * kRMPitch + k] = a;
        }
      }
    }
    __syncthreads();
    // pair counts per offset of the chunk: ballots over the 128 staged rows
    for (int k = warp; k < kn; k += kThreads / 32) {
      int c = 0;
#pragma unroll
      for (int r0 = 0; r0 < kTileRows; r0 += 32) c += __popc(__ballot_sync(0xffffffffu, s_tab[(r0 + lane) * kRMPitch + k] >= 0));
      if (lane == 0) s_cnt[k] = c;
    }
    if (RM) {
      int32_t* dst = nbr + tile * (kTileRows * kRM);
      for (int i = threadIdx.x; i < kTileRows * kRM; i += kThreads) {
        const int rr = i >> 5, k = i & (kRM - 1);
        dst[i] = k < kn ? s_tab[rr * kRMPitch + k] : -1;
      }
      if (rowmask && threadIdx.x < kTileRows) {
        const int64_t o = tile * kTileRows + threadIdx.x;
        uint32_t rm = 0;
        for (int k = 0; k < kn; ++k) rm |= (s_tab[threadIdx.x * kRMPitch + k] >= 0 ? 1u : 0u) << k;
        if (o < n_out) rowmask[o] = rm;
      }
    } else {
      for (int i = threadIdx.x; i < kn * kTileRows; i += kThreads) {
        const int k = i >> 7, rr = i & (kTileRows - 1);
        nbr[(int64_t)(kc + k) * n_pad + tile * kTileRows + rr] = s_tab[rr * kRMPitch + k];  // padding rows: -1
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kn; k += kThreads) tile_cnt[(int64_t)(kc + k) * ntiles + tile] = s_cnt[k];
    if (threadIdx.x == 0) {
      uint32_t bits = 0;
      for (int k = 0; k < kn; ++k) bits |= (s_cnt[k] > 0 ? 1u : 0u) << k;
      tile_mask[tile * mw + kc / 32] = bits;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_scan(const int32_t* __restrict__ tile_cnt, int64_t ntiles,
                                               int64_t* __restrict__ tile_off, int64_t* __restrict__ totals) {
  pdl_enter();
  __shared__ int64_t s_w[32];
  __shared__ int64_t s_carry;
  const int k = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < ntiles; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < ntiles ? tile_cnt[(int64_t)k * ntiles + i] : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_w[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    const int64_t carry = s_carry;
    const int64_t excl = carry + (warp > 0 ? s_w[warp - 1] : 0) + incl - v;
    if (i < ntiles) tile_off[(int64_t)k * ntiles + i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[k] = s_carry;
}

// Per-offset CSR offsets ptr[k] = sum of totals[0..k) computed on the device (block-local
// copy in shared memory; block 0 also publishes ptr[0..K]).  Then ballot/popc compaction of
// the tile's neighbour entries into the pair lists (output-ascending within an offset,
// S:157); for maps that are not symmetric also the transposed table nbrT[k][a] = o (dgrad).
template <bool RM>
__global__ void __launch_bounds__(kThreads, 8) k_emit(const int32_t* __restrict__ nbr, int64_t n_out, int64_t n_pad, int K,
                                                   const int64_t* __restrict__ totals, int64_t* __restrict__ ptr_out,
                                                   const int64_t* __restrict__ tile_off, int64_t ntiles,
                                                   int32_t* __restrict__ in_idx, int32_t* __restrict__ out_idx,
                                                   int32_t* __restrict__ nbrT, int64_t nT_pad,
                                                   uint32_t* __restrict__ tile_maskT, int mw) {
  pdl_enter();
  extern __shared__ int64_t s_ptr[];                  // [K + 1]
  int64_t* s_toff = s_ptr + K + 1;                    // [K] this tile's offset inside each offset's list
  int32_t* s_wc = (int32_t*)(s_toff + K);             // [K][4] pairs per (offset, warp of the tile)
  int32_t* s_tab = s_wc + 4 * K;                      // [128][33] (RM)
  const int64_t tile = blockIdx.x;
  const int r = threadIdx.x & (kTileRows - 1);
  const int64_t o = tile * kTileRows + r;
  const bool valid = o < n_out;
  const int lane = threadIdx.x & 31, wq = r >> 5;  // warp quarter of the 128-row tile
  const unsigned lt = (1u << lane) - 1u;
  if (threadIdx.x < 32) {  // warp 0: exclusive scan of the offset totals
    int64_t carry = 0;
    for (int b = 0; b < K; b += 32) {
      const int64_t v = b + lane < K ? totals[b + lane] : 0;
      int64_t x = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (b + lane < K) s_ptr[b + lane] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) s_ptr[K] = carry;
  }
  for (int k = threadIdx.x; k < K; k += kThreads) s_toff[k] = tile_off[(int64_t)k * ntiles + tile];
  if (RM) {  // 16 KB block: four independent 16-byte loads per thread, then scalar stores
    const int4* src = (const int4*)(nbr + tile * (kTileRows * kRM));
    int4 v[kTileRows * kRM / 4 / kThreads];
#pragma unroll
    for (int j = 0; j < kTileRows * kRM / 4 / kThreads; ++j) v[j] = __ldg(src + threadIdx.x + j * kThreads);
#pragma unroll
    for (int j = 0; j < kTileRows * kRM / 4 / kThreads; ++j) {
      const int i = 4 * (threadIdx.x + j * kThreads);
      int32_t* d = s_tab + (i >> 5) * kRMPitch + (i & (kRM - 1));
      d[0] = v[j].x;
      d[1] = v[j].y;
      d[2] = v[j].z;
      d[3] = v[j].w;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k <= K; k += kThreads) ptr_out[k] = s_ptr[k];
  auto get = [&](int k) -> int32_t {
    if (!valid) return -1;
    return RM ? s_tab[r * kRMPitch + k] : nbr[(int64_t)k * n_pad + o];
  };
  for (int k = threadIdx.x / kTileRows; k < K; k += kThreads / kTileRows) {
    const unsigned b = __ballot_sync(0xffffffffu, get(k) >= 0);
    if (lane == 0) s_wc[k * 4 + wq] = __popc(b);
  }
  __syncthreads();
  // first list position of every (offset, warp quarter): one thread per offset
  for (int k = threadIdx.x; k < K; k += kThreads) {
    int64_t base = s_ptr[k] + s_toff[k];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int32_t c = s_wc[k * 4 + w];
      s_wc[k * 4 + w] = (int32_t)(base - s_ptr[k]);  // offset inside offset k's list (< 2^31)
      base += c;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x / kTileRows; k < K; k += kThreads / kTileRows) {
    const int32_t a = get(k);
    const unsigned b = __ballot_sync(0xffffffffu, a >= 0);
    if (a < 0) continue;
    const int64_t pos = s_ptr[k] + s_wc[k * 4 + wq] + __popc(b & lt);
    in_idx[pos] = a;
    out_idx[pos] = (int32_t)o;
    if (nbrT) {
      nbrT[(int64_t)k * nT_pad + a] = (int32_t)o;
      atomicOr(tile_maskT + (int64_t)(a / kTileRows) * mw + (k >> 5), 1u << (k & 31));
    }
  }
}

// Permuted k-major table from the row-major block (K <= 32): position i holds row perm[i];
// out[k][i] = nbr_rm[perm[i]][k] (one 128-byte row load per position, coalesced k-major
// stores), plus the active-offset mask of every permuted 128-row tile.
// With `mirror` set (symmetric submanifold map) it also writes the dgrad tile mask: bit k of
// the dgrad view = bit mirror[k] of the forward mask.
__global__ void __launch_bounds__(kTileRows) k_permute_rm(const int32_t* __restrict__ nbr_rm, int64_t stride, int64_t n,
                                                          int K, const int32_t* __restrict__ perm,
                                                          int32_t* __restrict__ out, uint32_t* __restrict__ tmask,
                                                          const int32_t* __restrict__ mirror,
                                                          uint32_t* __restrict__ tmaskT) {
  pdl_enter();
  __shared__ uint32_t s_bits;
  if (threadIdx.x == 0) s_bits = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kTileRows + threadIdx.x;
  const int32_t r = i < n ? (perm ? perm[i] : (int32_t)i) : -1;
  int32_t v[kRM];
  if (r >= 0) {
    const int4* src = (const int4*)(nbr_rm + (int64_t)r * kRM);
#pragma unroll
    for (int j = 0; j < kRM / 4; ++j) {
      const int4 x = __ldg(src + j);
      v[4 * j] = x.x;
      v[4 * j + 1] = x.y;
      v[4 * j + 2] = x.z;
      v[4 * j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kRM; ++j) v[j] = -1;
  }
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < kRM; ++k) {
    if (k < K) {
      out[(int64_t)k * stride + i] = v[k];
      if (__any_sync(0xffffffffu, v[k] >= 0)) bits |= 1u << k;
    }
  }
  if ((threadIdx.x & 31) == 0) atomicOr(&s_bits, bits);
  __syncthreads();
  if (threadIdx.x == 0) tmask[blockIdx.x] = s_bits;
  if (mirror && threadIdx.x < 32) {
    const uint32_t bT = threadIdx.x < K ? ((s_bits >> __ldg(mirror + threadIdx.x)) & 1u) << threadIdx.x : 0u;
    const uint32_t m = __reduce_or_sync(0xffffffffu, bT);
    if (threadIdx.x == 0) tmaskT[blockIdx.x] = m;
  }
}

// Row masks of the dgrad table: bit k set when nbrT[k][a] >= 0 (K <= 32).
__global__ void k_rowmask_T(const int32_t* __restrict__ nbrT, int64_t stride, int64_t n, int K,
                            uint32_t* __restrict__ rowmask) {
  pdl_enter();
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    uint32_t rm = 0;
    for (int k = 0; k < K; ++k) rm |= (nbrT[(int64_t)k * stride + a] >= 0 ? 1u : 0u) << k;
    rowmask[a] = rm;
  }
}

// Neighbour table in permuted row order: out[k][i] = tab[k][perm[i]] (padding rows -1), and
// the active-offset mask of every permuted 128-row tile (K <= 32: one word).
__global__ void __launch_bounds__(kTileRows) k_permute_km(const int32_t* __restrict__ tab, int64_t stride, int64_t n,
                                                       int K, const int32_t* __restrict__ perm,
                                                       int32_t* __restrict__ out, uint32_t* __restrict__ tmask) {
  pdl_enter();
  __shared__ uint32_t s_bits;
  if (threadIdx.x == 0) s_bits = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kTileRows + threadIdx.x;
  const int32_t r = i < n ? perm[i] : -1;
  uint32_t bits = 0;
  for (int k = 0; k < K; ++k) {
    const int32_t a = r >= 0 ? tab[(int64_t)k * stride + r] : -1;
    out[(int64_t)k * stride + i] = a;
    if (__any_sync(0xffffffffu, a >= 0)) bits |= 1u << k;
  }
  if ((threadIdx.x & 31) == 0) atomicOr(&s_bits, bits);
  __syncthreads();
  if (threadIdx.x == 0) tmask[blockIdx.x] = s_bits;
}

// Dgrad tile masks of a symmetric map: bit k of tile t = bit mirror[k] of the forward mask.
__global__ void k_mirror_mask(const uint32_t* __restrict__ mask, int64_t ntiles, int mw, const int32_t* __restrict__ mirror,
                              int K, uint32_t* __restrict__ maskT) {
  pdl_enter();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x)
    for (int w = 0; w < mw; ++w) {
      uint32_t bits = 0;
      for (int j = 0; j < 32 && w * 32 + j < K; ++j) {
        const int q = mirror[w * 32 + j];
        bits |= ((mask[t * mw + (q >> 5)] >> (q & 31)) & 1u) << j;
      }
      maskT[t * mw + w] = bits;
    }
}

// Region enumeration + mirror indices, cached per thread by region description (the
// offsets of a region never change; a layer stack rebuilds maps for the same regions).
struct RegionInfo {
  std::vector<int32_t> offs;    // [K][D]
  int32_t K = 0;
  std::vector<int32_t> mirror;  // [K] index of -offset_k or -1
  bool closed = true;           // every offset's negation is in the set
};

// Device copy of (offsets, mirror) for this context, uploaded on first use; nullptr when the
// cache is full (the caller then uploads per build).
const int32_t* region_device(mk_context* ctx, const std::vector<int32_t>& offs, const std::vector<int32_t>& mirror) {
  constexpr size_t kMaxCached = 64;
  std::vector<int32_t> key(offs);
  key.insert(key.end(), mirror.begin(), mirror.end());
  std::lock_guard<std::mutex> lock(ctx->region_mu);
  for (auto& r : ctx->region_dev)
    if (r.first == key) return r.second;
  if (ctx->region_dev.size() >= kMaxCached) return nullptr;
  int32_t* d = nullptr;
  if (cudaMalloc(&d, sizeof(int32_t) * std::max<size_t>(key.size(), 1)) != cudaSuccess) return nullptr;
  if (!key.empty() && cudaMemcpy(d, key.data(), sizeof(int32_t) * key.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  ctx->region_dev.emplace_back(std::move(key), d);
  return d;
}

mk_status region_info(const mk_region* r, const RegionInfo** out) {
  std::vector<int32_t> key = {r->type, r->D, r->temporal_axis, r->n_offsets};
  for (int d = 0; d < r->D && d < MK_MAX_REGION; ++d) {
    key.push_back(r->size[d]);
    key.push_back(r->dilation[d]);
  }
  if (r->type == MK_CUSTOM && r->offsets && r->n_offsets > 0)
    key.insert(key.end(), r->offsets, r->offsets + (int64_t)r->n_offsets * r->D);
  thread_local std::deque<std::pair<std::vector<int32_t>, RegionInfo>> cache;  // stable element addresses
  for (auto& e : cache)
    if (e.first == key) {
      *out = &e.second;
      return MK_OK;
    }
  RegionInfo ri;
  mk_status st = region_enumerate(r, &ri.offs, &ri.K);
  if (st != MK_OK) return st;
  const int D = r->D, K = ri.K;
  std::map<std::vector<int32_t>, int32_t> index;
  for (int k = 0; k < K; ++k) index[std::vector<int32_t>(ri.offs.begin() + k * D, ri.offs.begin() + (k + 1) * D)] = k;
  ri.mirror.assign(K, -1);
  for (int k = 0; k < K; ++k) {
    std::vector<int32_t> neg(D);
    for (int d = 0; d < D; ++d) neg[d] = -ri.offs[k * D + d];
    auto it = index.find(neg);
    if (it == index.end()) ri.closed = false;
    else ri.mirror[k] = it->second;
  }
  if (cache.size() >= 16) cache.pop_front();
  cache.emplace_back(std::move(key), std::move(ri));
  *out = &cache.back().second;
  return MK_OK;
}

}  // namespace

namespace {
// h_ptr / n_pairs from the device totals; caller holds m->mu.
mk_status kmap_host_locked(mk_kmap* m) {
  if (m->host_ready) return MK_OK;
  cudaError_t e = cudaEventSynchronize(m->done);  // the build only, not the stream's later work
  int64_t* h = (int64_t*)pinned_stage(sizeof(int64_t) * m->K);
  if (!h) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "kmap: pinned staging failed");
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, m->d_totals, sizeof(int64_t) * m->K, cudaMemcpyDeviceToHost, m->aux);
  if (e == cudaSuccess) e = cudaStreamSynchronize(m->aux);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("kmap: pair count read-back: ") + cudaGetErrorString(e));
  m->h_ptr.assign(m->K + 1, 0);
  for (int k = 0; k < m->K; ++k) m->h_ptr[k + 1] = m->h_ptr[k] + h[k];
  m->n_pairs = m->h_ptr[m->K];
  if (m->n_pairs > INT32_MAX) MK_FAIL(MK_ERR_UNSUPPORTED, "kmap: more than 2^31 pairs");
  m->host_ready = true;
  return MK_OK;
}
}  // namespace

mk_status kmap_host(const mk_kmap* cm) {
  mk_kmap* m = const_cast<mk_kmap*>(cm);
  std::lock_guard<std::mutex> lk(*m->mu);
  return kmap_host_locked(m);
}

// Weight-gradient split-K plan (tensor-core path): the concatenated pair list is cut into
// per-CTA ranges of <= L pairs (L = 64 * ceil(|M| / #SM / 64)) and <= kWgradMaxSegs
// (range, offset) segments; every segment has its own partial slot; slots are in offset
// order.
mk_status kmap_wplan(const mk_kmap* cm, cudaStream_t s) {
  mk_kmap* m = const_cast<mk_kmap*>(cm);
  std::lock_guard<std::mutex> lk(*m->mu);
  mk_status st = kmap_host_locked(m);
  if (st != MK_OK) return st;
  if (m->wplan_ready) {
    if (s != m->wplan_stream && cudaStreamWaitEvent(s, m->wplan_ev, 0) != cudaSuccess)
      MK_FAIL(MK_ERR_CUDA, "kmap: stream wait failed");
    return MK_OK;
  }
  const int K = m->K;
  std::vector<int4> segs;
  std::vector<int32_t> seg_begin, slot_begin(K + 1, 0);
  const int64_t P = m->n_pairs;
  const int64_t L = std::max<int64_t>(64, ceil_div(ceil_div(std::max<int64_t>(P, 1), m->num_sms), 64) * 64);
  // Greedy cut of the concatenated pair list: a CTA takes up to L pairs and at most
  // kWgradMaxSegs segments (the kernel's per-CTA plan size), cutting at offset boundaries.
  int64_t cta_pairs = L;  // forces a new CTA at the first segment
  int cta_segs = 0;
  for (int k = 0; k < K; ++k) {
    for (int64_t b = m->h_ptr[k]; b < m->h_ptr[k + 1];) {
      if (cta_pairs >= L || cta_segs >= kWgradMaxSegs) {
        seg_begin.push_back((int32_t)segs.size());
        cta_pairs = 0;
        cta_segs = 0;
      }
      const int64_t e2 = std::min(m->h_ptr[k + 1], b + (L - cta_pairs));
      segs.push_back(make_int4(k, (int)b, (int)e2, (int)segs.size()));
      cta_pairs += e2 - b;
      ++cta_segs;
      b = e2;
    }
  }
  const int64_t ncta = (int64_t)seg_begin.size();
  seg_begin.push_back((int32_t)segs.size());
  for (int k = 0, i = 0; k <= K; ++k) {
    while (i < (int)segs.size() && segs[i].x < k) ++i;
    slot_begin[k] = i;
  }
  const size_t b_seg = sizeof(int4) * std::max<size_t>(1, segs.size());
  const size_t b_sb = sizeof(int32_t) * seg_begin.size(), b_kb = sizeof(int32_t) * (K + 1);
  const size_t total = b_seg + b_sb + b_kb;
  char* d = (char*)dev_alloc(m->alloc, total, m->stream);
  char* h = (char*)pinned_stage(total);
  if (!d || !h) {
    if (d) dev_free(m->alloc, d, m->stream);
    MK_FAIL(MK_ERR_OUT_OF_MEMORY, "kmap: weight-gradient plan allocation failed");
  }
  m->owned.push_back(d);
  if (!segs.empty()) std::memcpy(h, segs.data(), sizeof(int4) * segs.size());
  std::memcpy(h + b_seg, seg_begin.data(), b_sb);
  std::memcpy(h + b_seg + b_sb, slot_begin.data(), b_kb);
  cudaError_t e = cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s);
  pinned_in_flight(s);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->wplan_ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(m->wplan_ev, s);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("kmap: plan upload: ") + cudaGetErrorString(e));
  m->wseg = (int4*)d;
  m->wseg_begin = (int32_t*)(d + b_seg);
  m->wslot_begin = (int32_t*)(d + b_seg + b_sb);
  m->n_wcta = (int32_t)ncta;
  m->n_wslots = (int64_t)segs.size();
  m->wplan_stream = s;
  m->wplan_ready = true;
  return MK_OK;
}

}  // namespace mk

using namespace mk;

extern "C" {

mk_status mk_kmap_build(mk_context* ctx, const mk_coords* in, const mk_coords* out, const mk_region* region,
                        int32_t transposed, void* stream_, mk_kmap** out_map) {
  HostTimer ht("kmap_build");
  clear_error();
  cudaStream_t s = (cudaStream_t)stream_;
  if (!ctx || !in || !out || !region || !out_map) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_kmap_build: null argument");
  if (in->D != out->D || region->D != in->D)
    MK_FAIL(MK_ERR_DIMENSION_MISMATCH, "mk_kmap_build: input, output and region must have the same D");
  const int D = in->D;
  mk_status rs = coords_resolve(in);  // deferred row counts are needed from here on
  if (rs == MK_OK && out != in) rs = coords_resolve(out);
  if (rs != MK_OK) return rs;
  const RegionInfo* ri = nullptr;
  mk_status st = region_info(region, &ri);
  if (st != MK_OK) return st;
  const std::vector<int32_t>& offs = ri->offs;
  const int32_t K = ri->K;
  if (K > 4096) MK_FAIL(MK_ERR_UNSUPPORTED, "mk_kmap_build: more than 4096 kernel offsets");
  ht.mark("region");

  mk_kmap* m = new mk_kmap();
  m->alloc = ctx->alloc;
  m->stream = s;
  m->aux = ctx->aux;
  m->num_sms = ctx->num_sms;
  m->mu = new std::mutex();
  m->K = K;
  m->D = D;
  m->transposed = transposed ? 1 : 0;
  m->n_in = in->n;
  m->n_out = out->n;
  m->mask_words = (K + 31) / 32;
  const int mw = m->mask_words;
  // Offsets scale with the fine tensor stride: the input's for a conv, the output's for a
  // transposed conv (R14).
  const int32_t* sc = transposed ? out->tensor_stride : in->tensor_stride;
  Scale scale4;
  for (int d = 0; d < kMaxD; ++d) scale4.s[d] = d < D ? sc[d] : 1;
  const int sign = transposed ? -1 : 1;

  // mirror[k]: index of -offset_k (used to reuse nbr for dgrad on submanifold maps)
  m->mirror = ri->mirror;
  const bool symmetric = (in == out) && ri->closed;

  const int64_t n_out = out->n, n_in = in->n;
  const int64_t ntiles = std::max<int64_t>(1, ceil_div(n_out, kTileRows));
  const int64_t ntilesT = std::max<int64_t>(1, ceil_div(n_in, kTileRows));
  const int64_t n_pad = ntiles * kTileRows, nT_pad = ntilesT * kTileRows;  // table rows padded to whole tiles
  m->nbr_stride = n_pad;
  m->nbrT_stride = symmetric ? n_pad : nT_pad;
  // K <= 32: row-major staging + bitmask row ordering, and pair lists allocated at their
  // upper bound K * n_out so the build needs its one host sync only at the very end.
  // K > 32: k-major table, identity order, exact pair lists (sync after the count).
  const bool rm = K <= kRM;
  const bool upper_bound = rm;

  auto fail = [&](mk_status code, const std::string& msg) {
    mk_kmap_destroy(m);
    set_error(code, msg);
    return code;
  };
  auto alloc = [&](size_t bytes) -> void* {
    void* p = dev_alloc(m->alloc, bytes, s);
    if (p) m->owned.push_back(p);
    return p;
  };
  // scratch (freed stream-ordered at the end of the build)
  std::vector<void*> scratch;
  auto salloc = [&](size_t bytes) -> void* {
    void* p = dev_alloc(m->alloc, bytes, s);
    if (p) scratch.push_back(p);
    return p;
  };
  auto free_scratch = [&]() {
    for (void* p : scratch) dev_free(m->alloc, p, s);
    scratch.clear();
  };
  auto oom = [&]() {
    free_scratch();
    return fail(MK_ERR_OUT_OF_MEMORY, "mk_kmap_build: device allocation failed");
  };

  ht.mark("mirror");
  // Two device allocations per build: one persistent block (owned by the map) and one
  // scratch block, carved into 256-byte aligned arrays.
  struct Bump {
    size_t off = 0;
    size_t take(size_t b) {
      const size_t o = off;
      off += (b + 255) & ~size_t(255);
      return o;
    }
  };
  const bool sort_fwd = rm && n_out > 0, sort_bwd = rm && !symmetric && n_in > 0;
  const int64_t ub_pairs = upper_bound ? (int64_t)K * n_out : 0;
  Bump pb;
  const size_t o_offs = pb.take(sizeof(int32_t) * (K * D + K)), o_nbr = pb.take(sizeof(int32_t) * K * n_pad),
               o_tm = pb.take(sizeof(uint32_t) * ntiles * mw), o_tmT = pb.take(sizeof(uint32_t) * ntilesT * mw),
               o_ptr = pb.take(sizeof(int64_t) * (K + 1)), o_tot = pb.take(sizeof(int64_t) * K),
               o_nbrT = symmetric ? 0 : pb.take(sizeof(int32_t) * K * nT_pad),
               o_in = upper_bound ? pb.take(sizeof(int32_t) * (ub_pairs + 4)) : 0,
               o_out = upper_bound ? pb.take(sizeof(int32_t) * (ub_pairs + 4)) : 0,
               o_perm = sort_fwd ? pb.take(sizeof(int32_t) * n_pad) : 0,
               o_permT = sort_bwd ? pb.take(sizeof(int32_t) * nT_pad) : 0,
               o_tabP = sort_bwd ? pb.take(sizeof(int32_t) * K * nT_pad) : 0;
  Bump sbm;
  const size_t o_rm = rm ? sbm.take(sizeof(int32_t) * n_pad * kRM) : 0,
               o_toff = sbm.take(sizeof(int64_t) * K * ntiles), o_tcnt = sbm.take(sizeof(int32_t) * K * ntiles),
               o_rowm = rm ? sbm.take(sizeof(uint32_t) * std::max<int64_t>(1, std::max(n_out, n_in))) : 0;
  char* pbase = (char*)alloc(pb.off);
  char* sbase = (char*)salloc(sbm.off);
  if (!pbase || !sbase) return oom();
  int32_t* d_offs_own = (int32_t*)(pbase + o_offs);  // offsets, then mirror (if not cached)
  const int32_t* d_offs = d_offs_own;
  m->d_mirror = d_offs_own + K * D;
  m->nbr = (int32_t*)(pbase + o_nbr);
  m->tile_mask = (uint32_t*)(pbase + o_tm);
  m->tile_maskT = (uint32_t*)(pbase + o_tmT);
  m->ptr = (int64_t*)(pbase + o_ptr);
  if (!symmetric) m->nbrT = (int32_t*)(pbase + o_nbrT);
  int64_t* totals = (int64_t*)(pbase + o_tot);  // persistent: lazy host read-back
  m->d_totals = totals;
  if (upper_bound) {
    m->in_idx = (int32_t*)(pbase + o_in);
    m->out_idx = (int32_t*)(pbase + o_out);
  }
  if (sort_fwd) m->perm = (int32_t*)(pbase + o_perm);
  int32_t* tabP = sort_bwd ? (int32_t*)(pbase + o_tabP) : nullptr;
  if (sort_bwd) m->permT = (int32_t*)(pbase + o_permT);
  int32_t* nbr_rm = rm ? (int32_t*)(sbase + o_rm) : nullptr;
  int64_t* tile_off = (int64_t*)(sbase + o_toff);
  int32_t* tile_cnt = (int32_t*)(sbase + o_tcnt);
  uint32_t* rowmask = rm ? (uint32_t*)(sbase + o_rowm) : nullptr;

  cudaError_t e = cudaSuccess;
  auto ck = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
  };
  ht.mark("allocs");
  if (const int32_t* cached = region_device(ctx, offs, m->mirror)) {  // uploaded once per region
    d_offs = cached;
    m->d_mirror = cached + K * D;
  } else {  // cache full: one pinned H2D copy of the offsets and their mirror indices
    int32_t* h = (int32_t*)pinned_stage(sizeof(int32_t) * (K * D + K));
    if (!h) return oom();
    std::copy(offs.begin(), offs.end(), h);
    std::copy(m->mirror.begin(), m->mirror.end(), h + K * D);
    ck(cudaMemcpyAsync(d_offs_own, h, sizeof(int32_t) * (K * D + K), cudaMemcpyHostToDevice, s));
    pinned_in_flight(s);
  }
  if (!symmetric) {
    ck(cudaMemsetAsync(m->nbrT, 0xFF, sizeof(int32_t) * K * nT_pad, s));
    ck(cudaMemsetAsync(m->tile_maskT, 0, sizeof(uint32_t) * ntilesT * mw, s));
  }
  ht.mark("setup");
  static const bool fork_env = [] {
    const char* v = std::getenv("MK_KMAP_FORK");
    return !(v && v[0] == '0');
  }();
  const bool fork = fork_env && rm && n_out > 0 && symmetric && ctx->side;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  mk_status fork_st = MK_OK;
  if (rm && n_out > 0) {  // allocated on s before any fork (stream-ordered)
    m->perm = (int32_t*)alloc(sizeof(int32_t) * n_pad);
    if (!m->perm) return oom();
  }
  auto sort_and_permute = [&](cudaStream_t ss) {
    fork_st = radix_sort_perm(m->alloc, rowmask, n_out, K, m->perm, ss, ctx->barrier_slot(), ctx->num_sms);
    if (fork_st == MK_OK)
      ck(pdl_launch(k_permute_rm, (unsigned)ntiles, kTileRows, 0, ss, nbr_rm, n_pad, n_out, K, m->perm, m->nbr,
                    m->tile_mask, symmetric ? m->d_mirror : nullptr, m->tile_maskT));
  };
  if (n_out > 0) {
    const size_t smem = sizeof(int32_t) * (4 * K + K * D + kRM + kTileRows * kRMPitch);
    if (smem > 48 * 1024) {
      cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (rm)
      ck(pdl_launch(k_probe<true>, (unsigned)ntiles, kThreads, smem, s, out->keys, n_out, n_pad, in->table.ref(D),
                    d_offs, K, D, sign, scale4, nbr_rm, tile_cnt, ntiles, m->tile_mask, mw, rowmask));
    else
      ck(pdl_launch(k_probe<false>, (unsigned)ntiles, kThreads, smem, s, out->keys, n_out, n_pad, in->table.ref(D),
                    d_offs, K, D, sign, scale4, m->nbr, tile_cnt, ntiles, m->tile_mask, mw, nullptr));
    // Symmetric row-ordered maps: the row sort and the permuted table depend only on the probe,
    // the pair lists only on the probe and the scan, so the sort + permute run on the
    // context's side stream concurrently with scan + emit (joined before the build ends).
    if (fork) {
      ck(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      ck(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
      ck(cudaEventRecord(ev_fork, s));
      ck(cudaStreamWaitEvent(ctx->side, ev_fork, 0));
      sort_and_permute(ctx->side);
      ck(cudaEventRecord(ev_join, ctx->side));
    }
    ck(pdl_launch(k_scan, K, 1024, 0, s, tile_cnt, ntiles, tile_off, totals));
    ht.mark("probe+scan");
  } else {
    ck(cudaMemsetAsync(m->tile_mask, 0, sizeof(uint32_t) * ntiles * mw, s));
    ck(cudaMemsetAsync(m->nbr, 0xFF, sizeof(int32_t) * K * n_pad, s));
    ck(cudaMemsetAsync(totals, 0, sizeof(int64_t) * K, s));
    ck(cudaMemsetAsync(m->ptr, 0, sizeof(int64_t) * (K + 1), s));
  }
  ck(cudaGetLastError());
  // Host copy of the per-offset pair counts.  K > 32 maps size their pair lists exactly and
  // read the counts back here (one stream sync); K <= 32 maps defer it (mk::kmap_host).
  auto read_totals_now = [&]() -> bool {
    int64_t* h_tot = (int64_t*)pinned_stage(sizeof(int64_t) * K);
    if (!h_tot) return false;
    ck(cudaMemcpyAsync(h_tot, totals, sizeof(int64_t) * K, cudaMemcpyDeviceToHost, s));
    ck(cudaStreamSynchronize(s));
    m->h_ptr.assign(K + 1, 0);
    for (int k = 0; k < K; ++k) m->h_ptr[k + 1] = m->h_ptr[k] + (e == cudaSuccess ? h_tot[k] : 0);
    m->n_pairs = m->h_ptr[K];
    m->host_ready = true;
    return true;
  };
  int64_t pair_cap = (int64_t)K * n_out;
  if (!upper_bound) {
    if (!read_totals_now()) return oom();
    if (e != cudaSuccess) {
      free_scratch();
      return fail(MK_ERR_CUDA, std::string("mk_kmap_build: ") + cudaGetErrorString(e));
    }
    pair_cap = m->n_pairs;
  }
  if (!upper_bound && pair_cap > INT32_MAX) {
    free_scratch();
    return fail(MK_ERR_UNSUPPORTED, "mk_kmap_build: more than 2^31 pairs");
  }
  // +4 entries of padding: the wgrad kernel reads 16-byte aligned supersets of ranges
  if (!upper_bound) {
    m->in_idx = (int32_t*)alloc(sizeof(int32_t) * (pair_cap + 4));
    m->out_idx = (int32_t*)alloc(sizeof(int32_t) * (pair_cap + 4));
    if (!m->in_idx || !m->out_idx) return oom();
  }
  if (n_out > 0) {
    const size_t smem = sizeof(int64_t) * (2 * K + 1) + sizeof(int32_t) * (4 * K + (rm ? kTileRows * kRMPitch : 0));
    if (rm)
      ck(pdl_launch(k_emit<true>, (unsigned)ntiles, kThreads, smem, s, nbr_rm, n_out, n_pad, K, totals, m->ptr,
                    tile_off, ntiles, m->in_idx, m->out_idx, m->nbrT, nT_pad, m->tile_maskT, mw));
    else
      ck(pdl_launch(k_emit<false>, (unsigned)ntiles, kThreads, smem, s, m->nbr, n_out, n_pad, K, totals, m->ptr,
                    tile_off, ntiles, m->in_idx, m->out_idx, m->nbrT, nT_pad, m->tile_maskT, mw));
  }
  // Order the conv tiles' rows by neighbour bitmask (stable radix sort of the row masks):
  // rows sharing offsets share tiles, so the tensor-core kernels skip empty (tile, k) units.
  // The permutation is internal; the CSR above and all exported row orders are unchanged.
  if (rm && n_out > 0) {
    if (fork) {
      ck(cudaStreamWaitEvent(s, ev_join, 0));
      st = fork_st;
    } else {
      ht.mark("emit");
      sort_and_permute(s);
      st = fork_st;
    }
    if (st == MK_OK && !symmetric && n_in > 0) {
      ck(pdl_launch(k_rowmask_T, (unsigned)std::min<int64_t>(ceil_div(n_in, 256), 4096), 256, 0, s, m->nbrT, nT_pad,
                    n_in, K, rowmask));
      st = radix_sort_perm(m->alloc, rowmask, n_in, K, m->permT, s, ctx->barrier_slot(), ctx->num_sms);
      if (st == MK_OK) {
        ck(pdl_launch(k_permute_km, (unsigned)ntilesT, kTileRows, 0, s, m->nbrT, nT_pad, n_in, K, m->permT, tabP,
                      m->tile_maskT));
        m->nbrT = tabP;  // the unpermuted table stays owned (freed with the map) but is no longer read
      }
    }
    if (st != MK_OK) {
      free_scratch();
      return fail(st, "mk_kmap_build: row ordering failed");
    }
  }
  if (symmetric && !(rm && n_out > 0)) {  // (k_permute_rm already wrote the mirrored masks)
    ck(pdl_launch(k_mirror_mask, (unsigned)std::min<int64_t>(ceil_div(ntiles, 256), 1024), 256, 0, s, m->tile_mask,
                  ntiles, mw, m->d_mirror, K, m->tile_maskT));
  }
  if (symmetric) m->permT = m->perm;  // same row set, mirrored masks: same ordering
  if (ev_fork) cudaEventDestroy(ev_fork);  // released once complete
  if (ev_join) cudaEventDestroy(ev_join);
  ck(cudaGetLastError());
  free_scratch();  // stream-ordered: after every kernel above
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(m->done, s);
  if (e != cudaSuccess) return fail(MK_ERR_CUDA, std::string("mk_kmap_build: ") + cudaGetErrorString(e));
  *out_map = m;
  return MK_OK;
}

mk_status mk_kmap_info(const mk_kmap* m, int32_t* K, int64_t* n_pairs, int64_t* n_in, int64_t* n_out) {
  clear_error();
  if (!m) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_kmap_info: null handle");
  if (K) *K = m->K;
  if (n_pairs) {
    const mk_status st = kmap_host(m);
    if (st != MK_OK) return st;
    *n_pairs = m->n_pairs;
  }
  if (n_in) *n_in = m->n_in;
  if (n_out) *n_out = m->n_out;
  return MK_OK;
}

mk_status mk_kmap_export(const mk_kmap* m, int64_t* d_ptr, int32_t* d_in, int32_t* d_out, void* stream) {
  clear_error();
  if (!m) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_kmap_export: null handle");
  cudaStream_t s = (cudaStream_t)stream;
  const mk_status st = kmap_host(m);
  if (st != MK_OK) return st;
  if (d_ptr) MK_CUDA_TRY(cudaMemcpyAsync(d_ptr, m->ptr, sizeof(int64_t) * (m->K + 1), cudaMemcpyDeviceToDevice, s));
  if (m->n_pairs > 0) {
    if (d_in) MK_CUDA_TRY(cudaMemcpyAsync(d_in, m->in_idx, sizeof(int32_t) * m->n_pairs, cudaMemcpyDeviceToDevice, s));
    if (d_out) MK_CUDA_TRY(cudaMemcpyAsync(d_out, m->out_idx, sizeof(int32_t) * m->n_pairs, cudaMemcpyDeviceToDevice, s));
  }
  return MK_OK;
}

void mk_kmap_destroy(mk_kmap* m) {
  if (!m) return;
  for (void* p : m->owned) dev_free(m->alloc, p, m->stream);
  if (m->done) cudaEventDestroy(m->done);
  if (m->wplan_ev) cudaEventDestroy(m->wplan_ev);
  delete m->mu;
  delete m;
}

}  // extern "C"
