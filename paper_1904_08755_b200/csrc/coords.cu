// coords.cu — coordinate manager: quantization (Alg. 1), creation from integer
// rows (Eq. 1), strided output coordinates (R11), exact lookup and export.
//
// One sort-free pipeline serves all three constructors (a "key source" supplies row p's
// packed key and validation):
//   k_init    bucket table to the empty sentinel, first-point words to INT32_MAX.
//   k_insert  one thread per input row: build the key and claim-or-find its slot in the
//             bucketed open-addressing table (mk_internal.cuh) with one 128-bit atomicCAS of
//             the key itself (linear probing over slots); atomicMin records the smallest
//             input row of each key.
//   k_rank    winners (first[slot] == p) are ranked by a single-pass decoupled look-back
//             scan in input order => rows in first-occurrence order (R8), first point of a
//             voxel is its representative (R9).  Writes the row keys and the slot's row;
//             then (optional) point_to_row[p] = row of p's slot (waits for the key's first
//             point, which is in the same or an earlier block).
// The host then reads the error word and the row count (the one sync of the call).
#include <cuda/atomic>

#include <climits>
#include <cstring>
#include <vector>

#include <cstdlib>

#include "mk_internal.cuh"

namespace mk {

namespace {

constexpr int kBlock = 256;
#ifndef MK_TABLE_SLOTS_X2
#define MK_TABLE_SLOTS_X2 4
#endif
// Tables of at least this many buckets (64 MB, half of L2) get per-batch regions (TableRef).
#ifndef MK_SUB_MIN_BUCKETS
#define MK_SUB_MIN_BUCKETS (1u << 20)
#endif
#ifndef MK_RANK_ITEMS
#define MK_RANK_ITEMS 5
#endif
#ifndef MK_RANK_MINB
#define MK_RANK_MINB 1
#endif
constexpr int kItems = MK_RANK_ITEMS;  // consecutive points per thread in k_rank
constexpr int kTile = kBlock * kItems;

enum : uint32_t { E_NONE = 0, E_NONFINITE = 1, E_RANGE = 2, E_BATCH = 3, E_STRIDE = 4 };

__device__ __forceinline__ void report(unsigned long long* err, int64_t row, uint32_t code) {
  atomicMin(err, ((unsigned long long)row << 8) | code);
}

// ---------------------------------------------------------------- key sources
struct QuantSrc {  // Alg. 1 line 1: C_p' <- floor(C_p / v_l)   (R6: fp32 division, floor)
  const float* pts;
  const int32_t* batch;
  int D;
  float voxel;
  __device__ __forceinline__ uint32_t key(int64_t p, int4* k) const {
    int64_t c[kMaxD] = {0, 0, 0, 0, 0, 0, 0};
    bool nonfinite = false, range = false;
#pragma unroll
    for (int d = 0; d < kMaxD; ++d) {  // fully unrolled: c[] stays in registers
      if (d < D) {
        const float x = pts[p * D + d];
        if (!isfinite(x)) {
          nonfinite = true;
        } else {
          const float q = floorf(__fdiv_rn(x, voxel));
          if (!(q >= -2147483648.0f && q < 2147483648.0f)) range = true;
          else c[d] = (int64_t)q;
        }
      }
    }
    if (nonfinite) return E_NONFINITE;
    if (range) return E_RANGE;
    const int64_t b = batch ? batch[p] : 0;
    if (b < 0) return E_BATCH;
    return pack_key(c, D, b, k) ? E_NONE : E_RANGE;
  }
  // batch index of row p as the key will hold it (-1 or out of range: the key is invalid)
  __device__ __forceinline__ int64_t batch_of(int64_t p) const { return batch ? batch[p] : 0; }
};

struct IntSrc {  // integer rows [n][D+1], batch last (Eq. 1); multiples of the tensor stride
  const int32_t* rows;
  int D;
  int32_t ts[kMaxD];
  __device__ __forceinline__ uint32_t key(int64_t p, int4* k) const {
    int64_t c[kMaxD] = {0, 0, 0, 0, 0, 0, 0};
    const int32_t* r = rows + p * (D + 1);
#pragma unroll
    for (int d = 0; d < kMaxD; ++d) {
      if (d < D) {
        const int32_t v = r[d];
        if (v % ts[d] != 0) return E_STRIDE;
        c[d] = v;
      }
    }
    const int64_t b = r[D];
    if (b < 0) return E_BATCH;
    return pack_key(c, D, b, k) ? E_NONE : E_RANGE;
  }
  __device__ __forceinline__ int64_t batch_of(int64_t p) const { return rows[p * (D + 1) + D]; }
};

struct StrideSrc {  // u' = floor_div(u, s_out) * s_out per spatial axis (R7, R11)
  const int4* keys;
  int D;
  int64_t s[kMaxD];
  __device__ __forceinline__ uint32_t key(int64_t p, int4* k) const {
    const int4 in = keys[p];
    int64_t c[kMaxD] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int d = 0; d < kMaxD; ++d) {
      if (d < D) {
        const int64_t u = key_axis(in, D, d);
        int64_t q = u / s[d];
        if (q * s[d] != u && u < 0) q -= 1;
        const int64_t v = q * s[d];
        if (v < INT32_MIN || v > INT32_MAX) return E_RANGE;
        c[d] = v;
      }
    }
    return pack_key(c, D, key_batch(in, D), k) ? E_NONE : E_RANGE;
  }
  __device__ __forceinline__ int64_t batch_of(int64_t p) const { return key_batch(keys[p], D); }
};

struct ExpandSrc {  // f4: expanded row p = (input row p / K, offset p % K) -> u + i_k * s (R18)
  const int4* keys;
  const int32_t* offs;  // [K][D] device
  int K, D;
  int64_t s[kMaxD];
  __device__ __forceinline__ uint32_t key(int64_t p, int4* k) const {
    const int64_t r = p / K;
    const int j = (int)(p - r * K);
    const int4 in = keys[r];
    int64_t c[kMaxD] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int d = 0; d < kMaxD; ++d) {
      if (d < D) {
        const int64_t v = (int64_t)key_axis(in, D, d) + (int64_t)__ldg(offs + j * D + d) * s[d];
        if (v < INT32_MIN || v > INT32_MAX) return E_RANGE;
        c[d] = v;
      }
    }
    return pack_key(c, D, key_batch(in, D), k) ? E_NONE : E_RANGE;
  }
  __device__ __forceinline__ int64_t batch_of(int64_t p) const { return key_batch(keys[p / K], D); }
};

// ---------------------------------------------------------------- kernels
// Per-batch region layout (TableRef): histogram of the rows' batch indices (block-local in
// shared memory, then one global add per non-empty bin), then one block sizes the regions
// (buckets for >= MK_TABLE_SLOTS_X2 / 2 slots per row, like the flat table, at least 32)
// and lays them out by an exclusive scan.  A batch index outside [0, kMaxSub) or a layout
// larger than the allocation falls back to the flat table (nsub = 0).
// cnt[kMaxSub] counts, cnt[kMaxSub] = largest batch + 1, cnt[kMaxSub + 1] = overflow flag.
template <class Src>
__global__ void __launch_bounds__(kBlock) k_bhist(Src src, int64_t n, int32_t* __restrict__ cnt) {
  pdl_enter();
  __shared__ int32_t h[kMaxSub];
  __shared__ int32_t s_max, s_over;
  for (int i = threadIdx.x; i < kMaxSub; i += kBlock) h[i] = 0;
  if (threadIdx.x == 0) s_max = 0, s_over = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int32_t bmax = 0;
  const int64_t n_round = (n + 31) & ~(int64_t)31;  // whole warps in the loop (warp-aggregated adds)
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_round; p += (int64_t)gridDim.x * blockDim.x) {
    // the batch field alone (rows with an input error are reported by k_insert; a batch
    // index that no valid key can hold only makes the layout fall back to the flat table)
    const int64_t bb = p < n ? src.batch_of(p) : -1;
    uint32_t b = bb < 0 ? 0xFFFFFFFFu : bb < kMaxSub ? (uint32_t)bb : (uint32_t)kMaxSub;
    if (b == (uint32_t)kMaxSub) {
      s_over = 1;
      b = 0xFFFFFFFFu;
    }
    // rows are usually batch-major: one shared-memory add per distinct batch of the warp
    const unsigned same = __match_any_sync(0xffffffffu, b);
    if (b != 0xFFFFFFFFu && lane == __ffs(same) - 1) {
      atomicAdd(&h[b], __popc(same));
      bmax = max(bmax, (int32_t)b + 1);
    }
  }
  if (bmax) atomicMax(&s_max, bmax);
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxSub; i += kBlock)
    if (h[i]) atomicAdd(cnt + i, h[i]);
  if (threadIdx.x == 0) {
    if (s_max) atomicMax(cnt + kMaxSub, s_max);
    if (s_over) atomicOr(cnt + kMaxSub + 1, 1);
  }
}

__global__ void __launch_bounds__(1024) k_blayout(const int32_t* __restrict__ cnt, int64_t cap_buckets,
                                                  int2* __restrict__ sub) {
  pdl_enter();
  __shared__ int64_t s_part[1024 / 32];
  constexpr int kPer = kMaxSub / 1024;
  const int nsub = cnt[kMaxSub];
  int64_t size[kPer], tot = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int b = threadIdx.x * kPer + j;
    int64_t want = b < nsub ? ((int64_t)MK_TABLE_SLOTS_X2 * cnt[b] + 2 * kSlotsPerBucket - 1) / (2 * kSlotsPerBucket) : 0;
    size[j] = b < nsub ? (want > 32 ? want : 32) : 0;
    tot += size[j];
  }
  // block exclusive scan of the per-thread totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_part[warp] = incl;
  __syncthreads();
  int64_t off = incl - tot, all = 0;
  for (int w = 0; w < 1024 / 32; ++w) {
    if (w < warp) off += s_part[w];
    all += s_part[w];
  }
  const bool flat = cnt[kMaxSub + 1] != 0 || nsub == 0 || all > cap_buckets || all > (int64_t)UINT32_MAX;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int b = threadIdx.x * kPer + j;
    if (!flat && b < nsub) sub[1 + b] = make_int2((int32_t)off, (int32_t)size[j]);
    off += size[j];
  }
  if (threadIdx.x == 0) sub[0] = make_int2(flat ? 0 : nsub, flat ? -1 : (int32_t)all);
}

template <class Src>
__global__ void __launch_bounds__(kBlock) k_insert(Src src, int64_t n, TableRef t, int32_t* __restrict__ first,
                                                   int32_t* __restrict__ slot_of, unsigned long long* err) {
  pdl_enter();
  // Claim-or-find in one 128-bit atomicCAS of the key itself (sm_90+): the slot is ours or
  // already holds the key -> record the smallest point index of the key (atomicMin).
  const unsigned __int128 kEmpty = ~(unsigned __int128)0;
  int4* buckets = const_cast<int4*>(t.buckets);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int4 k;
    const uint32_t code = src.key(p, &k);
    uint32_t base = 0, size = 0;
    if (code != E_NONE || !t.region(k, &base, &size)) {
      if (code != E_NONE) report(err, p, code);
      slot_of[p] = -1;  // no slot: k_rank skips the row (the call fails anyway)
      continue;
    }
    unsigned __int128 kv;
    memcpy(&kv, &k, sizeof(kv));
    // slots of the region: [3 base, 3 (base + size)); first slot of the key's bucket
    const uint32_t s0 = base * kSlotsPerBucket, ns = size * kSlotsPerBucket;
    uint32_t h = hash_bucket(hash_key(k), size) * kSlotsPerBucket;
    while (true) {
      const unsigned __int128 old = atomicCAS((unsigned __int128*)slot_key(buckets, s0 + h), kEmpty, kv);
      if (old == kEmpty || old == kv) {
        atomicMin(first + s0 + h, (int32_t)p);
        slot_of[p] = (int32_t)(s0 + h);
        break;
      }
      h = h + 1 == ns ? 0u : h + 1;
    }
  }
}

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Decoupled look-back (single pass): called by all 32 lanes of warp 0; returns the
// exclusive prefix of `tile` given its aggregate.
__device__ int64_t lookback(unsigned long long* status, int64_t tile, int64_t agg) {
  using Ref = cuda::atomic_ref<unsigned long long, cuda::thread_scope_device>;
  constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 62) - 1;
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) Ref(status[0]).store(kInc | (unsigned long long)agg, cuda::memory_order_relaxed);
    return 0;
  }
  if (lane == 0) Ref(status[tile]).store(kAgg | (unsigned long long)agg, cuda::memory_order_relaxed);
  int64_t excl = 0;
  int64_t top = tile - 1;
  while (true) {
    const int64_t idx = top - lane;
    unsigned long long v = kInc;
    if (idx >= 0) {
      v = Ref(status[idx]).load(cuda::memory_order_relaxed);
      while ((v >> 62) == 0) v = Ref(status[idx]).load(cuda::memory_order_relaxed);
    }
    const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    const int first = inc ? __ffs(inc) - 1 : 32;
    excl += warp_sum64(lane <= first ? (int64_t)(v & kVal) : 0);
    if (inc) break;
    top -= 32;
  }
  if (lane == 0)
    Ref(status[tile]).store(kInc | (unsigned long long)(excl + agg), cuda::memory_order_relaxed);
  return excl;
}

template <class Src>
__global__ void __launch_bounds__(kBlock, MK_RANK_MINB) k_rank(Src src, int64_t n, const int32_t* __restrict__ first,
                                                 const int32_t* __restrict__ slot_of, int4* __restrict__ buckets,
                                                 int4* __restrict__ out_keys,
                                                 int32_t* __restrict__ first_point,
                                                 int32_t* __restrict__ p2r,
                                                 unsigned long long* status, unsigned int* ticket,
                                                 int64_t* count, const unsigned long long* err, Mailbox* mb,
                                                 unsigned long long seq) {
  pdl_enter();
  __shared__ int64_t s_tile;
  __shared__ int32_t s_warp[kBlock / 32];
  __shared__ int64_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kTile + (int64_t)threadIdx.x * kItems;
  bool win[kItems];
  int32_t slot[kItems];
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int64_t p = base + i;
    win[i] = false;
    if (p < n) {
      slot[i] = slot_of[p];
      win[i] = slot[i] >= 0 && first[slot[i]] == (int32_t)p;
    }
    cnt += win[i];
  }
  // block-exclusive scan of per-thread counts
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  int warp_off = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kBlock / 32; ++w) {
    if (w < warp) warp_off += s_warp[w];
    agg += s_warp[w];
  }
  if (warp == 0) {
    const int64_t pre = lookback(status, tile, agg);
    if (lane == 0) {
      s_prefix = pre;
      if ((tile + 1) * kTile >= n) {  // last tile: the row count is final (k_insert's errors too)
        *count = pre + agg;
        if (mb) mailbox_post(mb, seq, *(const volatile unsigned long long*)err, (unsigned long long)(pre + agg));
      }
    }
  }
  __syncthreads();
  int64_t row = s_prefix + warp_off + incl - cnt;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (!win[i]) continue;
    const int64_t p = base + i;
    int4 k;
    src.key(p, &k);
    out_keys[row] = k;
    *slot_val(buckets, (uint32_t)slot[i]) = (int32_t)row;
    if (first_point) first_point[row] = (int32_t)p;
    ++row;
  }
  if (!p2r) return;
  // Inverse map point -> row: the row of p's slot is written by the key's first point,
  // which is in this block or an earlier one (block order by ticket: it is running or
  // done), so the wait below terminates.
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int64_t p = base + i;
    if (p >= n) continue;
    int32_t r = -1;
    if (slot[i] >= 0) {
      const volatile int32_t* v = slot_val(buckets, (uint32_t)slot[i]);
      while ((r = *v) < 0) {
      }
    }
    p2r[p] = r;
  }
}

// Table init in one launch: bucket words to the empty sentinel (all ones: empty keys, rows
// -1), first-point words to INT32_MAX, look-back status words / ticket / count to 0, the
// error word to all ones.
__global__ void k_init(int4* __restrict__ buckets, int32_t* __restrict__ first, uint32_t nb, const int2* sub,
                       unsigned long long* __restrict__ small, int64_t n_small, unsigned long long* err) {
  pdl_enter();
  const int4 e = make_int4(-1, -1, -1, -1);
  if (sub && sub[0].x > 0) nb = (uint32_t)sub[0].y;  // per-batch regions: the buckets in use
  const int64_t words = (int64_t)nb * 4, slots = (int64_t)nb * kSlotsPerBucket;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x) {
    buckets[i] = e;
    if (i < slots) first[i] = INT32_MAX;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_small; i += (int64_t)gridDim.x * blockDim.x)
    small[i] = 0ull;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    err[0] = ~0ull;  // no error
    err[1] = 0ull;   // row count
  }
}

// Label reduction: candidate = label of the voxel's first point; any point whose
// label differs marks the voxel IGNORE (every writer of the second kernel writes the same
// value, so the result does not depend on the schedule).
__global__ void k_labels_first(const int32_t* __restrict__ first_point, const int32_t* __restrict__ labels,
                               int64_t n_rows, int32_t* __restrict__ row_labels) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x)
    row_labels[r] = __ldg(labels + __ldg(first_point + r));
}
__global__ void k_labels_mark(const int32_t* __restrict__ p2r, const int32_t* __restrict__ first_point,
                              const int32_t* __restrict__ labels, int64_t n, int32_t ignore,
                              int32_t* __restrict__ row_labels) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = __ldg(p2r + p);
    if (__ldg(labels + p) != __ldg(labels + __ldg(first_point + r))) row_labels[r] = ignore;
  }
}

__global__ void k_lookup(const int32_t* __restrict__ q, int64_t nq, int D, TableRef t, int32_t* __restrict__ rows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[kMaxD] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int d = 0; d < kMaxD; ++d)
      if (d < D) c[d] = q[i * (D + 1) + d];
    int4 k;
    rows[i] = pack_key(c, D, q[i * (D + 1) + D], &k) ? probe(t, k) : -1;
  }
}

__global__ void k_export(const int4* __restrict__ keys, int64_t n, int D, int32_t* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int4 k = keys[r];
    for (int d = 0; d < D; ++d) out[r * (D + 1) + d] = key_axis(k, D, d);
    out[r * (D + 1) + D] = key_batch(k, D);
  }
}

int grid_for(int64_t n, int block, int sms) {
  int64_t g = ceil_div(n, block);
  int64_t cap = (int64_t)sms * 16;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

// Carves one device allocation into 256-byte aligned pieces.
struct Carver {
  size_t off = 0;
  template <class T>
  size_t take(size_t count) {
    size_t o = off;
    off += (count * sizeof(T) + 255) & ~size_t(255);
    return o;
  }
};

// Status + message of a non-empty error word (first offending row << 8 | code).
mk_status report_input_error(unsigned long long err) {
  const int64_t row = (int64_t)(err >> 8);
  const uint32_t code = (uint32_t)(err & 0xFF);
  const mk_status st = code == E_NONFINITE ? MK_ERR_NONFINITE_INPUT
                     : code == E_RANGE     ? MK_ERR_COORD_RANGE
                     : code == E_STRIDE    ? MK_ERR_STRIDE
                                           : MK_ERR_INVALID_ARGUMENT;
  const char* what = code == E_NONFINITE ? "non-finite coordinate"
                   : code == E_RANGE     ? "coordinate outside the representable range"
                   : code == E_STRIDE    ? "coordinate not a multiple of the tensor stride"
                                         : "negative batch index";
  set_error(st, std::string("coords: ") + what + " at row " + std::to_string(row), row);
  return st;
}

template <class Src>
mk_status build_coords(mk_context* ctx, const Src& src, int64_t n, int D, const int32_t* ts,
                       cudaStream_t s, mk_coords** out, int32_t* d_p2r, int32_t* d_first, bool deferred = false) {
  HostTimer ht("build_coords");
  if (n < 0 || n > INT32_MAX) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "row count out of range [0, 2^31)");
  // buckets of 3 slots, >= MK_TABLE_SLOTS_X2 * n / 2 slots in total (default 4: load <= 1/2)
  const uint32_t nb =
      next_pow2(std::max<int64_t>(ceil_div(MK_TABLE_SLOTS_X2 * n, 2 * kSlotsPerBucket), 32));
  // Per-batch regions for tables that outgrow L2 (see TableRef): a region holds its batch's
  // share (at least 32 buckets), so the regions together fit in nb + 33 kMaxSub buckets.
  static const bool no_sub = [] {
    const char* e = std::getenv("MK_NO_SUBTABLES");
    return e && e[0] && e[0] != '0';
  }();
  const bool use_sub = !no_sub && nb >= MK_SUB_MIN_BUCKETS && (int64_t)nb + 33 * kMaxSub <= (int64_t)UINT32_MAX / 4;
  const int64_t cap = use_sub ? (int64_t)nb + 33 * kMaxSub : nb;  // buckets allocated
  const int64_t nslots = cap * kSlotsPerBucket;
  const int64_t ntiles = std::max<int64_t>(1, ceil_div(n, kTile));

  mk_coords* c = new mk_coords();
  c->alloc = ctx->alloc;
  c->stream = s;
  c->D = D;
  for (int d = 0; d < D; ++d) c->tensor_stride[d] = ts[d];

  // persistent: table keys, table values, row keys
  Carver pc;
  const size_t o_tk = pc.take<int4>((size_t)cap * 4), o_rk = pc.take<int4>(std::max<int64_t>(n, 1)),
               o_res = pc.take<unsigned long long>(2),  // (error word, count) for a deferred count
      o_sub = use_sub ? pc.take<int2>(1 + kMaxSub) : 0;
  char* pbase = (char*)dev_alloc(c->alloc, pc.off, s);
  if (!pbase) {
    delete c;
    MK_FAIL(MK_ERR_OUT_OF_MEMORY, "coords: device allocation failed");
  }
  c->owned.push_back(pbase);
  c->table.buckets = (int4*)(pbase + o_tk);
  c->table.bmask = nb - 1;
  c->table.sub = use_sub ? (int2*)(pbase + o_sub) : nullptr;
  c->keys = (int4*)(pbase + o_rk);

  // scratch: first point per slot, slot per row, look-back status, ticket, error word, count
  Carver sc;
  const size_t o_cl = sc.take<int32_t>(nslots), o_sl = sc.take<int32_t>(std::max<int64_t>(n, 1)),
               o_st = sc.take<unsigned long long>(ntiles), o_ti = sc.take<unsigned int>(1),
               o_er = sc.take<unsigned long long>(2),  // error word, then the row count
      o_hi = use_sub ? sc.take<int32_t>(kMaxSub + 2) : 0;
  char* sbase = (char*)dev_alloc(c->alloc, sc.off, s);
  if (!sbase) {
    mk_coords_destroy(c);
    MK_FAIL(MK_ERR_OUT_OF_MEMORY, "coords: scratch allocation failed");
  }
  auto fail_cuda = [&](cudaError_t e, const char* what) {
    dev_free(c->alloc, sbase, s);
    mk_coords_destroy(c);
    set_error(MK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return MK_ERR_CUDA;
  };
  int32_t* first = (int32_t*)(sbase + o_cl);
  int32_t* slot_of = (int32_t*)(sbase + o_sl);
  unsigned long long* status = (unsigned long long*)(sbase + o_st);
  unsigned int* ticket = (unsigned int*)(sbase + o_ti);
  unsigned long long* err = (unsigned long long*)(sbase + o_er);
  if (deferred && n > 0) err = (unsigned long long*)(pbase + o_res);  // outlives the call
  int64_t* count = (int64_t*)(err + 1);

  cudaError_t e;
  ht.mark("alloc");
  if (use_sub && n > 0) {  // per-batch region layout (device side, before the table init)
    int32_t* hist = (int32_t*)(sbase + o_hi);
    if ((e = cudaMemsetAsync(hist, 0, sizeof(int32_t) * (kMaxSub + 2), s)) != cudaSuccess)
      return fail_cuda(e, "memset");
    pdl_launch(k_bhist<Src>, grid_for(n, kBlock, ctx->num_sms / 4 > 0 ? ctx->num_sms / 4 : 1), kBlock, 0, s, src, n,
               hist);
    pdl_launch(k_blayout, 1, 1024, 0, s, (const int32_t*)hist, cap, c->table.sub);
  } else if (use_sub) {
    const int2 flat = make_int2(0, -1);
    if ((e = cudaMemcpyAsync(c->table.sub, &flat, sizeof(flat), cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return fail_cuda(e, "layout");
  }
  {
    // status[ntiles], ticket, count are contiguous 8-byte words from o_st; err follows.
    unsigned long long* small = (unsigned long long*)(sbase + o_st);
    const int64_t n_small = (int64_t)((o_er - o_st) / 8);
    pdl_launch(k_init, grid_for(std::max<int64_t>((int64_t)nb * 4, n_small), 256, ctx->num_sms), 256, 0, s,
               c->table.buckets, first, nb, (const int2*)c->table.sub, small, n_small, err);
  }
  static const bool no_mailbox = [] {  // MK_NO_MAILBOX=1: D2H copy + stream sync (A/B measurement)
    const char* v = std::getenv("MK_NO_MAILBOX");
    return v && v[0] && v[0] != '0';
  }();
  unsigned long long seq = 0;
  Mailbox* mb = nullptr;
  if (deferred && n > 0) {
    mb = mailbox_ring_slot(ctx, &seq);
    if (!mb) deferred = false;  // no pinned ring: the eager path below
  }
  if (!deferred && n > 0 && !no_mailbox) mb = mailbox(&seq);
  if (n > 0) {
    ht.mark("init");
    pdl_launch(k_insert<Src>, grid_for(n, kBlock, ctx->num_sms), kBlock, 0, s, src, n, c->table.ref(D), first,
               slot_of, err);
    ht.mark("insert");
    pdl_launch(k_rank<Src>, (int)ntiles, kBlock, 0, s, src, n, (const int32_t*)first, (const int32_t*)slot_of,
               c->table.buckets, c->keys, d_first, d_p2r, status, ticket, count, (const unsigned long long*)err, mb,
               seq);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "launch");
  }
  if (deferred && n > 0) {
    c->mu = new std::mutex();
    c->mb = mb;
    c->seq = seq;
    c->d_res = err;
    c->n = -1;
    if ((e = cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventRecord(c->ev, s)) != cudaSuccess)
      return fail_cuda(e, "event");
    dev_free(c->alloc, sbase, s);
    *out = c;
    return MK_OK;
  }
  struct Result {
    unsigned long long err;
    int64_t count;
  };
  Result h{~0ull, 0};
  if (mb) {
    // The last k_rank tile posts (error word, row count) into the host-mapped mailbox: the
    // call returns as soon as the count is known, while the tail of k_rank still runs
    // (everything after it is ordered on the stream).
    dev_free(c->alloc, sbase, s);
    ht.mark("launched");
    if ((e = mailbox_wait(mb, seq, s)) != cudaSuccess) {
      mk_coords_destroy(c);
      set_error(MK_ERR_CUDA, std::string("coords: ") + cudaGetErrorString(e));
      return MK_ERR_CUDA;
    }
    h.err = mb->w0;
    h.count = (int64_t)mb->w1;
  } else if (n > 0) {
    Result* hr = (Result*)pinned_stage(sizeof(Result));
    if (!hr) return fail_cuda(cudaErrorMemoryAllocation, "pinned staging");
    // err and count are adjacent device words: one 16-byte copy
    if ((e = cudaMemcpyAsync(hr, err, sizeof(Result), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return fail_cuda(e, "D2H");
    dev_free(c->alloc, sbase, s);
    ht.mark("launched");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) {
      mk_coords_destroy(c);
      set_error(MK_ERR_CUDA, std::string("coords: ") + cudaGetErrorString(e));
      return MK_ERR_CUDA;
    }
    h = *hr;
  } else {
    dev_free(c->alloc, sbase, s);
    if ((e = cudaGetLastError()) != cudaSuccess) {
      mk_coords_destroy(c);
      set_error(MK_ERR_CUDA, std::string("coords: ") + cudaGetErrorString(e));
      return MK_ERR_CUDA;
    }
  }
  ht.mark("synced");
  if (h.err != ~0ull) {
    mk_coords_destroy(c);
    return report_input_error(h.err);
  }
  c->n = n > 0 ? h.count : 0;
  *out = c;
  return MK_OK;
}

bool valid_stream_dim(int32_t D) { return D >= 1 && D <= MK_MAX_DIM; }

}  // namespace

mk_status coords_resolve(const mk_coords* cc) {
  if (!cc || !cc->mu) return MK_OK;  // eager handle: count known
  mk_coords* c = const_cast<mk_coords*>(cc);  // the count is fixed by the build: logically const
  std::lock_guard<std::mutex> lock(*c->mu);
  if (c->n >= 0) return c->err == ~0ull ? MK_OK : report_input_error(c->err);
  unsigned long long err = ~0ull, count = 0;
  const volatile unsigned long long* vseq = &c->mb->seq;
  for (uint32_t it = 1;; ++it) {
    if (*vseq == c->seq) {
      std::atomic_thread_fence(std::memory_order_acquire);
      const volatile Mailbox* vm = c->mb;
      err = vm->w0;
      count = vm->w1;
      std::atomic_thread_fence(std::memory_order_acquire);
      if (*vseq == c->seq) break;  // not overwritten while reading (the writer zeroes seq first)
    }
    if ((it & 255u) == 0) {
      const cudaError_t q = cudaEventQuery(c->ev);
      if (q == cudaSuccess && *vseq != c->seq) {  // done, but the slot was reused: device words
        unsigned long long r[2];
        const cudaError_t e = cudaMemcpy(r, c->d_res, sizeof(r), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
          set_error(MK_ERR_CUDA, std::string("coords: ") + cudaGetErrorString(e));
          return MK_ERR_CUDA;
        }
        err = r[0];
        count = r[1];
        break;
      }
      if (q != cudaSuccess && q != cudaErrorNotReady) {
        set_error(MK_ERR_CUDA, std::string("coords: ") + cudaGetErrorString(q));
        return MK_ERR_CUDA;
      }
    }
  }
  c->err = err;
  c->n = err != ~0ull ? 0 : (int64_t)count;
  if (err != ~0ull) return report_input_error(err);
  return MK_OK;
}

namespace {

}  // namespace
}  // namespace mk

using namespace mk;

extern "C" {

mk_status mk_coords_quantize(mk_context* ctx, const float* d_points, const int32_t* d_batch, int64_t n,
                             int32_t D, float voxel, void* stream, mk_coords** out, int32_t* d_point_to_row,
                             int32_t* d_first_point) {
  clear_error();
  if (!ctx || !out || (n > 0 && !d_points)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_quantize: null argument");
  if (!valid_stream_dim(D)) MK_FAIL(D > MK_MAX_DIM ? MK_ERR_UNSUPPORTED : MK_ERR_INVALID_ARGUMENT,
                                    "mk_coords_quantize: D must be in 1..7");
  if (!(voxel > 0.0f) || !isfinite(voxel)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_quantize: voxel must be > 0");
  QuantSrc src{d_points, d_batch, D, voxel};
  const int32_t ts[kMaxD] = {1, 1, 1, 1, 1, 1, 1};
  return build_coords(ctx, src, n, D, ts, (cudaStream_t)stream, out, d_point_to_row, d_first_point);
}

mk_status mk_coords_quantize_deferred(mk_context* ctx, const float* d_points, const int32_t* d_batch, int64_t n,
                                      int32_t D, float voxel, void* stream, mk_coords** out, int32_t* d_point_to_row,
                                      int32_t* d_first_point) {
  clear_error();
  if (!ctx || !out || (n > 0 && !d_points)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_quantize_deferred: null argument");
  if (!valid_stream_dim(D)) MK_FAIL(D > MK_MAX_DIM ? MK_ERR_UNSUPPORTED : MK_ERR_INVALID_ARGUMENT,
                                    "mk_coords_quantize_deferred: D must be in 1..7");
  if (!(voxel > 0.0f) || !isfinite(voxel))
    MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_quantize_deferred: voxel must be > 0");
  QuantSrc src{d_points, d_batch, D, voxel};
  const int32_t ts[kMaxD] = {1, 1, 1, 1, 1, 1, 1};
  return build_coords(ctx, src, n, D, ts, (cudaStream_t)stream, out, d_point_to_row, d_first_point, true);
}

mk_status mk_coords_create(mk_context* ctx, const int32_t* d_coords, int64_t n, int32_t D,
                           const int32_t* h_tensor_stride, void* stream, mk_coords** out, int32_t* d_inverse) {
  clear_error();
  if (!ctx || !out || (n > 0 && !d_coords)) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_create: null argument");
  if (!valid_stream_dim(D)) MK_FAIL(D > MK_MAX_DIM ? MK_ERR_UNSUPPORTED : MK_ERR_INVALID_ARGUMENT,
                                    "mk_coords_create: D must be in 1..7");
  IntSrc src;
  src.rows = d_coords;
  src.D = D;
  int32_t ts[kMaxD] = {1, 1, 1, 1, 1, 1, 1};
  for (int d = 0; d < D; ++d) {
    ts[d] = h_tensor_stride ? h_tensor_stride[d] : 1;
    if (ts[d] < 1) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_create: tensor stride must be >= 1");
  }
  for (int d = 0; d < kMaxD; ++d) src.ts[d] = ts[d];
  return build_coords(ctx, src, n, D, ts, (cudaStream_t)stream, out, d_inverse, nullptr);
}

mk_status mk_coords_stride(mk_context* ctx, const mk_coords* in, const int32_t* h_conv_stride, void* stream,
                           mk_coords** out) {
  clear_error();
  if (!ctx || !in || !out || !h_conv_stride) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_stride: null argument");
  StrideSrc src;
  src.keys = in->keys;
  src.D = in->D;
  int32_t ts[kMaxD] = {1, 1, 1, 1, 1, 1, 1};
  for (int d = 0; d < in->D; ++d) {
    if (h_conv_stride[d] < 1) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_stride: stride must be >= 1");
    const int64_t s = (int64_t)in->tensor_stride[d] * h_conv_stride[d];
    if (s > INT32_MAX) MK_FAIL(MK_ERR_COORD_RANGE, "mk_coords_stride: tensor stride overflows int32");
    ts[d] = (int32_t)s;
    src.s[d] = s;
  }
  for (int d = in->D; d < kMaxD; ++d) src.s[d] = 1;
  const mk_status rs = coords_resolve(in);
  if (rs != MK_OK) return rs;
  return build_coords(ctx, src, in->n, in->D, ts, (cudaStream_t)stream, out, nullptr, nullptr);
}

mk_status mk_coords_expand(mk_context* ctx, const mk_coords* in, const mk_region* region,
                           const int32_t* h_out_stride, void* stream, mk_coords** out) {
  clear_error();
  if (!ctx || !in || !region || !out) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_expand: null argument");
  if (region->D != in->D) MK_FAIL(MK_ERR_DIMENSION_MISMATCH, "mk_coords_expand: region and coordinates differ in D");
  std::vector<int32_t> offs;
  int32_t K = 0;
  mk_status st = region_enumerate(region, &offs, &K);
  if (st != MK_OK) return st;
  const int D = in->D;
  ExpandSrc src;
  src.keys = in->keys;
  src.K = K;
  src.D = D;
  int32_t ts[kMaxD] = {1, 1, 1, 1, 1, 1, 1};
  for (int d = 0; d < kMaxD; ++d) src.s[d] = 1;
  for (int d = 0; d < D; ++d) {
    ts[d] = h_out_stride ? h_out_stride[d] : in->tensor_stride[d];
    if (ts[d] < 1) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_expand: output stride must be >= 1");
    if (in->tensor_stride[d] % ts[d] != 0)
      MK_FAIL(MK_ERR_STRIDE, "mk_coords_expand: the output stride must divide the input tensor stride");
    src.s[d] = ts[d];
  }
  st = coords_resolve(in);
  if (st != MK_OK) return st;
  const int64_t n = in->n * (int64_t)K;
  if (n > INT32_MAX) MK_FAIL(MK_ERR_UNSUPPORTED, "mk_coords_expand: more than 2^31 candidate rows");
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* d_offs = (int32_t*)dev_alloc(ctx->alloc, sizeof(int32_t) * K * D, s);
  int32_t* h = (int32_t*)pinned_stage(sizeof(int32_t) * K * D);
  if (!d_offs || !h) {
    if (d_offs) dev_free(ctx->alloc, d_offs, s);
    MK_FAIL(MK_ERR_OUT_OF_MEMORY, "mk_coords_expand: allocation failed");
  }
  std::copy(offs.begin(), offs.end(), h);
  if (cudaMemcpyAsync(d_offs, h, sizeof(int32_t) * K * D, cudaMemcpyHostToDevice, s) != cudaSuccess) {
    dev_free(ctx->alloc, d_offs, s);
    MK_FAIL(MK_ERR_CUDA, "mk_coords_expand: offset upload failed");
  }
  pinned_in_flight(s);
  src.offs = d_offs;
  st = build_coords(ctx, src, n, D, ts, s, out, nullptr, nullptr);
  dev_free(ctx->alloc, d_offs, s);
  return st;
}

mk_status mk_coords_info(const mk_coords* c, int64_t* n, int32_t* D, int32_t* h_tensor_stride) {
  clear_error();
  if (!c) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_info: null handle");
  if (n) {
    const mk_status rs = coords_resolve(c);
    if (rs != MK_OK) return rs;
    *n = c->n;
  }
  if (D) *D = c->D;
  if (h_tensor_stride)
    for (int d = 0; d < c->D; ++d) h_tensor_stride[d] = c->tensor_stride[d];
  return MK_OK;
}

mk_status mk_coords_export(const mk_coords* c, int32_t* d_out, void* stream) {
  clear_error();
  if (!c) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_export: null argument");
  const mk_status rs = coords_resolve(c);
  if (rs != MK_OK) return rs;
  if (c->n > 0 && !d_out) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_export: null argument");
  if (c->n == 0) return MK_OK;
  k_export<<<grid_for(c->n, 256, 148), 256, 0, (cudaStream_t)stream>>>(c->keys, c->n, c->D, d_out);
  MK_LAUNCH_CHECK();
  return MK_OK;
}

mk_status mk_coords_labels(const int32_t* d_point_to_row, const int32_t* d_first_point, const int32_t* d_labels,
                           int64_t n_points, int64_t n_rows, int32_t ignore_label, int32_t* d_row_labels, void* stream) {
  clear_error();
  if (n_points < 0 || n_rows < 0 || n_rows > n_points)
    MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_labels: bad sizes (0 <= n_rows <= n_points)");
  if (n_rows == 0) return MK_OK;
  if (!d_point_to_row || !d_first_point || !d_labels || !d_row_labels)
    MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_labels: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  k_labels_first<<<grid_for(n_rows, 256, 148), 256, 0, s>>>(d_first_point, d_labels, n_rows, d_row_labels);
  MK_LAUNCH_CHECK();
  k_labels_mark<<<grid_for(n_points, 256, 148), 256, 0, s>>>(d_point_to_row, d_first_point, d_labels, n_points,
                                                             ignore_label, d_row_labels);
  MK_LAUNCH_CHECK();
  return MK_OK;
}

mk_status mk_coords_lookup(const mk_coords* c, const int32_t* d_queries, int64_t q, int32_t* d_rows, void* stream) {
  clear_error();
  if (!c || q < 0 || (q > 0 && (!d_queries || !d_rows))) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_coords_lookup: bad argument");
  if (q == 0) return MK_OK;
  k_lookup<<<grid_for(q, 256, 148), 256, 0, (cudaStream_t)stream>>>(d_queries, q, c->D, c->table.ref(c->D), d_rows);
  MK_LAUNCH_CHECK();
  return MK_OK;
}

void mk_coords_destroy(mk_coords* c) {
  if (!c) return;
  for (void* p : c->owned) dev_free(c->alloc, p, c->stream);
  if (c->ev) cudaEventDestroy(c->ev);
  delete c->mu;
  delete c;
}

}  // extern "C"

