// mk_internal.cuh — shared internals of libmk (device key layout, hash table, handles,
// error plumbing).  Not part of the ABI; see include/mk.h for the public contract.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "mk.h"

namespace mk {

// ------------------------------------------------------------------ errors
struct Error {
  mk_status status;
  std::string msg;
  int64_t row;
};

void set_error(mk_status s, const std::string& msg, int64_t row = -1);
void clear_error();
extern std::atomic<int64_t> g_launches;

#define MK_CUDA_TRY(expr)                                                                  \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      ::mk::set_error(_e == cudaErrorMemoryAllocation ? MK_ERR_OUT_OF_MEMORY : MK_ERR_CUDA, \
                      std::string(#expr ": ") + cudaGetErrorString(_e));                   \
      return _e == cudaErrorMemoryAllocation ? MK_ERR_OUT_OF_MEMORY : MK_ERR_CUDA;         \
    }                                                                                      \
  } while (0)

#define MK_LAUNCH_CHECK()                                                                  \
  do {                                                                                     \
    ::mk::g_launches.fetch_add(1, std::memory_order_relaxed);                              \
    MK_CUDA_TRY(cudaGetLastError());                                                       \
  } while (0)

#define MK_FAIL(status, msg)                 \
  do {                                       \
    ::mk::set_error((status), (msg));        \
    return (status);                         \
  } while (0)

// ------------------------------------------------------------------ launches
// Programmatic dependent launch (PDL).  A kernel started by pdl_launch() may be scheduled
// while its predecessor on the stream is still running, so it calls pdl_wait() in every CTA
// before it reads or writes global memory that earlier work touches (griddepcontrol.wait
// returns once the predecessor grid has completed and its writes are visible; it is a no-op
// for a normal launch).  pdl_trigger() lets the next PDL kernel be scheduled once every CTA
// of this grid has called it or exited.  Since every PDL kernel waits in every CTA, a
// kernel's completion implies the completion of everything before it on the stream.
// MK_NO_PDL=1 launches normally (A/B measurement).
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// The common prologue of a PDL kernel: wait for the predecessor, then let the successor in.
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

// ------------------------------------------------------------------ keys
// A coordinate row (u_1..u_D, b) is packed into one 128-bit key (int4) so that a table
// slot is a single 16-byte load (coalesced 128-bit coordinate access):
//   D <= 3 : (u_1, u_2, u_3, b)  with missing axes 0
//   D == 4 : (u_1, u_2, u_3, (u_4 << 16) | b)  with u_4 in [-2^15, 2^15), b <= 65534
// The empty sentinel is all ones; no valid key has w == -1 (b >= 0, and b != 0xFFFF
// for D == 4).
constexpr int32_t kEmptyWord = -1;

// Multiply-xor combine of the four key words and a murmur3 32-bit finaliser (cheap: the
// kernel-map builder hashes every (row, offset) query).
__host__ __device__ __forceinline__ uint32_t hash_key(int4 k) {
  uint32_t h = (uint32_t)k.x * 0x9E3779B1u;
  h ^= (uint32_t)k.y * 0x85EBCA77u;
  h = (h << 13) | (h >> 19);
  h ^= (uint32_t)k.z * 0xC2B2AE3Du;
  h ^= (uint32_t)k.w * 0x27D4EB2Fu;
  h ^= h >> 16;
  h *= 0x7FEB352Du;
  h ^= h >> 15;
  h *= 0x846CA68Bu;
  h ^= h >> 16;
  return h;
}

__host__ __device__ __forceinline__ bool key_eq(int4 a, int4 b) {
  return a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w;
}

// Largest D of the GPU path and the packed-key layouts (one 128-bit key per row):
//   D <= 3 : (u_0, u_1, u_2, b)                               missing axes 0
//   D == 4 : (u_0, u_1, u_2, u_3 << 16 | b)                   u_3 in [-2^15, 2^15), b <= 65534
//   D 5..7 : (u_0 << 12 | u_3, u_1 << 12 | u_4, u_2 << 12 | u_5, u_6 << 16 | b)
//            u_0..u_2 in [-2^19, 2^19) (20 bits), u_3..u_5 in [-2^11, 2^11) (12 bits),
//            u_6 in [-2^15, 2^15), b <= 65534 when D == 7 (else word 3 = b) — the 7D
//            space-time-chroma lattice of the TS-CRF (3D space, 3D colour, time).
constexpr int kMaxD = 7;

// Component d of a packed key.
__host__ __device__ __forceinline__ int32_t key_axis(int4 k, int D, int d) {
  const int32_t w = d == 0 ? k.x : d == 1 ? k.y : d == 2 ? k.z : k.w;
  if (D <= 3) return w;
  if (D == 4) return d < 3 ? w : (int32_t)(int16_t)((uint32_t)k.w >> 16);
  if (d < 3) return w >> 12;                                       // arithmetic: 20-bit signed
  if (d < 6) {
    const int32_t v = d == 3 ? k.x : d == 4 ? k.y : k.z;
    return (int32_t)((uint32_t)v << 20) >> 20;                      // 12-bit signed
  }
  return (int32_t)(int16_t)((uint32_t)k.w >> 16);                  // d == 6
}
__host__ __device__ __forceinline__ int32_t key_batch(int4 k, int D) {
  return (D == 4 || D == 7) ? (int32_t)((uint32_t)k.w & 0xFFFFu) : k.w;
}
// Packs components c[0..D) (int64, already range-checked by the caller for int32) and
// batch b.  Returns false when a component or b does not fit the layout above.
__host__ __device__ __forceinline__ bool pack_key(const int64_t* c, int D, int64_t b, int4* out) {
  // c[] is indexed with compile-time constants only (keeps it in registers)
  int4 k;
  if (D <= 4) {
    k.x = D > 0 ? (int32_t)c[0] : 0;
    k.y = D > 1 ? (int32_t)c[1] : 0;
    k.z = D > 2 ? (int32_t)c[2] : 0;
    if (D == 4) {
      if (c[3] < -32768 || c[3] > 32767 || b < 0 || b > 65534) return false;
      k.w = (int32_t)(((uint32_t)(uint16_t)(int16_t)c[3] << 16) | (uint32_t)b);
    } else {
      if (b < 0 || b > INT32_MAX) return false;
      k.w = (int32_t)b;
    }
  } else {
    const int64_t hi = 1 << 19, lo = 1 << 11;
    if (c[0] < -hi || c[0] >= hi || c[1] < -hi || c[1] >= hi || c[2] < -hi || c[2] >= hi) return false;
    const int64_t c3 = c[3], c4 = c[4], c5 = D > 5 ? c[5] : 0, c6 = D > 6 ? c[6] : 0;
    if (c3 < -lo || c3 >= lo || c4 < -lo || c4 >= lo || c5 < -lo || c5 >= lo) return false;
    k.x = (int32_t)(((uint32_t)c[0] << 12) | ((uint32_t)c3 & 0xFFFu));
    k.y = (int32_t)(((uint32_t)c[1] << 12) | ((uint32_t)c4 & 0xFFFu));
    k.z = (int32_t)(((uint32_t)c[2] << 12) | ((uint32_t)c5 & 0xFFFu));
    if (D == 7) {
      if (c6 < -32768 || c6 > 32767 || b < 0 || b > 65534) return false;
      k.w = (int32_t)(((uint32_t)(uint16_t)(int16_t)c6 << 16) | (uint32_t)b);
    } else {
      if (b < 0 || b > INT32_MAX) return false;
      k.w = (int32_t)b;
    }
  }
  *out = k;
  return true;
}

// ------------------------------------------------------------------ hash table
// Open addressing over 64-byte buckets (half a 128-byte line) of three 16-byte key slots
// and one 16-byte word holding the three slots' row values, laid out so that the first
// 32-byte sector holds key slot 0 and the rows:
//   bucket b = { key[0], (row[0], row[1], row[2], unused), key[1], key[2] }
// A key hashes to bucket hash_bucket(hash, buckets) and is stored in the first free slot of the
// linear-probing sequence of slots 3b, 3b+1, ... (wrapping), so the occupied slots of a
// bucket are a prefix and, once the table is built, row[j] >= 0 exactly when slot j is
// occupied.  A lookup reads the first sector (key 0 + rows) and stops there unless key 0
// is another key and slot 1 is occupied (rare at the table's load factor <= 1/2); only then
// it reads keys 1-2, and continues to the next bucket only when all three slots hold other
// keys.
constexpr int kSlotsPerBucket = 3;

__host__ __device__ __forceinline__ int4* slot_key(int4* buckets, uint32_t slot) {
  const uint32_t j = slot % 3u;
  return buckets + (size_t)(slot / 3u) * 4u + (j ? j + 1u : 0u);
}
__host__ __device__ __forceinline__ int32_t* slot_val(int4* buckets, uint32_t slot) {
  return (int32_t*)(buckets + (size_t)(slot / 3u) * 4u + 1u) + slot % 3u;
}

// One 32-byte sector in one 256-bit load (sm_100 LDG.E.ENL2.256).
__device__ __forceinline__ void load_sector(const int4* p, int4* a, int4* b) {
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(a->x), "=r"(a->y), "=r"(a->z), "=r"(a->w), "=r"(b->x), "=r"(b->y), "=r"(b->z), "=r"(b->w)
      : "l"(p));
}

// Lookup of q in bucket B given its first sector (k0, v): row, -1 (absent), or -2 (all three
// slots hold other keys: continue with the next bucket).
__device__ __forceinline__ int32_t bucket_rest(const int4* B, int4 q, int4 k0, int4 v) {
  if (key_eq(k0, q)) return v.x;
  if (k0.w == kEmptyWord || v.y < 0) return -1;  // slot 1 empty (occupied slots are a prefix)
  const int4 k1 = __ldg(B + 2);
  if (key_eq(k1, q)) return v.y;
  if (v.z < 0) return -1;
  const int4 k2 = __ldg(B + 3);
  if (key_eq(k2, q)) return v.z;
  return -2;
}

// Bucket of hash h in a region of `size` buckets: the high bits of h scaled to the size
// (multiply-shift; the regions need not be powers of two).
__host__ __device__ __forceinline__ uint32_t hash_bucket(uint32_t h, uint32_t size) {
  return (uint32_t)(((uint64_t)h * size) >> 32);
}

// Per-batch regions.  A large table (many scans in one batch, configs[4]) is split into one
// region per batch index, each sized from that batch's rows, so that the inserts and the
// kernel-map probes of one scan — issued in row order, i.e. scan after scan — touch one
// L2-sized region instead of a table far larger than L2.  The layout lives on the device
// (computed from a histogram of the batch indices, no host round trip):
//   sub[0] = (nsub, used buckets), sub[1 + b] = (first bucket, buckets) of batch b;
// nsub = 0 means one flat region (the table's nb buckets).  Within a region the probing
// sequence wraps inside the region.  Keys of a batch >= nsub are absent by construction.
struct TableRef {
  const int4* buckets;
  uint32_t nb;       // flat table: buckets
  const int2* sub;   // per-batch layout (see above) or null
  int D;             // key layout (for the batch field)
  // region of key q: false when q cannot be in the table (its batch has no region)
  __device__ __forceinline__ bool region(int4 q, uint32_t* base, uint32_t* size) const {
    if (sub) {
      const int nsub = __ldg(&sub[0].x);
      if (nsub > 0) {
        const uint32_t b = (uint32_t)key_batch(q, D);
        if (b >= (uint32_t)nsub) return false;
        const int2 r = __ldg(sub + 1 + b);
        *base = (uint32_t)r.x;
        *size = (uint32_t)r.y;
        return true;
      }
    }
    *base = 0;
    *size = nb;
    return true;
  }
};

// Continues the lookup of q after bucket b0 (which was full of other keys) in its region.
static __device__ __noinline__ int32_t probe_next(const int4* __restrict__ buckets, uint32_t base, uint32_t size,
                                                  int4 q, uint32_t b0) {
  uint32_t j = b0 - base;
  while (true) {
    j = j + 1 == size ? 0u : j + 1;
    const int4* B = buckets + (size_t)(base + j) * 4u;
    const int32_t r = bucket_rest(B, q, __ldg(B), __ldg(B + 1));
    if (r != -2) return r;
  }
}

// Thread-level lookup of key q; row or -1.
__device__ __forceinline__ int32_t probe(const TableRef& t, int4 q) {
  uint32_t base, size;
  if (!t.region(q, &base, &size)) return -1;
  const uint32_t b = base + hash_bucket(hash_key(q), size);
  const int4* B = t.buckets + (size_t)b * 4u;
  int4 k0, v;
  load_sector(B, &k0, &v);
  const int32_t r = bucket_rest(B, q, k0, v);
  return r != -2 ? r : probe_next(t.buckets, base, size, q, b);
}

// ------------------------------------------------------------------ handles
constexpr int kMaxSub = 4096;  // batches with their own region (larger batch indices: flat table)
struct Table {
  int4* buckets = nullptr;  // [nb][4] (see "hash table" above)
  uint32_t bmask = 0;       // nb - 1 of the flat table (nb is a power of two; 3 nb >= 2n slots)
  int2* sub = nullptr;      // per-batch region layout [1 + kMaxSub] (device) or null
  TableRef ref(int D) const { return TableRef{buckets, bmask + 1u, sub, D}; }
};

struct Alloc {
  mk_alloc_fn alloc = nullptr;
  mk_free_fn free_fn = nullptr;
  void* user = nullptr;
};

}  // namespace mk

namespace mk {
struct Mailbox;  // host-mapped result slot (below)
}  // namespace mk

struct mk_context {
  int device = 0;
  int num_sms = 148;
  int64_t l2_bytes = 126 << 20;  // device L2 size (cudaDeviceProp::l2CacheSize)
  mk::Alloc alloc;
  cudaStream_t aux = nullptr;  // private non-blocking stream for small lazy read-backs
  cudaStream_t side = nullptr;  // private non-blocking stream: map-build work forked off the caller's stream
  // Grow-only scratch buffer for the per-call weight-gradient partials (tens of MB, allocated
  // and freed every call otherwise: the stream-ordered pool then maps new memory every few
  // calls, a 0.3-2.5 ms host stall).  scratch_acquire() holds scratch_mu until
  // scratch_release(); a call on another stream than the last user first waits for its event.
  std::mutex scratch_mu;
  void* scratch = nullptr;
  size_t scratch_cap = 0;
  cudaStream_t scratch_stream = nullptr;
  cudaEvent_t scratch_ev = nullptr;
  // Device copies of kernel-region tables (offsets, then mirror indices), uploaded once per
  // region and kept for the context's lifetime (mk::region_device).
  std::mutex region_mu;
  std::vector<std::pair<std::vector<int32_t>, int32_t*>> region_dev;
  // Grid-barrier words of the cooperative sort: kBarSlots pairs, zero-initialised; a call
  // takes the next pair round robin (concurrent calls on different streams get different
  // pairs as long as fewer than kBarSlots sorts are in flight).
  // Host-mapped mailbox ring of the deferred quantize (lazily allocated, kMbSlots slots).
  static constexpr unsigned kMbSlots = 1024;
  mk::Mailbox* mb_ring = nullptr;
  std::atomic<unsigned long long> mb_seq{0};
  static constexpr unsigned kBarSlots = 256;
  unsigned* d_bar = nullptr;
  std::atomic<unsigned> bar_next{0};
  unsigned* barrier_slot() { return d_bar ? d_bar + 2 * (bar_next.fetch_add(1) % kBarSlots) : nullptr; }
};

struct mk_coords {
  mk::Alloc alloc;
  cudaStream_t stream = nullptr;  // stream the handle was created on (frees are ordered there)
  // Row count; -1 while pending (mk_coords_quantize_deferred): mk::coords_resolve reads it
  // from the mailbox slot (mb, seq) or, if the slot was reused, from the device words d_res
  // (error word, count) once the build event has completed.  Guarded by mu.
  int64_t n = 0;
  mk::Mailbox* mb = nullptr;
  unsigned long long seq = 0;
  unsigned long long err = ~0ull;  // input error found by a deferred build (reported at every use)
  const unsigned long long* d_res = nullptr;
  cudaEvent_t ev = nullptr;
  std::mutex* mu = nullptr;
  int32_t D = 0;
  int32_t tensor_stride[MK_MAX_DIM] = {1, 1, 1, 1, 1, 1, 1};
  int4* keys = nullptr;  // [n] packed rows, row order = first occurrence
  mk::Table table;
  std::vector<void*> owned;
};

struct mk_kmap {
  mk::Alloc alloc;
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;       // the context's private stream (lazy read-backs)
  int num_sms = 148;
  // Host-side counts are materialised lazily (mk::kmap_host / mk::kmap_wplan), guarded by
  // `mu`: the handle stays logically immutable (the values are fixed by the build).
  std::mutex* mu = nullptr;
  cudaEvent_t done = nullptr;       // recorded after the build's last kernel
  int64_t* d_totals = nullptr;      // [K] pairs per offset (device)
  bool host_ready = false;
  bool wplan_ready = false;
  cudaEvent_t wplan_ev = nullptr;   // recorded after the split-K plan upload
  cudaStream_t wplan_stream = nullptr;
  int32_t K = 0;
  int32_t D = 0;
  int32_t transposed = 0;
  int64_t n_in = 0, n_out = 0, n_pairs = 0;
  std::vector<int64_t> h_ptr;       // [K+1] host copy of the CSR offsets
  int64_t* ptr = nullptr;           // [K+1]
  int32_t* in_idx = nullptr;        // [n_pairs]
  int32_t* out_idx = nullptr;       // [n_pairs]
  // Dense neighbour tables used by the output-stationary convolution kernels:
  //   nbr[k][o]  = input row paired with output o at offset k, or -1       (forward)
  //   nbrT[k][a] = output row paired with input a at offset k, or -1        (dgrad)
  // When in == out (submanifold) and N^D is closed under negation, nbrT[k] == nbr[mirror[k]]
  // and nbrT is not stored (nbrT == nullptr).
  int32_t* nbr = nullptr;
  int32_t* nbrT = nullptr;
  int64_t nbr_stride = 0;   // rows of nbr, padded to a multiple of 128 (padding = -1)
  // Internal row order of the conv tiles (bitmask-sorted when K <= 32, else NULL = identity):
  // nbr / nbrT / the tile masks are stored in this order; position i holds row perm[i].
  int32_t* perm = nullptr;
  int32_t* permT = nullptr;
  int64_t nbrT_stride = 0;  // rows of the dgrad table (nbrT or, when symmetric, nbr)
  std::vector<int32_t> mirror;      // [K] index of -offset_k, or -1
  const int32_t* d_mirror = nullptr;     // [K]
  // Per 128-row tile bitmasks of non-empty offsets (mask words = ceil(K/32)):
  uint32_t* tile_mask = nullptr;    // [ceil(n_out/128)][mw]  forward tiles
  uint32_t* tile_maskT = nullptr;   // [ceil(n_in/128)][mw]   dgrad tiles (mirrored when symmetric)
  int32_t mask_words = 1;
  // Split-K plan of the weight gradient (tensor-core path): the concatenated pair list is
  // cut into n_wcta contiguous ranges; wseg = (k, begin, end, slot) for every non-empty
  // (range, offset) intersection, grouped by range (wseg_begin[n_wcta+1]); slots are in
  // offset order, wslot_begin[k] = first slot of offset k ([K+1]).
  int4* wseg = nullptr;
  int32_t* wseg_begin = nullptr;
  int32_t* wslot_begin = nullptr;
  int64_t n_wslots = 0;
  int32_t n_wcta = 0;
  std::vector<void*> owned;
};

namespace mk {
// Development aid: MK_HOST_TIMING=1 prints host-side timestamps of a call's stages (us).
struct HostTimer {
  const char* name;
  bool on;
  int n = 0;
  const char* lab[16];
  double t[16];
  static double now();
  explicit HostTimer(const char* nm);
  void mark(const char* l) {
    if (on && n < 16) {
      lab[n] = l;
      t[n++] = now();
    }
  }
  ~HostTimer();
};
void* dev_alloc(const Alloc& a, size_t bytes, cudaStream_t s);
void* scratch_acquire(mk_context* ctx, size_t bytes, cudaStream_t s);  // nullptr on failure (lock released)
void scratch_release(mk_context* ctx, cudaStream_t s);
void dev_free(const Alloc& a, void* p, cudaStream_t s);
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
uint32_t next_pow2(uint64_t v);
// Thread-local pinned staging buffer (context.cu).  pinned_stage() waits until the previous
// async copy that used it has completed; pinned_in_flight(s) marks it busy until `s`
// reaches the current point.
void* pinned_stage(size_t bytes);
void pinned_in_flight(cudaStream_t s);

// Host-mapped mailbox (context.cu): a kernel posts a few result words straight into pinned
// host memory, so a call that needs them on the host spins on a sequence number instead of
// a device->host copy plus a stream synchronize.  One mailbox per host thread (calls that
// wait on it are synchronous); the device pointer equals the host pointer under UVA.
struct Mailbox {
  unsigned long long seq;  // written last (release), polled by the host
  unsigned long long w0, w1, w2;
};
Mailbox* mailbox(unsigned long long* next_seq);  // nullptr if pinned memory is unavailable
// A slot of the context's mailbox ring for a deferred count (its sequence number in *seq);
// nullptr if the ring cannot be allocated.
Mailbox* mailbox_ring_slot(mk_context* ctx, unsigned long long* seq);
// Waits until mb->seq == seq, watching `s` for errors; returns cudaSuccess once posted.
cudaError_t mailbox_wait(const Mailbox* mb, unsigned long long seq, cudaStream_t s);
__device__ __forceinline__ void mailbox_post(Mailbox* mb, unsigned long long seq, unsigned long long w0,
                                             unsigned long long w1) {
  // seqlock writer: the slot is marked as being written (seq 0, never a valid sequence
  // number) before its words change, so a host reader of an older call that checks seq before
  // and after reading w0 / w1 can never accept a newer call's words (ring slots are reused
  // every kMbSlots calls)
  volatile Mailbox* v = mb;
  v->seq = 0ull;
  __threadfence_system();
  v->w0 = w0;
  v->w1 = w1;
  __threadfence_system();
  v->seq = seq;
}

// Table-building pipeline shared by quantize / create / stride (coords.cu).
// Region enumeration (region.cu):
mk_status region_enumerate(const mk_region* r, std::vector<int32_t>* offsets, int32_t* K);
// Lazy host state of a kernel map (kmap.cu): h_ptr / n_pairs, and the bf16 weight-gradient
// split-K plan (uploaded on `s`; other streams wait for it).
mk_status kmap_host(const mk_kmap* m);
mk_status kmap_wplan(const mk_kmap* m, cudaStream_t s);
constexpr int kWgradMaxSegs = 63;  // segments per CTA of the bf16 weight-gradient kernel
// Stable radix sort of keys (low `bits` bits) -> permutation (sort.cu).  Clobbers keys.
// bar: two zero-initialised device words private to this call's stream (grid barrier of
// the one-kernel cooperative sort), or nullptr for the three-kernels-per-pass path.
// Resolves a deferred row count (no-op when known); on an input error reports it like the
// eager quantize (status + message) and leaves the handle with 0 rows.
mk_status coords_resolve(const mk_coords* c);

mk_status radix_sort_perm(const Alloc& a, uint32_t* keys, int64_t n, int bits, int32_t* perm, cudaStream_t s,
                          unsigned* bar = nullptr, int num_sms = 148);
}  // namespace mk
