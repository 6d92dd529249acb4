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
#include <map>

#include "mk_internal.cuh"

namespace mk {
namespace {

constexpr int kTileRows = 128;
constexpr int kThreads = 256;

// u + sign * off * scale, per spatial axis, batch unchanged (R18).  False when the
// shifted coordinate cannot exist (outside int32 or the packed-key domain).
__device__ __forceinline__ bool shift_key(int4 u, int D, const int32_t* off, int sign, int4 scale, int4* q) {
  int64_t c[4] = {0, 0, 0, 0};
  const int32_t sc[4] = {scale.x, scale.y, scale.z, scale.w};
#pragma unroll
  for (int d = 0; d < 4; ++d) {  // fully unrolled: c[] and sc[] stay in registers
    if (d < D) {
      const int64_t v = (int64_t)key_axis(u, D, d) + (int64_t)sign * off[d] * sc[d];
      if (v < INT32_MIN || v > INT32_MAX) return false;
      c[d] = v;
    }
  }
  return pack_key(c, D, key_batch(u, D), q);
}

__global__ void __launch_bounds__(kThreads) k_probe(const int4* __restrict__ okeys, int64_t n_out, int64_t n_pad,
                                                    const int4* __restrict__ tkeys, const int32_t* __restrict__ tvals,
                                                    uint32_t mask, const int32_t* __restrict__ offs, int K, int D,
                                                    int sign, int4 scale4, int32_t* __restrict__ nbr,
                                                    int32_t* __restrict__ tile_cnt, int64_t ntiles,
                                                    uint32_t* __restrict__ tile_mask, int mw,
                                                    uint32_t* __restrict__ rowmask) {
  extern __shared__ int32_t sm[];
  int32_t* s_off = sm;              // [K*D]
  int32_t* s_cnt = sm + K * D;      // [K]
  uint32_t* s_rm = (uint32_t*)(s_cnt + K);  // [128] row masks (K <= 32)
  for (int i = threadIdx.x; i < K * D; i += kThreads) s_off[i] = offs[i];
  for (int i = threadIdx.x; i < K; i += kThreads) s_cnt[i] = 0;
  if (threadIdx.x < kTileRows) s_rm[threadIdx.x] = 0;
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t o = tile * kTileRows + (threadIdx.x & (kTileRows - 1));
  const bool valid = o < n_out;
  int4 u = make_int4(0, 0, 0, 0);
  if (valid) u = okeys[o];
  uint32_t rm = 0;
  for (int k = threadIdx.x / kTileRows; k < K; k += kThreads / kTileRows) {
    int32_t a = -1;
    int4 q;
    if (valid && shift_key(u, D, s_off + k * D, sign, scale4, &q)) a = probe(tkeys, tvals, mask, q);
    nbr[(int64_t)k * n_pad + o] = a;  // rows padded to whole tiles (-1)
    if (a >= 0 && k < 32) rm |= 1u << k;
    const unsigned b = __ballot_sync(0xffffffffu, a >= 0);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(s_cnt + k, __popc(b));
  }
  if (rowmask) atomicOr(s_rm + (threadIdx.x & (kTileRows - 1)), rm);
  __syncthreads();
  if (rowmask && threadIdx.x < kTileRows && valid) rowmask[o] = s_rm[threadIdx.x];
  for (int k = threadIdx.x; k < K; k += kThreads) tile_cnt[(int64_t)k * ntiles + tile] = s_cnt[k];
  for (int w = threadIdx.x; w < mw; w += kThreads) {
    uint32_t bits = 0;
    for (int j = 0; j < 32 && w * 32 + j < K; ++j) bits |= (s_cnt[w * 32 + j] > 0 ? 1u : 0u) << j;
    tile_mask[tile * mw + w] = bits;
  }
}

__global__ void __launch_bounds__(1024) k_scan(const int32_t* __restrict__ tile_cnt, int64_t ntiles,
                                               int64_t* __restrict__ tile_off, int64_t* __restrict__ totals) {
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

__global__ void __launch_bounds__(kThreads) k_emit(const int32_t* __restrict__ nbr, int64_t n_out, int64_t n_pad, int K,
                                                   const int64_t* __restrict__ ptr, const int64_t* __restrict__ tile_off,
                                                   int64_t ntiles, int32_t* __restrict__ in_idx,
                                                   int32_t* __restrict__ out_idx, int32_t* __restrict__ nbrT,
                                                   int64_t nT_pad, uint32_t* __restrict__ tile_maskT, int mw) {
  extern __shared__ int32_t s_wc[];  // [K][4] pairs per (offset, warp of the tile)
  const int64_t tile = blockIdx.x;
  const int r = threadIdx.x & (kTileRows - 1);
  const int64_t o = tile * kTileRows + r;
  const bool valid = o < n_out;
  const int lane = threadIdx.x & 31, wq = r >> 5;  // warp quarter of the 128-row tile
  const unsigned lt = (1u << lane) - 1u;
  for (int k = threadIdx.x / kTileRows; k < K; k += kThreads / kTileRows) {
    const int32_t a = valid ? nbr[(int64_t)k * n_pad + o] : -1;
    const unsigned b = __ballot_sync(0xffffffffu, a >= 0);
    if (lane == 0) s_wc[k * 4 + wq] = __popc(b);
  }
  __syncthreads();
  for (int k = threadIdx.x / kTileRows; k < K; k += kThreads / kTileRows) {
    const int32_t a = valid ? nbr[(int64_t)k * n_pad + o] : -1;
    const unsigned b = __ballot_sync(0xffffffffu, a >= 0);
    if (a < 0) continue;
    int64_t pos = ptr[k] + tile_off[(int64_t)k * ntiles + tile] + __popc(b & lt);
    for (int w = 0; w < wq; ++w) pos += s_wc[k * 4 + w];
    in_idx[pos] = a;
    out_idx[pos] = (int32_t)o;
    if (nbrT) {
      nbrT[(int64_t)k * nT_pad + a] = (int32_t)o;
      atomicOr(tile_maskT + (int64_t)(a / kTileRows) * mw + (k >> 5), 1u << (k & 31));
    }
  }
}

// Row masks of the dgrad table: bit k set when nbrT[k][a] >= 0 (K <= 32).
__global__ void k_rowmask_T(const int32_t* __restrict__ nbrT, int64_t stride, int64_t n, int K,
                            uint32_t* __restrict__ rowmask) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    uint32_t rm = 0;
    for (int k = 0; k < K; ++k) rm |= (nbrT[(int64_t)k * stride + a] >= 0 ? 1u : 0u) << k;
    rowmask[a] = rm;
  }
}

// Neighbour table in permuted row order: out[k][i] = tab[k][perm[i]] (padding rows -1), and
// the active-offset mask of every permuted 128-row tile (K <= 32: one word).
__global__ void __launch_bounds__(kTileRows) k_permute(const int32_t* __restrict__ tab, int64_t stride, int64_t n,
                                                       int K, const int32_t* __restrict__ perm,
                                                       int32_t* __restrict__ out, uint32_t* __restrict__ tmask) {
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

}  // namespace
}  // namespace mk

using namespace mk;

extern "C" {

mk_status mk_kmap_build(mk_context* ctx, const mk_coords* in, const mk_coords* out, const mk_region* region,
                        int32_t transposed, void* stream_, mk_kmap** out_map) {
  clear_error();
  cudaStream_t s = (cudaStream_t)stream_;
  if (!ctx || !in || !out || !region || !out_map) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_kmap_build: null argument");
  if (in->D != out->D || region->D != in->D)
    MK_FAIL(MK_ERR_DIMENSION_MISMATCH, "mk_kmap_build: input, output and region must have the same D");
  const int D = in->D;
  std::vector<int32_t> offs;
  int32_t K = 0;
  mk_status st = region_enumerate(region, &offs, &K);
  if (st != MK_OK) return st;
  if (K > 4096) MK_FAIL(MK_ERR_UNSUPPORTED, "mk_kmap_build: more than 4096 kernel offsets");

  mk_kmap* m = new mk_kmap();
  m->alloc = ctx->alloc;
  m->stream = s;
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
  const int4 scale4 = make_int4(sc[0], D > 1 ? sc[1] : 1, D > 2 ? sc[2] : 1, D > 3 ? sc[3] : 1);
  const int sign = transposed ? -1 : 1;

  // mirror[k]: index of -offset_k (used to reuse nbr for dgrad on submanifold maps)
  std::map<std::vector<int32_t>, int32_t> index;
  for (int k = 0; k < K; ++k) index[std::vector<int32_t>(offs.begin() + k * D, offs.begin() + (k + 1) * D)] = k;
  m->mirror.assign(K, -1);
  bool symmetric = (in == out);
  for (int k = 0; k < K; ++k) {
    std::vector<int32_t> neg(D);
    for (int d = 0; d < D; ++d) neg[d] = -offs[k * D + d];
    auto it = index.find(neg);
    if (it == index.end()) symmetric = false;
    else m->mirror[k] = it->second;
  }

  const int64_t n_out = out->n, n_in = in->n;
  const int64_t ntiles = std::max<int64_t>(1, ceil_div(n_out, kTileRows));
  const int64_t ntilesT = std::max<int64_t>(1, ceil_div(n_in, kTileRows));
  const int64_t n_pad = ntiles * kTileRows, nT_pad = ntilesT * kTileRows;  // table rows padded to whole tiles
  m->nbr_stride = n_pad;
  m->nbrT_stride = symmetric ? n_pad : nT_pad;

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

  // persistent: offsets/mirror, ptr, nbr, tile masks (+ nbrT / maskT when not symmetric)
  int32_t* d_offs = (int32_t*)alloc(sizeof(int32_t) * (K * D + K));  // offsets, then mirror
  m->d_mirror = d_offs ? d_offs + K * D : nullptr;
  m->nbr = (int32_t*)alloc(sizeof(int32_t) * (int64_t)K * n_pad);
  m->tile_mask = (uint32_t*)alloc(sizeof(uint32_t) * ntiles * mw);
  m->tile_maskT = (uint32_t*)alloc(sizeof(uint32_t) * ntilesT * mw);
  if (!symmetric) m->nbrT = (int32_t*)alloc(sizeof(int32_t) * (int64_t)K * nT_pad);
  // scratch: tile counts, tile offsets, totals
  void* scratch = dev_alloc(m->alloc, sizeof(int32_t) * K * ntiles + sizeof(int64_t) * K * ntiles + 256 +
                                          sizeof(int64_t) * K, s);
  if (!m->d_mirror || !d_offs || !m->nbr || !m->tile_mask || !m->tile_maskT || (!symmetric && !m->nbrT) ||
      !scratch) {
    if (scratch) dev_free(m->alloc, scratch, s);
    return fail(MK_ERR_OUT_OF_MEMORY, "mk_kmap_build: device allocation failed");
  }
  // Row masks for the bitmask ordering of the conv tiles (K <= 32 offsets only).
  const bool sort_rows = K <= 32;
  uint32_t* rowmask = sort_rows ? (uint32_t*)dev_alloc(m->alloc, sizeof(uint32_t) * std::max<int64_t>(1, std::max(n_out, n_in)), s) : nullptr;
  if (sort_rows && !rowmask) {
    dev_free(m->alloc, scratch, s);
    return fail(MK_ERR_OUT_OF_MEMORY, "mk_kmap_build: device allocation failed");
  }
  int64_t* tile_off = (int64_t*)scratch;
  int64_t* totals = tile_off + K * ntiles;
  int32_t* tile_cnt = (int32_t*)(totals + K);

  cudaError_t e = cudaSuccess;
  auto ck = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
  };
  {  // one pinned H2D copy of the offsets and their mirror indices
    int32_t* h = (int32_t*)pinned_stage(sizeof(int32_t) * (K * D + K));
    if (!h) {
      dev_free(m->alloc, scratch, s);
      return fail(MK_ERR_OUT_OF_MEMORY, "mk_kmap_build: pinned staging failed");
    }
    std::copy(offs.begin(), offs.end(), h);
    std::copy(m->mirror.begin(), m->mirror.end(), h + K * D);
    ck(cudaMemcpyAsync(d_offs, h, sizeof(int32_t) * (K * D + K), cudaMemcpyHostToDevice, s));
    pinned_in_flight(s);
  }
  if (!symmetric) {
    ck(cudaMemsetAsync(m->nbrT, 0xFF, sizeof(int32_t) * K * nT_pad, s));
    ck(cudaMemsetAsync(m->tile_maskT, 0, sizeof(uint32_t) * ntilesT * mw, s));
  }
  if (n_out > 0) {
    k_probe<<<(unsigned)ntiles, kThreads, sizeof(int32_t) * (K * D + K + kTileRows), s>>>(
        out->keys, n_out, n_pad, in->table.keys, in->table.vals, in->table.mask, d_offs, K, D, sign, scale4, m->nbr,
        tile_cnt, ntiles, m->tile_mask, mw, rowmask);
    g_launches++;
    k_scan<<<K, 1024, 0, s>>>(tile_cnt, ntiles, tile_off, totals);
    g_launches++;
  } else {
    ck(cudaMemsetAsync(m->tile_mask, 0, sizeof(uint32_t) * ntiles * mw, s));
    ck(cudaMemsetAsync(m->nbr, 0xFF, sizeof(int32_t) * K * n_pad, s));
    ck(cudaMemsetAsync(totals, 0, sizeof(int64_t) * K, s));
  }
  ck(cudaGetLastError());
  int64_t* h_tot = (int64_t*)pinned_stage(sizeof(int64_t) * K);
  if (!h_tot) {
    dev_free(m->alloc, scratch, s);
    return fail(MK_ERR_OUT_OF_MEMORY, "mk_kmap_build: pinned staging failed");
  }
  ck(cudaMemcpyAsync(h_tot, totals, sizeof(int64_t) * K, cudaMemcpyDeviceToHost, s));
  ck(cudaStreamSynchronize(s));
  if (e != cudaSuccess) {
    dev_free(m->alloc, scratch, s);
    return fail(MK_ERR_CUDA, std::string("mk_kmap_build: ") + cudaGetErrorString(e));
  }
  m->h_ptr.assign(K + 1, 0);
  for (int k = 0; k < K; ++k) m->h_ptr[k + 1] = m->h_ptr[k] + h_tot[k];
  m->n_pairs = m->h_ptr[K];
  if (m->n_pairs > INT32_MAX) {
    dev_free(m->alloc, scratch, s);
    return fail(MK_ERR_UNSUPPORTED, "mk_kmap_build: more than 2^31 pairs");
  }
  // +4 entries of padding: the wgrad kernel bulk-copies 16-byte aligned supersets of ranges
  m->in_idx = (int32_t*)alloc(sizeof(int32_t) * (m->n_pairs + 4));
  m->out_idx = (int32_t*)alloc(sizeof(int32_t) * (m->n_pairs + 4));
  if (!m->in_idx || !m->out_idx) {
    dev_free(m->alloc, scratch, s);
    return fail(MK_ERR_OUT_OF_MEMORY, "mk_kmap_build: device allocation failed");
  }
  {  // CSR offsets + weight-gradient split-K plan: one device block, one pinned H2D copy
    std::vector<int4> segs;
    std::vector<int32_t> seg_begin, slot_begin(K + 1, 0);
    const int64_t P = m->n_pairs;
    int64_t L = std::max<int64_t>(64, ceil_div(ceil_div(std::max<int64_t>(P, 1), ctx->num_sms), 64) * 64);
    const int64_t ncta = P > 0 ? ceil_div(P, L) : 0;
    for (int64_t c = 0; c < ncta; ++c) {
      seg_begin.push_back((int32_t)segs.size());
      const int64_t cb = c * L, ce = std::min(P, cb + L);
      for (int k = 0; k < K; ++k) {
        const int64_t b = std::max(cb, m->h_ptr[k]), e2 = std::min(ce, m->h_ptr[k + 1]);
        if (b < e2) segs.push_back(make_int4(k, (int)b, (int)e2, (int)segs.size()));
      }
    }
    seg_begin.push_back((int32_t)segs.size());
    for (int k = 0, i = 0; k <= K; ++k) {
      while (i < (int)segs.size() && segs[i].x < k) ++i;
      slot_begin[k] = i;
    }
    m->n_wcta = (int32_t)ncta;
    m->n_wslots = (int64_t)segs.size();
    const size_t b_ptr = (sizeof(int64_t) * (K + 1) + 15) & ~size_t(15), b_seg = sizeof(int4) * std::max<size_t>(1, segs.size());
    const size_t b_sb = sizeof(int32_t) * seg_begin.size(), b_kb = sizeof(int32_t) * (K + 1);
    const size_t total = b_ptr + b_seg + b_sb + b_kb;
    char* d = (char*)alloc(total);
    char* h = (char*)pinned_stage(total);
    if (!d || !h) {
      dev_free(m->alloc, scratch, s);
      return fail(MK_ERR_OUT_OF_MEMORY, "mk_kmap_build: allocation failed");
    }
    std::memcpy(h, m->h_ptr.data(), sizeof(int64_t) * (K + 1));
    if (!segs.empty()) std::memcpy(h + b_ptr, segs.data(), sizeof(int4) * segs.size());
    std::memcpy(h + b_ptr + b_seg, seg_begin.data(), b_sb);
    std::memcpy(h + b_ptr + b_seg + b_sb, slot_begin.data(), b_kb);
    ck(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s));
    pinned_in_flight(s);
    m->ptr = (int64_t*)d;  // b_ptr is padded to 16 bytes so the int4 plan stays aligned
    m->wseg = (int4*)(d + b_ptr);
    m->wseg_begin = (int32_t*)(d + b_ptr + b_seg);
    m->wslot_begin = (int32_t*)(d + b_ptr + b_seg + b_sb);
  }
  if (n_out > 0) {
    k_emit<<<(unsigned)ntiles, kThreads, sizeof(int32_t) * K * 4, s>>>(m->nbr, n_out, n_pad, K, m->ptr, tile_off,
                                                                        ntiles, m->in_idx, m->out_idx, m->nbrT, nT_pad,
                                                                        m->tile_maskT, mw);
    g_launches++;
  }
  // Order the conv tiles' rows by neighbour bitmask (stable radix sort of the row masks):
  // rows sharing offsets share tiles, so the tensor-core kernels skip empty (tile, k) units.
  // The permutation is internal; the CSR above and all exported row orders are unchanged.
  if (sort_rows && n_out > 0) {
    auto permute = [&](int32_t*& tab, int64_t stride, int64_t n, int64_t nt, uint32_t* tmask, int32_t*& perm_out) {
      int32_t* perm = (int32_t*)alloc(sizeof(int32_t) * stride);
      int32_t* tabP = (int32_t*)alloc(sizeof(int32_t) * (int64_t)K * stride);
      if (!perm || !tabP) return MK_ERR_OUT_OF_MEMORY;
      mk_status st2 = radix_sort_perm(m->alloc, rowmask, n, K, perm, s);
      if (st2 != MK_OK) return st2;
      k_permute<<<(unsigned)nt, kTileRows, 0, s>>>(tab, stride, n, K, perm, tabP, tmask);
      g_launches++;
      tab = tabP;  // the unpermuted table stays owned (freed with the map) but is no longer read
      perm_out = perm;
      return MK_OK;
    };
    mk_status st2 = permute(m->nbr, n_pad, n_out, ntiles, m->tile_mask, m->perm);
    if (st2 == MK_OK && !symmetric && n_in > 0) {
      k_rowmask_T<<<(unsigned)std::min<int64_t>(ceil_div(n_in, 256), 4096), 256, 0, s>>>(m->nbrT, nT_pad, n_in, K, rowmask);
      g_launches++;
      st2 = permute(m->nbrT, nT_pad, n_in, ntilesT, m->tile_maskT, m->permT);
    }
    if (st2 != MK_OK) {
      dev_free(m->alloc, rowmask, s);
      dev_free(m->alloc, scratch, s);
      return fail(st2, "mk_kmap_build: row ordering failed");
    }
  }
  if (rowmask) dev_free(m->alloc, rowmask, s);
  if (symmetric) {
    k_mirror_mask<<<(unsigned)std::min<int64_t>(ceil_div(ntiles, 256), 1024), 256, 0, s>>>(m->tile_mask, ntiles, mw,
                                                                                          m->d_mirror, K, m->tile_maskT);
    g_launches++;
    m->permT = m->perm;  // same row set, mirrored masks: same ordering
  }
  ck(cudaGetLastError());
  dev_free(m->alloc, scratch, s);
  if (e != cudaSuccess) return fail(MK_ERR_CUDA, std::string("mk_kmap_build: ") + cudaGetErrorString(e));
  *out_map = m;
  return MK_OK;
}

mk_status mk_kmap_info(const mk_kmap* m, int32_t* K, int64_t* n_pairs, int64_t* n_in, int64_t* n_out) {
  clear_error();
  if (!m) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_kmap_info: null handle");
  if (K) *K = m->K;
  if (n_pairs) *n_pairs = m->n_pairs;
  if (n_in) *n_in = m->n_in;
  if (n_out) *n_out = m->n_out;
  return MK_OK;
}

mk_status mk_kmap_export(const mk_kmap* m, int64_t* d_ptr, int32_t* d_in, int32_t* d_out, void* stream) {
  clear_error();
  if (!m) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_kmap_export: null handle");
  cudaStream_t s = (cudaStream_t)stream;
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
  delete m;
}

}  // extern "C"
