// conv_umma.cu — bf16 tcgen05 (UMMA) kernels of the generalized sparse convolution.
//
// k_conv_umma<CH>: output-stationary gather-GEMM for forward, dgrad and the transposed conv
//   (Alg. 2 P:189-201 reorganised per output tile).  Persistent, one CTA per SM,
//   warp-specialised:
//     warps 0-3  producers: for every (tile of 128 output rows, non-empty offset k,
//                channel chunk c) gather the 128 neighbour rows x[nb(k,row)][c*CH..] into a
//                swizzled K-major smem stage with 16-byte cp.async (absent neighbours are
//                zero-filled, no global read), and bulk-copy (TMA engine) the pre-swizzled
//                weight chunk W_k[:, c] into the same stage.
//     warp 8     one elected thread issues tcgen05.mma (M=128, N=C_out, K=16) into a TMEM
//                accumulator; tcgen05.commit frees the stage / publishes the tile.
//     warps 4-7  epilogue: tcgen05.ld the 128 x C_out fp32 accumulator (double-buffered in
//                TMEM so it overlaps the next tile's MMAs), convert, store whole rows.
//   Every output row is produced by exactly one CTA from all its offsets: no atomics, fixed
//   summation order, rows without neighbours are written as 0.
// k_wgrad_umma: dW_k = sum_p G[o_p] x X[a_p]^T over the pairs of offset k (split-K).  The
//   concatenated pair list is cut into per-CTA ranges; each (CTA, offset) segment is an
//   accumulation unit: gathered G rows form the MN-major A operand (M = C_out padded to
//   128), gathered X rows the MN-major B operand (N = C_in), K = pairs.  Segment partials
//   go to a workspace and are summed per offset in a fixed order (deterministic).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "conv.cuh"
#include "sm100.cuh"

namespace mk {
namespace {

using namespace sm100;

constexpr int kTileM = 128;
constexpr int kProdWarps = 4;
constexpr int kEpiWarps = 4;
constexpr int kMmaWarp = kProdWarps + kEpiWarps;  // warp 8
constexpr int kThreads = (kProdWarps + kEpiWarps + 1) * 32;
constexpr int kMaxSmem = 227 * 1024;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return (uint8_t*)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

// ------------------------------------------------------------------ weight packing
// Writes W_k chunk images in the exact swizzled K-major smem layout of the B operand:
// image(k, c) = rows n in [0, c_y), channels [c*CH, c*CH+CH) of the reduction dimension.
//   forward: B(n, kx) = W[k][n][kx]   (n = c_out, kx = c_in)
//   dgrad  : B(n, kx) = W[k][kx][n]   (n = c_in,  kx = c_out)  i.e. W_k^T
__global__ void k_pack_w(const __nv_bfloat16* __restrict__ W, int K, int c_out, int c_in, int trans, int CH,
                         uint8_t* __restrict__ out) {
  const int c_y = trans ? c_in : c_out, c_x = trans ? c_out : c_in;
  const int nch = c_x / CH, J = CH / 8, RB = CH * 2;
  const int64_t total = (int64_t)K * nch * c_y * J;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % J);
    const int n = (int)((idx / J) % c_y);
    const int c = (int)((idx / ((int64_t)J * c_y)) % nch);
    const int k = (int)(idx / ((int64_t)J * c_y * nch));
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int kx = c * CH + j * 8 + e;
      v[e] = trans ? W[((int64_t)k * c_out + kx) * c_in + n] : W[((int64_t)k * c_out + n) * c_in + kx];
    }
    uint8_t* dst = out + ((int64_t)k * nch + c) * c_y * RB + swz(n, j, RB);
    *(uint4*)dst = *(const uint4*)v;
  }
}

// ------------------------------------------------------------------ forward / dgrad
struct FwdParams {
  CUtensorMap tmap_x;      // x as a 2-D [n_src][c_x] bf16 tensor, box {CH, 1}, swizzle = CH*2 bytes
  const __nv_bfloat16* x;  // [n_src][c_x]
  const uint8_t* wpack;    // [K][nch] images of c_y * CH bf16
  void* y;                 // [n_rows][c_y]
  NbrView nb;
  int64_t n_rows, ntiles;
  int c_x, c_y, nch, out_f32, stages, lag;
  uint32_t a_bytes, b_bytes, stage_bytes, tmem_cols;
};

__device__ __forceinline__ int tile_active_count(const NbrView& nb, int64_t tile) {
  int n = 0;
  for (int w = 0; w < nb.mw; ++w) n += __popc(__ldg(nb.mask + tile * nb.mw + w));
  return n;
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Enumerates the (tile, mask word) units of a CTA in processing order: tiles blockIdx.x,
// blockIdx.x + gridDim.x, ...; inside a tile the words with at least one active offset.
struct UnitIter {
  const uint32_t* mask;
  int64_t ntiles;
  int mw;
  int64_t tile;
  int w;
  uint32_t bits;
  __device__ UnitIter(const NbrView& nb, int64_t ntiles_) : mask(nb.mask), ntiles(ntiles_), mw(nb.mw) {
    tile = blockIdx.x;
    w = -1;
    bits = 0;
  }
  __device__ __forceinline__ bool next() {
    while (true) {
      if (++w >= mw) {
        w = 0;
        tile += gridDim.x;
      }
      if (tile >= ntiles) return false;
      bits = __ldg(mask + tile * mw + w);
      if (bits) return true;
    }
  }
};

// Per-warp completion signalling for cp.async stages: every stage a warp issues is one
// cp.async group; once `lag` newer groups exist, the oldest is waited for, made visible to
// the async proxy (the tensor cores read it) and announced with ONE arrival per warp on the
// stage's full barrier (instead of one arrival per thread).
struct StageSignal {
  int lag, pending;
  uint32_t s, S;
  __device__ StageSignal(int lag_, uint32_t S_) : lag(lag_), pending(0), s(0), S(S_) {}
  __device__ __forceinline__ void arrive_oldest(uint64_t* full) {
    fence_proxy_async_smem();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(full + s);
    if (++s == S) s = 0;
    --pending;
  }
  __device__ __forceinline__ void issued(uint64_t* full) {
    cp_async_commit();
    if (++pending > lag) {
      cp_async_wait_n(lag);
      arrive_oldest(full);
    }
  }
  __device__ __forceinline__ void drain(uint64_t* full) {
    cp_async_wait_n(0);
    while (pending > 0) arrive_oldest(full);
  }
};

#ifdef MK_TRACE
__device__ unsigned long long g_trace[4][4096];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(role, i, v) \
  do {                    \
    if (blockIdx.x == 0 && (i) < 4096) g_trace[role][i] = (v); \
  } while (0)
#else
#define TRACE(role, i, v) \
  do {                    \
  } while (0)
#endif

constexpr int kNbrBuf = 32 * kTileM;  // int32 entries per staging buffer (32 offsets x 128 rows)

// Bulk-copies (TMA engine) the neighbour indices of unit `u` — 128 rows per active offset,
// one 512-byte row segment each — into a staging buffer; completion on `bar`.
__device__ __forceinline__ void stage_nbr(const NbrView& nb, const UnitIter& u, int32_t* buf, uint64_t* bar) {
  mbar_arrive_expect_tx(bar, (uint32_t)__popc(u.bits) * kTileM * 4);
  uint32_t bits = u.bits;
  for (int j = 0; bits; ++j) {
    const int k = u.w * 32 + __ffs(bits) - 1;
    bits &= bits - 1;
    bulk_g2s(buf + j * kTileM, nb.tab + (int64_t)nb.kk(k) * nb.n + u.tile * kTileM, kTileM * 4, bar);
  }
}

template <int CH>
__global__ void __launch_bounds__(kThreads, 1) k_conv_umma(const __grid_constant__ FwdParams p) {
  constexpr int J = CH / 8;    // 16-byte chunks per gathered row
  constexpr int RB = CH * 2;   // bytes per gathered row (= swizzle span)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = p.stages;
  int32_t* nbr_s = (int32_t*)(smem + (size_t)S * p.stage_bytes);  // [2][32][128]
  uint64_t* full = (uint64_t*)(nbr_s + 2 * kNbrBuf);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* nfull = tempty + 2;
  uint32_t* tmem_slot = (uint32_t*)(nfull + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, kProdWarps + 1);  // one per producer warp + the weight bulk copy
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, kEpiWarps * 32);
      mbar_init(nfull + b, 1);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc_dyn(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp < kProdWarps) {
    // ---------------------------------------------------------------- producers
    // 128 threads gather the 128 rows x CH channels of a stage with 16-byte cp.async (8
    // threads per 128-byte row => coalesced), absent neighbours zero-filled; thread 0
    // bulk-copies the weight chunk.  One barrier arrival per warp (StageSignal).
    const int t = threadIdx.x;
    UnitIter cur(p.nb, p.ntiles), st(p.nb, p.ntiles);
    if (t == 0)
      for (int b = 0; b < 2; ++b)
        if (st.next()) stage_nbr(p.nb, st, nbr_s + b * kNbrBuf, nfull + b);
    StageSignal sig(p.lag, (uint32_t)S);
    uint32_t s = 0, ph = 0, ub = 0, nph = 0;
#ifdef MK_TRACE
    int tr_g = 0, tr_u = 0;
#endif
    while (cur.next()) {
#ifdef MK_TRACE
      if (t == 0) TRACE(3, 2 * tr_u, gtime());
#endif
      mbar_wait(nfull + ub, (nph >> ub) & 1u);
#ifdef MK_TRACE
      if (t == 0) TRACE(3, 2 * tr_u + 1, gtime());
      ++tr_u;
#endif
      nph ^= 1u << ub;
      const int32_t* nb_u = nbr_s + ub * kNbrBuf;
      uint32_t bits = cur.bits;
      for (int j = 0; bits; ++j) {
        const int k = cur.w * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
        int32_t src[J];
#pragma unroll
        for (int i = 0; i < J; ++i) src[i] = nb_u[j * kTileM + (i * 128 + t) / J];
        for (int c = 0; c < p.nch; ++c) {
#ifdef MK_TRACE
          if (t == 0) TRACE(0, 2 * tr_g, gtime());
#endif
          mbar_wait(empty + s, ph ^ 1);
#ifdef MK_TRACE
          if (t == 0) TRACE(0, 2 * tr_g + 1, gtime());
          ++tr_g;
#endif
          uint8_t* stage = smem + (size_t)s * p.stage_bytes;
          const uint32_t a_s = smem_u32(stage);
#pragma unroll
          for (int i = 0; i < J; ++i) {
            const int idx = i * 128 + t;
            const int r = idx / J, jj = idx % J;
            // absent neighbour: zero the row in smem (no global request at all)
            if (src[i] >= 0) cp_async16(a_s + swz(r, jj, RB), p.x + (int64_t)src[i] * p.c_x + c * CH + jj * 8, 16u);
            else st_shared_zero16(a_s + swz(r, jj, RB));
          }
          if (t == 0) {
            mbar_arrive_expect_tx(full + s, p.b_bytes);
            bulk_g2s(stage + p.a_bytes, p.wpack + ((int64_t)k * p.nch + c) * p.b_bytes, p.b_bytes, full + s);
          }
          sig.issued(full);
          if (++s == (uint32_t)S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      named_bar_sync(1, kProdWarps * 32);  // every producer is done reading buffer ub
      if (t == 0 && st.next()) {
        fence_proxy_async_smem();
        stage_nbr(p.nb, st, nbr_s + ub * kNbrBuf, nfull + ub);
      }
      ub ^= 1;
    }
    sig.drain(full);
  } else if (warp == kMmaWarp) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(kTileM, p.c_y, 0, 0);
      const uint32_t lay = layout_code(RB);
      uint32_t s = 0, ph = 0, tl = 0;
#ifdef MK_TRACE
      int tr_m = 0;
#endif
      for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        if (tile_active_count(p.nb, tile) == 0) continue;
        const uint32_t b = tl & 1, tph = (tl >> 1) & 1;
        mbar_wait(tempty + b, tph ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + b * (uint32_t)p.c_y;
        uint32_t acc = 0;
        for (int w = 0; w < p.nb.mw; ++w) {
          const int nk = __popc(__ldg(p.nb.mask + tile * p.nb.mw + w));
          for (int q = 0; q < nk * p.nch; ++q) {
            mbar_wait(full + s, ph);
#ifdef MK_TRACE
            TRACE(1, tr_m, gtime());
            ++tr_m;
#endif
            tc_fence_after();
            const uint32_t a_s = smem_u32(smem + (size_t)s * p.stage_bytes);
            const uint32_t b_s = a_s + p.a_bytes;
#pragma unroll
            for (int kk = 0; kk < CH / 16; ++kk) {
              const uint64_t ad = smem_desc(a_s + kk * 32, 16, 8 * RB, lay);
              const uint64_t bd = smem_desc(b_s + kk * 32, 16, 8 * RB, lay);
              umma_f16(d, ad, bd, idesc, acc);
              acc = 1;
            }
            umma_commit(empty + s);
            if (++s == (uint32_t)S) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        umma_commit(tfull + b);
        ++tl;
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter owned by this warp
    uint32_t tl = 0;
    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
      const int64_t row = tile * kTileM + q * 32 + lane;
      const bool valid = row < p.n_rows;
      if (tile_active_count(p.nb, tile) == 0) {
        if (valid) {
          if (p.out_f32) {
            float4* yr = (float4*)((float*)p.y + row * p.c_y);
            for (int c = 0; c < p.c_y / 4; ++c) yr[c] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            uint4* yr = (uint4*)((__nv_bfloat16*)p.y + row * p.c_y);
            for (int c = 0; c < p.c_y / 8; ++c) yr[c] = make_uint4(0, 0, 0, 0);
          }
        }
        continue;
      }
      const uint32_t b = tl & 1, tph = (tl >> 1) & 1;
      mbar_wait(tfull + b, tph);
#ifdef MK_TRACE
      if (q == 0 && lane == 0) TRACE(2, 2 * tl, gtime());
#endif
      tc_fence_after();
      const uint32_t tl_addr = tbase + ((uint32_t)(q * 32) << 16) + b * (uint32_t)p.c_y;
      for (int col0 = 0; col0 < p.c_y; col0 += 16) {
        uint32_t v[16];
        tmem_ld16(tl_addr + col0, v);
        tmem_ld_wait();
        if (valid) {
          if (p.out_f32) {
            float4* yr = (float4*)((float*)p.y + row * p.c_y + col0);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              yr[e] = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]),
                                  __uint_as_float(v[4 * e + 2]), __uint_as_float(v[4 * e + 3]));
          } else {
            uint32_t h[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              __nv_bfloat162 t2 = __floats2bfloat162_rn(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
              h[e] = *(uint32_t*)&t2;
            }
            uint4* yr = (uint4*)((__nv_bfloat16*)p.y + row * p.c_y + col0);
            yr[0] = make_uint4(h[0], h[1], h[2], h[3]);
            yr[1] = make_uint4(h[4], h[5], h[6], h[7]);
          }
        }
      }
      tc_fence_before();
#ifdef MK_TRACE
      if (q == 0 && lane == 0) TRACE(2, 2 * tl + 1, gtime());
#endif
      mbar_arrive(tempty + b);
      ++tl;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tbase, p.tmem_cols);
}

// ------------------------------------------------------------------ weight gradient
struct WgradParams {
  CUtensorMap tmap_g;      // g as [n_out][c_out], box {pwa, 1}
  CUtensorMap tmap_x;      // x as [n_in][c_in],  box {pwb, 1}
  const __nv_bfloat16* g;  // [n_out][c_out]
  const __nv_bfloat16* x;  // [n_in][c_in]
  const int32_t* in_idx;
  const int32_t* out_idx;
  const int4* segs;          // (k, begin, end, slot), grouped by CTA
  const int32_t* seg_begin;  // [n_cta + 1]
  float* part;               // [n_slots][c_out][c_in]
  int c_out, c_in, stages, halves, lag;
  int pwa, pwb;              // panel widths (channels) of A (G) and B (X)
  uint32_t a_bytes, b_bytes, stage_bytes, tmem_cols;
};

constexpr int kPairsPerStage = 64;
constexpr int kUnitPairs = 1024;            // pairs per index-staging unit (16 stages)
constexpr int kIdxBuf = kUnitPairs + 8;     // int32 entries per staged index array

// Enumerates the index-staging units of a CTA: every segment (k, begin, end, slot) of the
// CTA cut into runs of at most kUnitPairs pairs (multiples of the 64-pair stage).
struct WUnitIter {
  const int4* segs;
  int si, se;
  int4 sg;
  int b, e;
  __device__ WUnitIter(const int4* s, int sb, int se_) : segs(s), si(sb - 1), se(se_), b(0), e(0) { sg = make_int4(0, 0, 0, 0); }
  __device__ __forceinline__ bool next() {
    if (e < sg.z) {  // more of the current segment
      b = e;
      e = min(b + kUnitPairs, sg.z);
      return true;
    }
    while (++si < se) {
      sg = __ldg(segs + si);
      if (sg.y < sg.z) {
        b = sg.y;
        e = min(b + kUnitPairs, sg.z);
        return true;
      }
    }
    return false;
  }
};

// Bulk-copies out_idx / in_idx of the unit's pairs (16-byte aligned superset) into `buf`.
__device__ __forceinline__ void stage_idx(const int32_t* out_idx, const int32_t* in_idx, const WUnitIter& u,
                                          int32_t* buf, uint64_t* bar) {
  const int b4 = u.b & ~3, e4 = (u.e + 3) & ~3;
  const uint32_t bytes = (uint32_t)(e4 - b4) * 4;
  mbar_arrive_expect_tx(bar, 2 * bytes);
  bulk_g2s(buf, out_idx + b4, bytes, bar);
  bulk_g2s(buf + kIdxBuf, in_idx + b4, bytes, bar);
}

__global__ void __launch_bounds__(kThreads, 1) k_wgrad_umma(const __grid_constant__ WgradParams p) {
  constexpr int PS = kPairsPerStage;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = p.stages;
  int32_t* idx_s = (int32_t*)(smem + (size_t)S * p.stage_bytes);  // [2][out, in][kIdxBuf]
  uint64_t* full = (uint64_t*)(idx_s + 4 * kIdxBuf);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 1;
  uint64_t* nfull = tempty + 1;
  uint32_t* tmem_slot = (uint32_t*)(nfull + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rba = p.pwa * 2, rbb = p.pwb * 2;              // panel row bytes
  const int npa = p.c_out / p.pwa, npb = p.c_in / p.pwb;   // real panels
  const uint32_t panel_a = PS * rba, panel_b = PS * rbb;   // panel strides (LBO)

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, kProdWarps);
      mbar_init(empty + s, 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kEpiWarps * 32);
    mbar_init(nfull, 1);
    mbar_init(nfull + 1, 1);
    fence_mbar_init();
  }
  // zero the padding panels of A (M padded to 128 per half) once; never overwritten
  {
    const int tot_pa = (int)(p.a_bytes / panel_a);
    for (int s = 0; s < S; ++s)
      for (int pa = npa; pa < tot_pa; ++pa) {
        uint4* z = (uint4*)(smem + (size_t)s * p.stage_bytes + (size_t)pa * panel_a);
        for (int i = threadIdx.x; i < (int)(panel_a / 16); i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
      }
  }
  if (warp == kMmaWarp) tmem_alloc_dyn(tmem_slot, p.tmem_cols);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int sb = p.seg_begin[blockIdx.x], se = p.seg_begin[blockIdx.x + 1];

  if (warp < kProdWarps) {
    // 128 threads gather, per 64-pair stage, the G rows (A panels) and X rows (B panels) of
    // the pairs with 16-byte cp.async; pairs past the segment end are zero-filled.  One
    // barrier arrival per warp (StageSignal).
    const int t = threadIdx.x;
    const int ca = p.c_out / 8, cb = p.c_in / 8;  // 16-byte chunks per G row / X row
    const int ja = rba / 16, jb = rbb / 16;       // chunks per panel row
    WUnitIter cur(p.segs, sb, se), st(p.segs, sb, se);
    if (t == 0)
      for (int b = 0; b < 2; ++b)
        if (st.next()) stage_idx(p.out_idx, p.in_idx, st, idx_s + b * 2 * kIdxBuf, nfull + b);
    StageSignal sig(p.lag, (uint32_t)S);
    uint32_t s = 0, ph = 0, ub = 0, nph = 0;
    while (cur.next()) {
      mbar_wait(nfull + ub, (nph >> ub) & 1u);
      nph ^= 1u << ub;
      const int32_t* oi = idx_s + ub * 2 * kIdxBuf;
      const int32_t* ii = oi + kIdxBuf;
      const int b4 = cur.b & ~3;
      for (int b0 = cur.b; b0 < cur.e; b0 += PS) {
        mbar_wait(empty + s, ph ^ 1);
        const uint32_t a_s = smem_u32(smem + (size_t)s * p.stage_bytes), b_s = a_s + p.a_bytes;
        for (int idx = t; idx < PS * ca; idx += kProdWarps * 32) {  // G rows -> A panels
          const int pr = idx / ca, ch = idx - pr * ca;
          const int pi = b0 + pr;
          const bool ok = pi < cur.e;
          const int pa = ch / ja, j = ch - pa * ja;
          if (ok) cp_async16(a_s + pa * panel_a + swz(pr, j, rba), p.g + (int64_t)oi[pi - b4] * p.c_out + ch * 8, 16u);
          else st_shared_zero16(a_s + pa * panel_a + swz(pr, j, rba));
        }
        for (int idx = t; idx < PS * cb; idx += kProdWarps * 32) {  // X rows -> B panels
          const int pr = idx / cb, ch = idx - pr * cb;
          const int pi = b0 + pr;
          const bool ok = pi < cur.e;
          const int pb = ch / jb, j = ch - pb * jb;
          if (ok) cp_async16(b_s + pb * panel_b + swz(pr, j, rbb), p.x + (int64_t)ii[pi - b4] * p.c_in + ch * 8, 16u);
          else st_shared_zero16(b_s + pb * panel_b + swz(pr, j, rbb));
        }
        sig.issued(full);
        if (++s == (uint32_t)S) {
          s = 0;
          ph ^= 1;
        }
      }
      named_bar_sync(1, kProdWarps * 32);
      if (t == 0 && st.next()) {
        fence_proxy_async_smem();
        stage_idx(p.out_idx, p.in_idx, st, idx_s + ub * 2 * kIdxBuf, nfull + ub);
      }
      ub ^= 1;
    }
    sig.drain(full);
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(kTileM, p.c_in, 1, 1);
      const uint32_t la = layout_code(rba), lb = layout_code(rbb);
      uint32_t s = 0, ph = 0, n_seg = 0;
      for (int si = sb; si < se; ++si) {
        const int4 sg = p.segs[si];
        if (sg.y >= sg.z) continue;
        mbar_wait(tempty, (n_seg & 1) ^ 1);
        tc_fence_after();
        uint32_t acc = 0;
        for (int b0 = sg.y; b0 < sg.z; b0 += PS) {
          mbar_wait(full + s, ph);
          tc_fence_after();
          const uint32_t a_s = smem_u32(smem + (size_t)s * p.stage_bytes), b_s = a_s + p.a_bytes;
#pragma unroll
          for (int kk = 0; kk < PS / 16; ++kk) {
            const uint64_t bd = smem_desc(b_s + kk * 16 * rbb, panel_b, 8 * rbb, lb);
            for (int h = 0; h < p.halves; ++h) {
              const uint32_t a_half = a_s + h * (128 / p.pwa) * panel_a;
              const uint64_t ad = smem_desc(a_half + kk * 16 * rba, panel_a, 8 * rba, la);
              umma_f16(tbase + h * (uint32_t)p.c_in, ad, bd, idesc, acc);
            }
            acc = 1;
          }
          umma_commit(empty + s);
          if (++s == (uint32_t)S) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(tfull);
        ++n_seg;
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    uint32_t n_seg = 0;
    for (int si = sb; si < se; ++si) {
      const int4 sg = p.segs[si];
      if (sg.y >= sg.z) continue;
      mbar_wait(tfull, n_seg & 1);
      tc_fence_after();
      for (int h = 0; h < p.halves; ++h) {
        const int co = h * 128 + q * 32 + lane;
        float* dst = p.part + ((int64_t)sg.w * p.c_out + co) * p.c_in;
        const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + h * (uint32_t)p.c_in;
        for (int col0 = 0; col0 < p.c_in; col0 += 16) {
          uint32_t v[16];
          tmem_ld16(ta + col0, v);
          tmem_ld_wait();
          if (co < p.c_out) {
            float4* d4 = (float4*)(dst + col0);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              d4[e] = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]),
                                  __uint_as_float(v[4 * e + 2]), __uint_as_float(v[4 * e + 3]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
      ++n_seg;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tbase, p.tmem_cols);
}


// ------------------------------------------------------------------ host: tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (EncodeTiledFn)f;
  }();
  return fn;
}

// A [rows][cols] bf16 row-major tensor viewed for row gathers: box {box_cols, 1}, swizzle
// matching a K-major / MN-major UMMA panel of box_cols * 2 bytes; out-of-range rows
// (index -1) are zero-filled by the TMA unit.
bool make_row_map(CUtensorMap* m, const void* base, int64_t rows, int cols, int box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || ((uintptr_t)base & 15) || rows < 1) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, 1};
  const cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle sw = box_cols * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : box_cols * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                     : CU_TENSOR_MAP_SWIZZLE_32B;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

uint32_t pow2_cols(uint32_t c) {
  uint32_t r = 32;
  while (r < c) r <<= 1;
  return r;
}

template <class F>
void set_smem_once(F* f, int bytes) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

#ifdef MK_TRACE
extern "C" int mk_debug_trace(unsigned long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_trace, sizeof(g_trace));
}
#endif

mk_status launch_conv_bf16(mk_context* ctx, const NbrView& nb, const void* x, int64_t n_src, int c_x, const void* W,
                            int c_in_w, int c_out_w, void* y, int c_y, mk_dtype out_dt, int64_t n_rows, bool trans,
                            cudaStream_t s) {
  if (n_rows == 0) return MK_OK;
  const int CH = c_x % 64 == 0 ? 64 : c_x % 32 == 0 ? 32 : 16;
  const int nch = c_x / CH;
  FwdParams p;
  p.x = (const __nv_bfloat16*)x;
  p.y = y;
  p.nb = nb;
  p.n_rows = n_rows;
  p.ntiles = ceil_div(n_rows, kTileM);
  p.c_x = c_x;
  p.c_y = c_y;
  p.nch = nch;
  p.out_f32 = out_dt == MK_F32;
  p.a_bytes = kTileM * CH * 2;
  p.b_bytes = (uint32_t)c_y * CH * 2;
  p.stage_bytes = (p.a_bytes + p.b_bytes + 1023) & ~1023u;
  const int reserve = 1024 + 256 + 2 * kNbrBuf * 4;
  p.stages = std::min<int>(8, (kMaxSmem - reserve) / (int)p.stage_bytes);
  if (p.stages < 2) MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 conv: channel counts too large for the smem pipeline");

  p.tmem_cols = pow2_cols(2 * c_y);
  if (p.tmem_cols > 512) MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 conv: C_out above 256");
  p.lag = std::min(4, p.stages - 1);
  const size_t wbytes = (size_t)nb.K * nch * p.b_bytes;
  uint8_t* wpack = (uint8_t*)dev_alloc(ctx->alloc, wbytes, s);
  if (!wpack) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "bf16 conv: weight pack allocation failed");
  {
    const int64_t chunks = (int64_t)nb.K * nch * c_y * (CH / 8);
    const int grid = (int)std::min<int64_t>(ceil_div(chunks, 256), 4 * ctx->num_sms);
    k_pack_w<<<grid, 256, 0, s>>>((const __nv_bfloat16*)W, nb.K, c_out_w, c_in_w, trans ? 1 : 0, CH, wpack);
    g_launches++;
  }
  p.wpack = wpack;
  if (!make_row_map(&p.tmap_x, n_src > 0 ? x : (const void*)wpack, std::max<int64_t>(n_src, 1), c_x, CH)) {
    dev_free(ctx->alloc, wpack, s);
    MK_FAIL(MK_ERR_CUDA, "bf16 conv: cuTensorMapEncodeTiled failed (features must be 16-byte aligned)");
  }
  const int smem = p.stages * (int)p.stage_bytes + reserve;
  const int grid = (int)std::min<int64_t>(p.ntiles, ctx->num_sms);
  if (CH == 64) {
    set_smem_once(k_conv_umma<64>, smem);
    k_conv_umma<64><<<grid, kThreads, smem, s>>>(p);
  } else if (CH == 32) {
    set_smem_once(k_conv_umma<32>, smem);
    k_conv_umma<32><<<grid, kThreads, smem, s>>>(p);
  } else {
    set_smem_once(k_conv_umma<16>, smem);
    k_conv_umma<16><<<grid, kThreads, smem, s>>>(p);
  }
  g_launches++;
  cudaError_t e = cudaGetLastError();
  dev_free(ctx->alloc, wpack, s);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("bf16 conv launch: ") + cudaGetErrorString(e));
  return MK_OK;
}

mk_status launch_wgrad_bf16(mk_context* ctx, const mk_kmap* m, const void* g, int c_out, const void* x, int c_in,
                            float* dW, cudaStream_t s) {
  const int64_t te = (int64_t)c_out * c_in;
  WgradParams p;
  p.g = (const __nv_bfloat16*)g;
  p.x = (const __nv_bfloat16*)x;
  p.in_idx = m->in_idx;
  p.out_idx = m->out_idx;
  p.segs = m->wseg;
  p.seg_begin = m->wseg_begin;
  p.c_out = c_out;
  p.c_in = c_in;
  p.pwa = c_out % 64 == 0 ? 64 : c_out % 32 == 0 ? 32 : 16;
  p.pwb = c_in % 64 == 0 ? 64 : c_in % 32 == 0 ? 32 : 16;
  p.halves = c_out > 128 ? 2 : 1;
  if (c_out > 256) MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 wgrad: C_out above 256");
  p.a_bytes = (uint32_t)(p.halves * 128) * kPairsPerStage * 2;  // M padded to 128 per half
  p.b_bytes = (uint32_t)c_in * kPairsPerStage * 2;
  p.stage_bytes = (p.a_bytes + p.b_bytes + 1023) & ~1023u;
  const int reserve = 1024 + 256 + 4 * kIdxBuf * 4;
  p.stages = std::min<int>(6, (kMaxSmem - reserve) / (int)p.stage_bytes);
  p.tmem_cols = pow2_cols((uint32_t)(p.halves * c_in));
  p.lag = std::min(4, p.stages - 1);
  if (p.stages < 2 || p.tmem_cols > 512) MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 wgrad: channel counts too large");
  if (m->n_wslots > 0 &&
      (!make_row_map(&p.tmap_g, g, std::max<int64_t>(m->n_out, 1), c_out, p.pwa) ||
       !make_row_map(&p.tmap_x, x, std::max<int64_t>(m->n_in, 1), c_in, p.pwb)))
    MK_FAIL(MK_ERR_CUDA, "bf16 wgrad: cuTensorMapEncodeTiled failed (features must be 16-byte aligned)");
  float* part = nullptr;
  if (m->n_wslots > 0) {
    part = (float*)dev_alloc(ctx->alloc, sizeof(float) * m->n_wslots * te, s);
    if (!part) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "bf16 wgrad: workspace allocation failed");
    p.part = part;
    const int smem = p.stages * (int)p.stage_bytes + reserve;
    set_smem_once(k_wgrad_umma, smem);
    k_wgrad_umma<<<m->n_wcta, kThreads, smem, s>>>(p);
    g_launches++;
  }
  dim3 rg((unsigned)ceil_div(te, 256), (unsigned)m->K);
  k_reduce_partials<<<rg, 256, 0, s>>>(m->wslot_begin, part, te, dW);
  g_launches++;
  cudaError_t e = cudaGetLastError();
  if (part) dev_free(ctx->alloc, part, s);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("bf16 wgrad launch: ") + cudaGetErrorString(e));
  return MK_OK;
}

}  // namespace mk
