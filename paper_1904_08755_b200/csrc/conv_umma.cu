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
constexpr int kEpiWarps = 4;  // epilogue warps (TMEM lane quarters 0-3) of both kernels
// Forward / dgrad kernel: small CTAs (2 per SM co-reside, the hardware scheduler balances
// the bitmask-sorted tiles, whose work varies ~4x): 4 gather warps, 4 epilogue warps, the
// MMA warp and the W stager.
constexpr int kFwdProd = 4;
// (epilogue warps 4-7 on the TMEM lane quarters, then the MMA warp and the W stager; the
// two-CTA instance has 8 producer warps, see k_conv_umma)
constexpr int kMaxSmem = 227 * 1024;

// Rounds a dynamic shared-memory pointer up to 1024 bytes.  The offset is added to the
// pointer itself (no integer round trip), so the compiler keeps the shared state space
// and every access derived from it is an LDS/STS, not a generic load.
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}
template <class T>
__device__ __forceinline__ T* align16(void* p) {
  return (T*)((uint8_t*)p + ((16u - (smem_u32(p) & 15u)) & 15u));
}

// ------------------------------------------------------------------ weight packing
// Writes W_k chunk images in the exact swizzled K-major smem layout of the B operand:
// image(k, c) = rows n in [0, c_y), channels [c*CH, c*CH+CH) of the reduction dimension.
//   forward: B(n, kx) = W[k][n][kx]   (n = c_out, kx = c_in)
//   dgrad  : B(n, kx) = W[k][kx][n]   (n = c_in,  kx = c_out)  i.e. W_k^T
__global__ void k_pack_w(const __nv_bfloat16* __restrict__ W, int K, int c_out, int c_in, int trans, int CH,
                         uint8_t* __restrict__ out) {
  pdl_enter();
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
#ifdef MK_TRACE
__device__ unsigned long long g_trace[4][8192];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(role, i, v) \
  do {                    \
    if (blockIdx.x == 0 && (i) < 8192) g_trace[role][i] = (v); \
  } while (0)
__device__ unsigned long long g_acct[32][8];
__device__ unsigned long long g_cta[4096][4];  // per-CTA [start ns, end ns, smid, steps]
#define ACCT_WAIT(slot, bar, par)                              \
  do {                                                         \
    const long long _t0 = clock64();                           \
    mbar_wait(bar, par);                                       \
    acct[slot] += clock64() - _t0;                             \
  } while (0)
#define ACCT_WAIT_SLEEP(slot, bar, par)                        \
  do {                                                         \
    const long long _t0 = clock64();                           \
    mbar_wait_sleep(bar, par);                                 \
    acct[slot] += clock64() - _t0;                             \
  } while (0)
#define ACCT_DECL long long acct[8] = {0, 0, 0, 0, 0, 0, 0, 0}; const long long acct_t0 = clock64();
#define ACCT_NOW(v) const long long v = clock64()
#define ACCT_ADD(slot, t0) (acct[slot] += clock64() - (t0))
#define ACCT_DUMP                                                                             \
  do {                                                                                        \
    if (blockIdx.x == 100 && lane == 0) {                                                     \
      for (int _i = 0; _i < 7; ++_i) g_acct[warp][_i] = acct[_i];                             \
      g_acct[warp][7] = clock64() - acct_t0;                                                  \
    }                                                                                         \
  } while (0)
#else
#define ACCT_WAIT(slot, bar, par) mbar_wait(bar, par)
#define ACCT_WAIT_SLEEP(slot, bar, par) mbar_wait_sleep(bar, par)
#define ACCT_NOW(v)
#define ACCT_ADD(slot, t0)
#define ACCT_DECL
#define ACCT_DUMP \
  do {            \
  } while (0)
#define TRACE(role, i, v) \
  do {                    \
  } while (0)
#endif

struct FwdParams {
  const __nv_bfloat16* x;  // [n_src][c_x]
  const uint8_t* wpack;    // [K][nch] images of c_y * CH bf16 (swizzled K-major B operand)
  void* y;                 // [n_rows][c_y]
  NbrView nb;
  int64_t n_rows, ntiles;
  int c_x, c_y, nch, out_f32;
  int cw;  // output columns per CTA (the MMA's N): blockIdx.y takes columns [cw*blockIdx.y, +cw) of c_y
  uint32_t b_img;  // bytes of one full W chunk image (c_y rows); a CTA copies its cw-row slice
  int dbg;  // development switch (env MK_DEBUG_CONV): bit 0 = no MMAs, bit 1 = no gathers; 0 in production
  int sa;  // A stage slots
  int np;  // producer warps (np divides sa)
  int ga;  // stage slots released together by one tcgen05.commit (sa % ga == 0)
  int sw;  // W chunk slots (a ring: W_k chunks are prefetched several offsets ahead)
  int tb;  // tiles per CTA (one TMEM accumulator each: tb * cw <= 512 columns)
  int grp;  // MMA steps cover all nch chunks of a (unit, tile)
  int off32;  // n_src * c_x < 2^31: 32-bit element offsets in the gathers
  int accum;  // fp32 output accumulated in place (y += conv) instead of overwritten
  int fold;  // tile order (see cta_tile)
  int ncb;   // commit barriers in the ring (power of two)
  uint32_t a_bytes, b_bytes, tmem_cols;
  Epilogue ep;  // fused scale / shift / residual / ReLU (forward only; identity otherwise)
};

// 16 consecutive outputs of one row through the fused epilogue (v: fp32 bit patterns).
__device__ __forceinline__ void epi16(const FwdParams& p, int64_t row, int col0, uint32_t (&v)[16]) {
  float res[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) res[e] = 0.f;
  if (p.ep.residual) {
    if (p.out_f32) {
      const float4* rr = (const float4*)((const float*)p.ep.residual + row * p.c_y + col0);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 f = __ldg(rr + e);
        res[4 * e] = f.x, res[4 * e + 1] = f.y, res[4 * e + 2] = f.z, res[4 * e + 3] = f.w;
      }
    } else {
      const uint4* rr = (const uint4*)((const __nv_bfloat16*)p.ep.residual + row * p.c_y + col0);
      auto lo = [](uint32_t u) { return __uint_as_float(u << 16); };           // bf16 -> fp32 is exact:
      auto hi = [](uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); };  // the top 16 bits
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 u = __ldg(rr + h);
        res[8 * h + 0] = lo(u.x), res[8 * h + 1] = hi(u.x), res[8 * h + 2] = lo(u.y), res[8 * h + 3] = hi(u.y);
        res[8 * h + 4] = lo(u.z), res[8 * h + 5] = hi(u.z), res[8 * h + 6] = lo(u.w), res[8 * h + 7] = hi(u.w);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(epi_apply(p.ep, __uint_as_float(v[e]), col0 + e, res[e]));
}

__device__ __forceinline__ void store16(const FwdParams& p, int64_t row, int col0, const uint32_t (&v)[16]) {
  if (p.out_f32) {
    float4* yr = (float4*)((float*)p.y + row * p.c_y + col0);
    if (p.accum) {  // y += conv (fp32 running sum: the bf16x3 split terms, conv_split.cu)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 o = yr[e];
        yr[e] = make_float4(o.x + __uint_as_float(v[4 * e]), o.y + __uint_as_float(v[4 * e + 1]),
                            o.z + __uint_as_float(v[4 * e + 2]), o.w + __uint_as_float(v[4 * e + 3]));
      }
      return;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      yr[e] = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]), __uint_as_float(v[4 * e + 2]),
                          __uint_as_float(v[4 * e + 3]));
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

constexpr int kMaxK = 128;  // offsets supported by the tensor-core conv (4 mask words)
// Ring of commit barriers: the MMA thread's j-th group commit (covering steps up to
// (j+1)*ga - 1) arrives on cb[j % ncb]; anyone needing "all MMAs of step <= x done" waits
// for commit x / ga at parity (j / ncb) & 1.  ncb (a power of two, sized by the host) exceeds
// the number of commits the MMA can issue past any awaited one — the W stager waits for the
// commit of the unit upr units back, so ncb > upr * tb * nch / ga + sa — so a
// waiter can never confuse phases.
constexpr int kNCB = 16;  // minimum commit-ring size

// Per-CTA plan, built once in shared memory by warp 0: the CTA's tiles are
// blockIdx.x * tb + i (adjacent in the map's bitmask-sorted row order, so they share most
// offsets).  A unit is an offset k active in at least one of them: tw = bitmask of those
// tiles.  Units are visited starting at offset blockIdx.x % K (concurrent CTAs then fetch
// different W_k).  g0[u] = first global step of unit u, a step = (unit, tile, chunk).
struct Plan {
  int n_units;
  int n_steps;
  uint32_t active_tiles;  // tiles with at least one offset
  uint8_t k[kMaxK];       // offset of unit u  (K <= 128 < 256)
  uint8_t tw[kMaxK];      // tiles of unit u
  int32_t g0[kMaxK + 1];
};

// First tile of this CTA.  Rows are bitmask-sorted ascending, which puts the densest
// masks (most offsets per tile, up to ~4x the work) at the end; CTAs take batches from the
// end first so the heaviest work is scheduled in the first wave (longest-first).
__device__ __forceinline__ int64_t cta_tile0(const FwdParams& p) {
  const int64_t nb = (p.ntiles + p.tb - 1) / p.tb;
  return (nb - 1 - (int64_t)blockIdx.x) * p.tb;
}
// i-th tile of this CTA, or -1.  fold = 0: tb adjacent tiles, heaviest batches first.
// fold = 1: positions j = tb*blockIdx + i of the order 0, N-1, 1, N-2, ... (tiles taken from
// both ends of the bitmask-sorted order, so every CTA gets a similar amount of work and the
// grid is a single wave).
__device__ __forceinline__ int64_t cta_tile(const FwdParams& p, int i) {
  if (!p.fold) {
    const int64_t t = cta_tile0(p) + i;
    return t < p.ntiles ? t : -1;
  }
  const int64_t j = (int64_t)blockIdx.x * p.tb + i;
  if (j >= p.ntiles) return -1;
  return (j & 1) ? p.ntiles - 1 - (j >> 1) : (j >> 1);
}

__device__ void build_plan(const FwdParams& p, Plan* pl) {
  const int lane = threadIdx.x & 31;
  int nt = 0;
  while (nt < p.tb && cta_tile(p, nt) >= 0) ++nt;
  const int K = p.nb.K;
  const int rot = (int)(blockIdx.x % (unsigned)K);
  uint32_t act = 0;
  int base_units = 0, base_steps = 0;
  for (int kb = 0; kb < K; kb += 32) {
    // lane handles offset k = (rot + kb + lane) % K in visiting order
    const int v = kb + lane;
    const int k = v < K ? (rot + v) % K : 0;
    uint32_t tw = 0;
    if (v < K)
      for (int i = 0; i < nt; ++i) tw |= ((__ldg(p.nb.mask + cta_tile(p, i) * p.nb.mw + (k >> 5)) >> (k & 31)) & 1u) << i;
    act |= __reduce_or_sync(0xffffffffu, tw);
    const bool has = tw != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, has);
    const int pos = base_units + __popc(bal & ((1u << lane) - 1u));
    int steps = has ? __popc(tw) * p.nch : 0;
    int incl = steps;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (has) {
      pl->k[pos] = (uint8_t)k;
      pl->tw[pos] = (uint8_t)tw;
      pl->g0[pos] = base_steps + incl - steps;
    }
    base_units += __popc(bal);
    base_steps += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) {
    pl->n_units = base_units;
    pl->n_steps = base_steps;
    pl->g0[base_units] = base_steps;
    pl->active_tiles = act;
  }
}

// Output-stationary gather-GEMM over the CTA's tb tiles, offset-outer (see file header).
// NPW: gather producer warps (4: up to three CTAs per SM; 8: two CTAs per SM, 16 issuing warps).
template <int CH, bool EPI, int NPW>  // EPI: the fused epilogue is compiled in (plain convs keep the lean kernel)
__global__ void __launch_bounds__((NPW + 6) * 32, 2) k_conv_umma(const __grid_constant__ FwdParams p) {
  constexpr int kFwdEpi0 = NPW, kFwdMma = NPW + 4, kFwdStage = NPW + 5;
  constexpr int J = CH / 8;    // 16-byte chunks per gathered row
  constexpr int RB = CH * 2;   // bytes per gathered row (= swizzle span)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* a_base = smem;
  uint8_t* w_base = a_base + (size_t)p.sa * p.a_bytes;
  int32_t* nbr_s = (int32_t*)(w_base + (size_t)p.sw * p.b_bytes);  // [NPW][3][128] index buffers
  Plan* pl = (Plan*)(nbr_s + NPW * 3 * kTileM);
  uint64_t* a_full = (uint64_t*)(((uintptr_t)(pl + 1) + 15) & ~(uintptr_t)15);
  uint64_t* cb = a_full + p.sa;  // [ncb] commit ring (stage slots and W slots are released by it)
  uint64_t* w_full = cb + p.ncb;
  uint64_t* tfull = w_full + p.sw;
  uint32_t* tmem_slot = (uint32_t*)(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile0 = cta_tile0(p);
  const int y0 = (int)blockIdx.y * p.cw;        // this CTA's output columns [y0, y0 + cwj)
  const int cwj = min(p.cw, p.c_y - y0);
  const uint32_t wb = (uint32_t)cwj * RB;       // bytes of this CTA's slice of a W chunk

  // prologue that touches no global memory overlaps the predecessor kernel (PDL)
  if (threadIdx.x == 32) {
    for (int s = 0; s < p.sa; ++s) mbar_init(a_full + s, 32);  // one cp.async arrival per lane
    for (int j = 0; j < p.ncb; ++j) mbar_init(cb + j, 1);
    for (int s = 0; s < p.sw; ++s) mbar_init(w_full + s, 1);
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == kFwdMma) tmem_alloc_dyn(tmem_slot, p.tmem_cols);
  pdl_enter();
  if (warp == 0) build_plan(p, pl);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int n_units = pl->n_units, n_steps = pl->n_steps;
  ACCT_DECL
#ifdef MK_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_cta[blockIdx.x][0] = gtime();
    g_cta[blockIdx.x][2] = smid;
    g_cta[blockIdx.x][3] = (unsigned long long)n_steps;
  }
#endif

  if (warp < p.np) {
    // ------------------------------------------------------------ gather producers
    // Step g (128 rows x CH channels of one (unit, tile, chunk)) belongs to warp g % np and
    // uses stage slot g % sa (np divides sa; by default np = sa).  Lane group
    // q4 = lane/8 owns rows [32 q4, 32 q4 + 32), 8 lanes per 128-byte row (4 full lines per
    // instruction); absent neighbours are zero-filled by cp.async with a 0-byte source.
    // Completion is announced by the copy engine itself: every lane's
    // cp.async.mbarrier.arrive.noinc fires when its copies have landed (the slot's full
    // barrier expects 32 arrivals), so the warp never waits for its own gathers.  The
    // step's 128 neighbour indices are prefetched two steps ahead (ring of 3 buffers, in
    // the cp.async group of the step two before); wait_group 1 keeps the ring safe.
    int32_t* ibuf = nbr_s + warp * 3 * kTileM;
    int u = 0;
    auto locate = [&](int g, int* k, int64_t* tile, int* c) {
      while (pl->g0[u + 1] <= g) ++u;
      const int q = g - pl->g0[u];
      const int j = q / p.nch;
      *c = q - j * p.nch;
      uint32_t tw = pl->tw[u];
      for (int t = 0; t < j; ++t) tw &= tw - 1;
      *tile = cta_tile(p, __ffs(tw) - 1);
      *k = pl->k[u];
    };
    auto fetch_idx = [&](int g, int buf) {
      int k, c;
      int64_t tile;
      locate(g, &k, &tile, &c);
      cp_async16(smem_u32(ibuf + buf * kTileM) + lane * 16,
                 p.nb.tab + (int64_t)p.nb.kk(k) * p.nb.n + tile * kTileM + lane * 4, 16u);
      return c;
    };
    const int np = p.np;
    constexpr int RG = kTileM / (32 / J);  // rows per lane group (32 / J groups of J lanes)
    const int q4 = lane / J, jj = lane & (J - 1);
    const int c_x = p.c_x;
    // indices of the warp's first two steps
    int cq[3] = {0, 0, 0};  // channel chunk of the step whose indices sit in buffer i
    if (warp < n_steps) cq[0] = fetch_idx(warp, 0);
    if (warp + np < n_steps) cq[1] = fetch_idx(warp + np, 1);
    cp_async_commit();
    cp_async_wait_n(0);
    __syncwarp();
    int jl = 0;  // warp-local step index
    for (int g = warp; g < n_steps; g += np, ++jl) {
      const int b = jl % 3;
      const int c = cq[b];
      if (g + 2 * np < n_steps) cq[(jl + 2) % 3] = fetch_idx(g + 2 * np, (jl + 2) % 3);
      const int slot = g % p.sa;
      if (g >= p.sa) {  // slot reuse: all MMAs of step g - sa done
        const int j = (g - p.sa) / p.ga;
        ACCT_WAIT(0, cb + (j & (p.ncb - 1)), (uint32_t)(j / p.ncb) & 1u);
      }
      ACCT_NOW(t_issue);
      const uint32_t a_s = smem_u32(a_base + (size_t)slot * p.a_bytes);
      const int32_t* ix = ibuf + b * kTileM;
      const __nv_bfloat16* xc = p.x + c * CH;
      if (p.dbg & 2) {
      } else if (p.off32) {
        // lane group q4 = lane / J owns rows [q4 RG, q4 RG + RG), lane jj its 16-byte column:
        // one 16-byte index load per 4 rows, 32-bit element offsets, ignore-src zero fill
#pragma unroll 2
        for (int i = 0; i < RG; i += 4) {
          const int4 a4 = *(const int4*)(ix + q4 * RG + i);
          const int av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = q4 * RG + i + e;
            cp_async16_z(a_s + swz(r, jj, RB), xc + ((uint32_t)max(av[e], 0) * (uint32_t)c_x + jj * 8), av[e] < 0);
          }
        }
      } else if (J == 8) {
#pragma unroll 2
        for (int i = 0; i < 32; i += 4) {
          const int4 a4 = *(const int4*)(ix + q4 * 32 + i);
          const int av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = q4 * 32 + i + e;
            cp_async16(a_s + swz(r, jj, RB), xc + (int64_t)max(av[e], 0) * p.c_x + jj * 8, av[e] >= 0 ? 16u : 0u);
          }
        }
      } else {
#pragma unroll 4
        for (int sl = lane; sl < 128 * J; sl += 32) {
          const int r = sl / J, j2 = sl % J;
          const int32_t av = ix[r];
          cp_async16(a_s + swz(r, j2, RB), xc + (int64_t)max(av, 0) * p.c_x + j2 * 8, av >= 0 ? 16u : 0u);
        }
      }
      cp_async_arrive_noinc(a_full + slot);
      cp_async_commit();
      ACCT_ADD(1, t_issue);
      ACCT_NOW(t_wg);
      cp_async_wait_n(1);  // group of step g - np done: the index buffer of step g + np is complete
      __syncwarp();
      ACCT_ADD(3, t_wg);
#ifdef MK_TRACE
      acct[4] += 1;
#endif
    }
    cp_async_wait_n(0);
  } else if (warp == kFwdStage) {
    // ------------------------------------------------------------ W stager (one thread)
    // Bulk copies (TMA engine) of the W_k chunks of every unit into a ring of sw slots.  A
    // slot is free once every MMA of its previous unit uo completed; no extra commit is spent
    // on that: the group commit covering uo's last step (commit ring cb) implies it.
    // Deadlock-free because the ring holds >= ga units.
    if (lane == 0) {
      uint32_t ws = 0;
      const int upr = p.sw / p.nch;  // units held by the ring
      for (int u = 0; u < n_units; ++u) {
        const int uo = u - upr;
        if (uo >= 0) {
          const int j = (pl->g0[uo + 1] - 1) / p.ga;  // commit covering uo's last step
          ACCT_WAIT(0, cb + (j & (p.ncb - 1)), (uint32_t)(j / p.ncb) & 1u);
        }
        for (int c = 0; c < p.nch; ++c) {
          mbar_arrive_expect_tx(w_full + ws, wb);
          bulk_g2s(w_base + (size_t)ws * p.b_bytes, p.wpack + ((int64_t)pl->k[u] * p.nch + c) * p.b_img + y0 * RB, wb,
                   w_full + ws);
          if (++ws == (uint32_t)p.sw) ws = 0;
        }
      }
    }
    __syncwarp();
  } else if (warp == kFwdMma) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop with warp-uniform values (so descriptors live in uniform
    // registers: no per-MMA R2UR); lane 0 issues the tcgen05 instructions.  Descriptors are
    // a constant high part | (smem address >> 4); slot / phase counters are incremental;
    // one commit per group of ga stage slots.
    {
      const uint32_t idesc = idesc_bf16(kTileM, (uint32_t)cwj, 0, 0);
      const uint64_t dhi = smem_desc(0, 16, 8 * RB, layout_code(RB));
      const uint32_t a0 = __shfl_sync(0xffffffffu, smem_u32(a_base) >> 4, 0), astep = p.a_bytes >> 4;
      const uint32_t w0 = __shfl_sync(0xffffffffu, smem_u32(w_base) >> 4, 0), wstep = p.b_bytes >> 4;
      const uint32_t tb0 = __shfl_sync(0xffffffffu, tbase, 0);
      uint32_t s = 0, sph = 0, gq = 0;     // A slot, its phase, position inside the commit group
      uint32_t ncommit = 0;                // group commits issued (commit ring index)
      uint32_t ws = 0, wph = 0;            // W ring position of the unit's first chunk
      uint32_t init = 0;                   // tiles whose accumulator holds data
      for (int u = 0; u < n_units; ++u) {
        const uint32_t tw = __shfl_sync(0xffffffffu, (uint32_t)pl->tw[u], 0);
        {  // wait for the unit's W chunks
          uint32_t x = ws, xph = wph;
          for (int c = 0; c < p.nch; ++c) {
            ACCT_WAIT(1, w_full + x, xph);
            if (++x == (uint32_t)p.sw) {
              x = 0;
              xph ^= 1;
            }
          }
        }
        tc_fence_after();
        for (uint32_t b = tw; b; b &= b - 1) {
          const int i = __ffs(b) - 1;
          const uint32_t d = tb0 + (uint32_t)(i * p.cw);
          uint32_t acc = (init >> i) & 1u;
          uint32_t x = ws;
          if (p.grp) {
            // grouped: the nch chunk steps of this (unit, tile) as one MMA step — one fence,
            // one elected block of nch * CH / 16 UMMAs and one commit (ga == nch) instead of
            // nch of each (the MMA warp's per-step overhead bounds the C = 96 kernel)
            uint32_t s2 = s, ph2 = sph;
            for (int c = 0; c < p.nch; ++c) {
              ACCT_WAIT(2, a_full + s2, ph2);
              if (++s2 == (uint32_t)p.sa) {
                s2 = 0;
                ph2 ^= 1;
              }
            }
            ACCT_NOW(t_f);
            fence_proxy_async_smem();
            tc_fence_after();
            ACCT_ADD(3, t_f);
            ACCT_NOW(t_i);
            if (elect_one() && !(p.dbg & 1)) {
              uint32_t sc = s, xc = x;
              for (int c = 0; c < p.nch; ++c) {
                const uint32_t alo = a0 + sc * astep, blo = w0 + xc * wstep;
#pragma unroll
                for (int kk = 0; kk < CH / 16; ++kk)
                  umma_f16(d, dhi | (uint64_t)(alo + kk * 2), dhi | (uint64_t)(blo + kk * 2), idesc,
                           acc | (uint32_t)c | (uint32_t)kk);
                if (++sc == (uint32_t)p.sa) sc = 0;
                if (++xc == (uint32_t)p.sw) xc = 0;
              }
              umma_commit(cb + (ncommit & (uint32_t)(p.ncb - 1)));
            }
            ++ncommit;
            __syncwarp();
            ACCT_ADD(4, t_i);
#ifdef MK_TRACE
            acct[6] += p.nch;
#endif
            s = s2;
            sph = ph2;
            init |= 1u << i;
            continue;
          }
          for (int c = 0; c < p.nch; ++c) {
            ACCT_WAIT(2, a_full + s, sph);
            ACCT_NOW(t_f);
            fence_proxy_async_smem();  // the cp.async (generic proxy) rows -> tcgen05 (async proxy)
            tc_fence_after();
            const uint32_t alo = a0 + s * astep, blo = w0 + x * wstep;
            ACCT_ADD(3, t_f);
            ACCT_NOW(t_i);
            if (elect_one() && !(p.dbg & 1)) {
#pragma unroll
              for (int kk = 0; kk < CH / 16; ++kk)
                umma_f16(d, dhi | (uint64_t)(alo + kk * 2), dhi | (uint64_t)(blo + kk * 2), idesc, acc | (uint32_t)kk);
            }
            acc = 1;
            __syncwarp();
            ACCT_ADD(4, t_i);
            ACCT_NOW(t_c);
            // a commit stalls the next MMAs ~250 cycles (tools/ubench_umma.cu): one per ga steps
            if (++gq == (uint32_t)p.ga) {
              if (elect_one()) umma_commit(cb + (ncommit & (uint32_t)(p.ncb - 1)));
              ++ncommit;
              gq = 0;
            }
            __syncwarp();
            ACCT_ADD(5, t_c);
#ifdef MK_TRACE
            acct[6] += 1;
#endif
            if (++s == (uint32_t)p.sa) {
              s = 0;
              sph ^= 1;
            }
            if (++x == (uint32_t)p.sw) x = 0;
          }
          init |= 1u << i;
        }
        for (int c = 0; c < p.nch; ++c)
          if (++ws == (uint32_t)p.sw) {
            ws = 0;
            wph ^= 1;
          }
      }
      if (n_steps > 0 && elect_one()) umma_commit(tfull);
      __syncwarp();
    }
  } else if (warp >= kFwdEpi0 && warp < kFwdEpi0 + 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter owned by this warp
    if (n_steps > 0) {
      ACCT_WAIT(0, tfull, 0);
      tc_fence_after();
    }
    const uint32_t act = pl->active_tiles;
    for (int i = 0; i < p.tb; ++i) {
      const int64_t tile = cta_tile(p, i);
      if (tile < 0) break;
      const int64_t pos = tile * kTileM + q * 32 + lane;  // position in the map's row order
      const bool valid = pos < p.n_rows;
      const int64_t row = valid ? p.nb.row_of(pos) : 0;
      if (!((act >> i) & 1u)) {  // no offset in this tile: the conv output is 0
        if (valid)
          for (int col0 = y0; col0 < y0 + cwj; col0 += 16) {
            uint32_t v[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = 0u;
            if (EPI) epi16(p, row, col0, v);
            store16(p, row, col0, v);
          }
        continue;
      }
      const uint32_t tl_addr = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(i * p.cw);
      for (int col0 = 0; col0 < cwj; col0 += 16) {
        uint32_t v[16];
        tmem_ld16(tl_addr + col0, v);
        tmem_ld_wait();
        if (valid) {
          if (EPI) epi16(p, row, y0 + col0, v);
          store16(p, row, y0 + col0, v);
        }
      }
    }
  }
#ifdef MK_TRACE
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < 4096) g_cta[blockIdx.x][1] = gtime();
#endif
  ACCT_DUMP;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kFwdMma) tmem_dealloc(tbase, p.tmem_cols);
}

// ------------------------------------------------------------------ weight gradient
struct WgradParams {
  const __nv_bfloat16* g;  // [n_out][c_out]
  const __nv_bfloat16* x;  // [n_in][c_in]
  const int32_t* in_idx;
  const int32_t* out_idx;
  const int4* segs;          // (k, begin, end, slot), grouped by CTA
  const int32_t* seg_begin;  // [n_cta + 1]
  const int64_t* ptr;        // [K + 1] device CSR offsets (device-side plans)
  int32_t* jtab;             // strided plan: [2K] (first CTA, CTAs) of every offset, written by CTA 0
  int K;
  int mode;                  // plan: 0 contiguous ranges, 1 host segments, 2 strided per-offset chunks
  float* part;               // [n_slots][c_out][c_in]
  int c_out, c_in, halves;
  int mrows;                 // UMMA M: 64 when C_out <= 64 (no zero panel), else 128 per half
  int sa, ga;                // stage slots, slots per commit group
  int wps;                   // producer warps per stage slot (each gathers 64 / wps pairs of a step)
  int a_pad;                 // A holds zeroed padding panels (else a_bytes = the real panels only)
  int nacc;                  // TMEM accumulators per half the K steps alternate between (1 or 2)
  int off32;                 // n_out * c_out and n_in * c_in < 2^31: 32-bit element offsets
  unsigned* gsync;           // strided plan: per-epoch arrival counters (zeroed), or nullptr
  int sync_b, sync_s, sync_emax;  // rounds per epoch, epochs of slack, counter capacity
  int pwa, pwb;              // panel widths (channels) of A (G) and B (X)
  uint32_t a_bytes, b_bytes, slot_bytes, tmem_cols;
};

constexpr int kPairsPerStage = 64;

// Pairs per CTA of the weight-gradient split (the same rule as kmap_wplan's host plan):
// L = 64 * ceil(ceil(P / n_cta) / 64), at least 64.
__host__ __device__ __forceinline__ int64_t wgrad_range(int64_t P, int64_t n_cta) {
  const int64_t per = (P > 0 ? P : 1) / n_cta + (((P > 0 ? P : 1) % n_cta) != 0);
  const int64_t L = ((per + 63) / 64) * 64;
  return L < 64 ? 64 : L;
}

// dW_k = sum of the partials of offset k's segments, in CTA order (deterministic).  With the
// device plan, segment (c, k) sits in slot c + k and offset k spans CTAs ptr[k] / L ..
// (ptr[k+1] - 1) / L.
__global__ void k_reduce_partials_dev(const int64_t* __restrict__ ptr, int n_cta, const float* __restrict__ part,
                                      int64_t tile_elems, float* __restrict__ dW) {
  pdl_enter();
  const int k = blockIdx.y;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= tile_elems) return;
  const int64_t L = wgrad_range(__ldg(ptr + gridDim.y), n_cta);
  const int64_t b = __ldg(ptr + k), en = __ldg(ptr + k + 1);
  float s = 0.f;
  if (b < en)
    for (int64_t c = b / L; c <= (en - 1) / L; ++c) s += part[(c + k) * tile_elems + e];
  dW[(int64_t)k * tile_elems + e] = s;
}
// Strided plan (mode 2): dW_k = sum of the partials of offset k's CTAs jtab[k] ..
// jtab[k] + jtab[K + k] - 1 in CTA order (deterministic).
__global__ void k_reduce_partials_jtab(const int32_t* __restrict__ jtab, int K, const float* __restrict__ part,
                                       int64_t tile_elems, float* __restrict__ dW) {
  pdl_enter();
  const int k = blockIdx.y;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= tile_elems) return;
  const int c0 = __ldg(jtab + k), n = __ldg(jtab + K + k);
  float s = 0.f;
  for (int c = c0; c < c0 + n; ++c) s += part[(int64_t)c * tile_elems + e];
  dW[(int64_t)k * tile_elems + e] = s;
}
constexpr int kMaxSegs = kWgradMaxSegs + 1;  // per-CTA plan capacity (kmap_wplan cuts ranges to fit)

// Weight gradient: split-K over the pairs.  Step g = 64 pairs of one segment (k, range) of
// this CTA, done by producer warp g % sa in its own stage slot (warp-per-stage, as in the
// forward kernel): the warp prefetches the next step's 64 out/in indices (4-byte cp.async,
// private double buffer), gathers the 64 G rows into the MN-major A panels and the 64 X
// rows into the MN-major B panels (16-byte cp.async, zero-fill past the segment end),
// waits for its group and arrives once.  The MMA thread accumulates a segment in TMEM
// (M = C_out padded to 128 with a constant zero panel, N = C_in, K = 16 pairs), commits
// stage slots in groups, and publishes the segment to the epilogue, which writes the fp32
// partial dW_k tile of the segment's slot.
// NP producer warps (>= the stage slots in use); NP = 16: one CTA per SM; NP = 8: two CTAs
// per SM; NP = 4: three (shared memory split accordingly).
template <int NP, bool P3>  // P3: the period-3 gather path is compiled in (C = 48 / 96 operands)
__global__ void __launch_bounds__((NP + 5) * 32, NP >= 16 ? 1 : NP >= 8 ? 2 : 3)
    k_wgrad_umma(const __grid_constant__ WgradParams p) {
  constexpr int kEpiWarp0 = NP;                    // epilogue warps (TMEM lane quarters 0-3)
  constexpr int kMmaWarp = NP + kEpiWarps;         // the MMA issuer
  constexpr int kThreads = (NP + kEpiWarps + 1) * 32;
  constexpr int PS = kPairsPerStage;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  int32_t* ibuf_all = (int32_t*)(smem + (size_t)p.sa * p.slot_bytes);  // [sa * wps][2][2][64] (one per producer warp)
  int32_t* seg_g0 = ibuf_all + p.sa * p.wps * 4 * PS;                  // [kMaxSegs + 1]
  int4* s_segs = align16<int4>(seg_g0 + kMaxSegs + 2);  // [kMaxSegs]
  int* s_nseg = (int*)(s_segs + kMaxSegs);
  int64_t* s_rng = align16<int64_t>(s_nseg + 1);  // strided plan: [ptr_k, ptr_k+1, j, J]
  uint64_t* a_full = align16<uint64_t>(s_rng + 4);
  uint64_t* a_empty = a_full + p.sa;
  uint64_t* tfull = a_empty + p.sa;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);
  volatile int* s_sync = (volatile int*)(tmem_slot + 1);  // [epochs, allowed epochs, MMA steps done]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rba = p.pwa * 2, rbb = p.pwb * 2;             // panel row bytes
  const int npa = p.c_out / p.pwa;  // real A panels
  const uint32_t panel_a = PS * rba, panel_b = PS * rbb;  // panel strides (LBO)

  pdl_enter();
  if (warp == 0) {  // plan: this CTA's segments and the first step of every segment
    int nseg = 0;
    if (p.mode == 2) {
      // Strided per-offset plan: offset k gets J_k CTAs (one more than its share of the
      // 64-pair chunks beyond one per non-empty offset, largest remainder first); CTA j of
      // offset k takes chunks j, j + J_k, j + 2 J_k, ... of k's output-sorted pair list and
      // accumulates all of them into ONE partial.  Every offset then advances through its
      // pairs at the same relative speed, so the CTAs running at any moment all read the
      // same window of output rows (and their neighbours): the G and X rows they gather stay
      // in L2 even when the features are far larger than L2 (configs[4]).  K <= 32.
      const int k = lane;
      const int64_t b = k < p.K ? __ldg(p.ptr + k) : 0, en = k < p.K ? __ldg(p.ptr + k + 1) : 0;
      const int64_t ck = (en - b + PS - 1) / PS;
      int64_t C = ck;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) C += __shfl_xor_sync(0xffffffffu, C, o);
      const int nz = __popc(__ballot_sync(0xffffffffu, ck > 0));
      const int64_t spare = (int64_t)gridDim.x - nz;
      int J = 0;
      int64_t rem = -1;
      if (ck > 0 && C > 0) {
        J = 1 + (int)(spare * ck / C);
        rem = spare * ck % C;
      }
      int given = J;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) given += __shfl_xor_sync(0xffffffffu, given, o);
      const int extra = (int)gridDim.x - given;  // < nz
      int rank = 0;  // lanes with a larger remainder (ties: lower offset first)
      for (int l = 0; l < 32; ++l) {
        const int64_t rl = __shfl_sync(0xffffffffu, rem, l);
        rank += (rl > rem) || (rl == rem && l < lane);
      }
      if (rem >= 0 && rank < extra) ++J;
      int c0 = J;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, c0, o);
        if (lane >= o) c0 += y;
      }
      c0 -= J;
      if (blockIdx.x == 0 && k < p.K) {  // for the reduction: CTAs c0 .. c0 + min(J, ck) - 1
        p.jtab[k] = c0;
        p.jtab[p.K + k] = (int)min((int64_t)J, ck);
      }
      const int c = (int)blockIdx.x;
      // the CTA's offset; CTAs j >= ck of an offset (more CTAs than chunks) stay idle
      const unsigned mine = __ballot_sync(0xffffffffu, J > 0 && c >= c0 && c < c0 + J && c - c0 < ck);
      if (lane == 0) seg_g0[0] = 0;
      __syncwarp();
      if (mine) {
        const int km = __ffs(mine) - 1;
        if (lane == km) {
          const int j = c - c0;
          s_rng[0] = b;
          s_rng[1] = en;
          s_rng[2] = j;
          s_rng[3] = J;
          s_segs[0] = make_int4(k, 0, 0, c);
          seg_g0[1] = (int)((ck - j + J - 1) / J);
        }
        nseg = 1;
      }
      __syncwarp();
      if (lane == 0) *s_nseg = nseg;
      // Epoch throttle: the CTAs drift apart over ~1000 rounds (one chunk each), which widens
      // the window of rows read at once beyond L2.  With gsync, every CTA arrives at a global
      // counter after each epoch of sync_b rounds and its producers stay within sync_s epochs of
      // the last epoch all CTAs completed (all CTAs are co-resident: grid = CTAs per SM x SMs).
      int rounds = J > 0 ? (int)((ck + J - 1) / J) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
      if (lane == 0) {
        s_sync[0] = p.gsync ? min((rounds + p.sync_b - 1) / p.sync_b, p.sync_emax) : 0;
        s_sync[1] = p.gsync ? p.sync_s + 1 : INT_MAX;
        s_sync[2] = 0;
      }
    } else if (p.segs) {  // host plan (kmap_wplan)
      const int sb = p.seg_begin[blockIdx.x], se = min(p.seg_begin[blockIdx.x + 1], sb + kMaxSegs);
      nseg = se - sb;
      for (int i = lane; i < nseg; i += 32) s_segs[i] = p.segs[sb + i];
    } else {  // device plan: CTA c takes pairs [c L, (c+1) L); segment (c, k) uses slot c + k
      const int64_t P = __ldg(p.ptr + p.K), L = wgrad_range(P, gridDim.x);
      const int64_t cb = (int64_t)blockIdx.x * L, ce = min(P, cb + L);
      for (int k0 = 0; k0 < p.K; k0 += 32) {
        const int k = k0 + lane;
        int64_t b = 0, e = 0;
        if (k < p.K) {
          b = max(cb, __ldg(p.ptr + k));
          e = min(ce, __ldg(p.ptr + k + 1));
        }
        const bool has = k < p.K && b < e;
        const unsigned bal = __ballot_sync(0xffffffffu, has);
        if (has) s_segs[nseg + __popc(bal & ((1u << lane) - 1u))] = make_int4(k, (int)b, (int)e, (int)blockIdx.x + k);
        nseg += __popc(bal);
      }
    }
    __syncwarp();
    int base = 0;
    for (int i0 = 0; i0 < nseg && p.mode != 2; i0 += 32) {
      const int i = i0 + lane;
      const int4 sg = i < nseg ? s_segs[i] : make_int4(0, 0, 0, 0);
      const int st = i < nseg ? (sg.z - sg.y + PS - 1) / PS : 0;
      int incl = st;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (i < nseg) seg_g0[i] = base + incl - st;
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0 && p.mode != 2) {
      seg_g0[nseg] = base;
      *s_nseg = nseg;
    }
  }
  if (threadIdx.x == 32) {
    if (p.mode != 2) {
      s_sync[0] = 0;
      s_sync[1] = INT_MAX;
      s_sync[2] = 0;
    }
    for (int s = 0; s < p.sa; ++s) {
      mbar_init(a_full + s, p.wps);
      mbar_init(a_empty + s, 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kEpiWarps * 32);
    fence_mbar_init();
  }
  // zero the padding panels of A (M padded to 128 per half) once; never overwritten.  Without
  // them (a_pad = 0, default) the padding rows of the UMMA read whatever follows the real
  // panels (the slot's B panels or the next slot): they only feed accumulator rows >= C_out,
  // which are never stored.
  if (p.a_pad) {
    const int tot_pa = (int)(p.a_bytes / panel_a);
    for (int s = 0; s < p.sa; ++s)
      for (int pa = npa; pa < tot_pa; ++pa) {
        uint4* z = (uint4*)(smem + (size_t)s * p.slot_bytes + (size_t)pa * panel_a);
        for (int i = threadIdx.x; i < (int)(panel_a / 16); i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
      }
  }
  if (warp == kMmaWarp) tmem_alloc_dyn(tmem_slot, p.tmem_cols);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int nseg = *s_nseg;
  const int n_steps = seg_g0[nseg];
  ACCT_DECL

  if (warp < p.sa * p.wps) {
    // ------------------------------------------------------------ gather producers
    // Warp w fills stage slot w / wps with pairs [PW part, PW part + PW) of the slot's steps
    // (PW = 64 / wps, part = w % wps): when the channel counts leave fewer slots than
    // producer warps, every warp still gathers (more warps issuing = more gathers in flight).
    const int slot = warp / p.wps, part = warp - slot * p.wps, PW = PS / p.wps, pr0 = part * PW, pr1 = pr0 + PW;
    int32_t* ib_w = ibuf_all + warp * 4 * PS;  // [2][out, in][64]
    int si = 0;
    const int64_t r_b = s_rng[0], r_e = s_rng[1], r_j = s_rng[2], r_J = s_rng[3];
    auto locate = [&](int g, int* b0, int* e) {
      if (p.mode == 2) {  // chunk j + g J of the offset
        *b0 = (int)(r_b + (r_j + (int64_t)g * r_J) * PS);
        *e = (int)r_e;
        return;
      }
      while (seg_g0[si + 1] <= g) ++si;
      const int4 sg = s_segs[si];
      *b0 = sg.y + (g - seg_g0[si]) * PS;
      *e = sg.z;
    };
    auto fetch_idx = [&](int b0, int e, int buf) {
      int32_t* d = ib_w + buf * 2 * PS;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = pr0 + lane + 32 * h;
        if (i < pr1 && b0 + i < e) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(d + i)), "l"(p.out_idx + b0 + i) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(d + PS + i)), "l"(p.in_idx + b0 + i)
                       : "memory");
        }
      }
    };
    int g = slot, b0 = 0, e = 0, b0n = 0, en = 0;
    if (g < n_steps) {
      locate(g, &b0, &e);
      fetch_idx(b0, e, 0);
      cp_async_commit();
      cp_async_wait_n(0);
      __syncwarp();
    }
    uint32_t my = 0, ib = 0;
    const int ca = p.c_out / 8, cb = p.c_in / 8;  // 16-byte chunks per G row / X row
    const __nv_bfloat16* const g_base = p.g;
    const __nv_bfloat16* const x_base = p.x;
    const int c_out_r = p.c_out, c_in_r = p.c_in;
    const int ja = rba / 16, jb = rbb / 16;       // chunks per panel row (2, 4 or 8)
    const int lja = __ffs(ja) - 1, ljb = __ffs(jb) - 1;  // (panel = chunk >> l: no integer division)
    // Period-3 path (96 % c8 == 0, 96 / c8 rows a multiple of 8: C = 48, 96): three warp
    // instructions cover 96 / c8 whole rows, and since the swizzle pattern repeats every 8 rows
    // each lane's (row, smem offset, source offset) triple per instruction is fixed: ~6
    // instructions per 16-byte copy instead of ~30 with the running (row, chunk) carry.
    struct Per3 {
      int r[3], d[3], c[3];
      int rows;
    };
    auto per3 = [&](int c8, int jx, int ljx, uint32_t panel, int rbx) {
      Per3 t;
      t.rows = 0;
      if (P3 && p.off32 && c8 > 0 && (32 % c8) != 0 && 96 % c8 == 0 && (96 / c8) % 8 == 0) {
        t.rows = 96 / c8;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int q = lane + 32 * i, r = q / c8, ch = q - r * c8;
          t.r[i] = r;
          t.c[i] = ch * 8;
          t.d[i] = (int)((uint32_t)(ch >> ljx) * panel + swz((uint32_t)r, (uint32_t)(ch & (jx - 1)), (uint32_t)rbx));
        }
      }
      return t;
    };
    const Per3 pa3 = per3(c_out_r / 8, ja, lja, panel_a, rba), pb3 = per3(c_in_r / 8, jb, ljb, panel_b, rbb);
    for (; g < n_steps; g += p.sa) {
      const bool have_n = g + p.sa < n_steps;
      if (have_n) {
        locate(g + p.sa, &b0n, &en);
        fetch_idx(b0n, en, ib ^ 1);
      }
      if (g / p.sync_b >= s_sync[1]) {  // epoch throttle (strided plan)
        while (g / p.sync_b >= s_sync[1]) __nanosleep(128);
      }
      ACCT_WAIT(0, a_empty + slot / p.ga, (my & 1) ^ 1);
      ACCT_NOW(t_issue);
      const uint32_t a_s = smem_u32(smem + (size_t)slot * p.slot_bytes), b_s = a_s + p.a_bytes;
      const int32_t* oi = ib_w + ib * 2 * PS;
      const int32_t* ii = oi + PS;
      // G rows -> A panels, X rows -> B panels.  Fast path when a row's chunk count divides
      // the warp: each lane keeps one chunk column (no per-element divisions).
      if (P3 && pa3.rows) {
        for (int R0 = pr0; R0 < pr1; R0 += pa3.rows) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int pr = R0 + pa3.r[i];
            const bool v = b0 + pr < e;
            const uint32_t row = v ? (uint32_t)oi[pr] : 0u;  // (32-bit element offsets: host-checked)
            cp_async16_z(a_s + (uint32_t)(R0 * rba + pa3.d[i]), g_base + (row * (uint32_t)c_out_r + pa3.c[i]), !v);
          }
        }
      } else if ((32 % ca) == 0) {
        const int ch = lane % ca, pa = ch / ja, j = ch - pa * ja;
        const __nv_bfloat16* src = p.g + ch * 8;
        const uint32_t dst0 = a_s + pa * panel_a;
#pragma unroll 4
        for (int pr = pr0 + lane / ca; pr < pr1; pr += 32 / ca) {
          const uint32_t dst = dst0 + swz(pr, j, rba);
          if (b0 + pr < e) cp_async16(dst, src + (int64_t)oi[pr] * p.c_out, 16u);
          else st_shared_zero16(dst);
        }
      } else {  // consecutive lanes take consecutive 16-byte chunks (whole sectors per row)
        int pr = pr0 + lane / ca, ch = lane - (lane / ca) * ca;
        const int dpr = 32 / ca, dch = 32 - dpr * ca;
        const __nv_bfloat16* const gsrc = g_base;  // registers: the asm memory clobbers would reload params
        const int cst = c_out_r;
#pragma unroll 2
        for (; pr < pr1;) {
          const int pa = ch >> lja, j = ch & (ja - 1);
          const uint32_t dst = a_s + pa * panel_a + swz(pr, j, rba);
          if (b0 + pr < e) cp_async16(dst, gsrc + (int64_t)oi[pr] * cst + ch * 8, 16u);
          else st_shared_zero16(dst);
          pr += dpr;
          ch += dch;
          if (ch >= ca) {
            ch -= ca;
            ++pr;
          }
        }
      }
      if (P3 && pb3.rows) {
        for (int R0 = pr0; R0 < pr1; R0 += pb3.rows) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int pr = R0 + pb3.r[i];
            const bool v = b0 + pr < e;
            const uint32_t row = v ? (uint32_t)ii[pr] : 0u;
            cp_async16_z(b_s + (uint32_t)(R0 * rbb + pb3.d[i]), x_base + (row * (uint32_t)c_in_r + pb3.c[i]), !v);
          }
        }
      } else if ((32 % cb) == 0) {
        const int ch = lane % cb, pb = ch / jb, j = ch - pb * jb;
        const __nv_bfloat16* src = p.x + ch * 8;
        const uint32_t dst0 = b_s + pb * panel_b;
#pragma unroll 4
        for (int pr = pr0 + lane / cb; pr < pr1; pr += 32 / cb) {
          const uint32_t dst = dst0 + swz(pr, j, rbb);
          if (b0 + pr < e) cp_async16(dst, src + (int64_t)ii[pr] * p.c_in, 16u);
          else st_shared_zero16(dst);
        }
      } else {
        int pr = pr0 + lane / cb, ch = lane - (lane / cb) * cb;
        const int dpr = 32 / cb, dch = 32 - dpr * cb;
        const __nv_bfloat16* const xsrc = x_base;
        const int cst = c_in_r;
#pragma unroll 2
        for (; pr < pr1;) {
          const int pb = ch >> ljb, j = ch & (jb - 1);
          const uint32_t dst = b_s + pb * panel_b + swz(pr, j, rbb);
          if (b0 + pr < e) cp_async16(dst, xsrc + (int64_t)ii[pr] * cst + ch * 8, 16u);
          else st_shared_zero16(dst);
          pr += dpr;
          ch += dch;
          if (ch >= cb) {
            ch -= cb;
            ++pr;
          }
        }
      }
      cp_async_commit();
      ACCT_ADD(1, t_issue);
      ACCT_NOW(t_land);
      cp_async_wait_n(0);
      fence_proxy_async_smem();
      __syncwarp();
      ACCT_ADD(2, t_land);
      if (lane == 0) mbar_arrive(a_full + slot);
      ++my;
#ifdef MK_TRACE
      acct[3] += 1;
#endif
      ib ^= 1;
      b0 = b0n;
      e = en;
    }
  } else if (warp == kMmaWarp) {
    {  // whole warp, warp-uniform values, lane 0 issues (see the forward kernel)
      const bool leader = lane == 0;
      const uint32_t idesc = idesc_bf16((uint32_t)p.mrows, p.c_in, 1, 1);
      const uint64_t ahi = smem_desc(0, panel_a, 8 * rba, layout_code(rba));
      const uint64_t bhi = smem_desc(0, panel_b, 8 * rbb, layout_code(rbb));
      const uint32_t s0 = __shfl_sync(0xffffffffu, smem_u32(smem) >> 4, 0), sstep = p.slot_bytes >> 4,
                     boff = p.a_bytes >> 4;
      const uint32_t tb0 = __shfl_sync(0xffffffffu, tbase, 0);
      const uint32_t ka = (16 * rba) >> 4, kb = (16 * rbb) >> 4, hstep = ((128 / p.pwa) * panel_a) >> 4;
      uint32_t s = 0, sph = 0, gq = 0;
      for (int i = 0; i < nseg; ++i) {
        mbar_wait(tempty, (i & 1) ^ 1);
        tc_fence_after();
        uint32_t acc = 0;
        const int q0 = __shfl_sync(0xffffffffu, seg_g0[i], 0), q1 = __shfl_sync(0xffffffffu, seg_g0[i + 1], 0);
        for (int q = q0; q < q1; ++q) {
          ACCT_WAIT(2, a_full + s, sph);
          ACCT_NOW(t_mma);
          tc_fence_after();
          const uint32_t alo = s0 + s * sstep, blo = alo + boff;
          ACCT_ADD(5, t_mma);
          ACCT_NOW(t_iss);
          // nacc = 2: the K steps alternate between two accumulators (summed by the epilogue),
          // so consecutive UMMAs do not wait on each other's accumulator (tools/ubench_umma.cu)
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < PS / 16; ++kk) {
              const uint32_t a = p.nacc == 2 ? (uint32_t)(kk & 1) : 0u;
              for (int h = 0; h < p.halves; ++h)
                umma_f16(tb0 + (a * p.halves + h) * (uint32_t)p.c_in, ahi | (uint64_t)(alo + h * hstep + kk * ka),
                         bhi | (uint64_t)(blo + kk * kb), idesc, acc | (uint32_t)(kk >= p.nacc));
            }
          }
          acc = 1;
          __syncwarp();
          ACCT_ADD(3, t_iss);
          ACCT_NOW(t_cm);
          if (++gq == (uint32_t)p.ga) {
            if (elect_one()) umma_commit(a_empty + s / p.ga);
            gq = 0;
          }
          if (leader) s_sync[2] = q + 1;  // steps consumed (the epoch throttle's progress)
          __syncwarp();
          ACCT_ADD(6, t_cm);
#ifdef MK_TRACE
          acct[4] += 1;
#endif
          if (++s == (uint32_t)p.sa) {
            s = 0;
            sph ^= 1;
          }
        }
        if (elect_one()) umma_commit(tfull);
        __syncwarp();
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
    const int q = warp & 3;
    if (warp == kEpiWarp0 && lane == 0 && s_sync[0] > 0) {
      // epoch throttle: arrive after each local epoch, open the next epochs once all CTAs
      // arrived; bounded spins (a wait that never ends disables the throttle instead)
      const int E = s_sync[0];
      long long spins = 0;
      for (int e = 0; e < E; ++e) {
        const int target = min((e + 1) * p.sync_b, n_steps);
        while (s_sync[2] < target) __nanosleep(256);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.gsync + e) : "memory");
        unsigned v;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.gsync + e) : "memory");
          if (v >= gridDim.x || ++spins > (1LL << 22)) break;
          __nanosleep(128);
        }
        if (v < gridDim.x) {
          s_sync[1] = INT_MAX;
          break;
        }
        s_sync[1] = e + 2 + p.sync_s;
      }
      s_sync[1] = INT_MAX;
    }
    __syncwarp();
    for (int i = 0; i < nseg; ++i) {
      const int4 sg = s_segs[i];
      ACCT_WAIT(0, tfull, i & 1);
      tc_fence_after();
      for (int h = 0; h < p.halves; ++h) {
        // M = 128: row m in TMEM lane m.  M = 64: row m in lane (m % 16) + 32 * (m / 16)
        // (half sub-partitions), so lanes 16..31 of each quarter hold no row.
        const int co = p.mrows == 64 ? (lane < 16 ? q * 16 + lane : p.c_out) : h * 128 + q * 32 + lane;
        float* dst = p.part + ((int64_t)sg.w * p.c_out + co) * p.c_in;
        const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + h * (uint32_t)p.c_in;
        for (int col0 = 0; col0 < p.c_in; col0 += 16) {
          uint32_t v[16];
          tmem_ld16(ta + col0, v);
          tmem_ld_wait();
          if (p.nacc == 2) {  // second accumulator (odd K steps)
            uint32_t v2[16];
            tmem_ld16(ta + (uint32_t)(p.halves * p.c_in) + col0, v2);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) + __uint_as_float(v2[e]));
          }
          if (co < p.c_out) {
            float4* d4 = (float4*)(dst + col0);
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4)
              d4[e4] = make_float4(__uint_as_float(v[4 * e4]), __uint_as_float(v[4 * e4 + 1]),
                                   __uint_as_float(v[4 * e4 + 2]), __uint_as_float(v[4 * e4 + 3]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
    }
  }
  ACCT_DUMP;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tbase, p.tmem_cols);
}


uint32_t pow2_cols(uint32_t c) {
  uint32_t r = 32;
  while (r < c) r <<= 1;
  return r;
}

// Raises a kernel's dynamic smem limit; the attribute call (~1 us of host time) is made only
// when the requested size grows past what was set before for that kernel.
template <class F>
void set_smem_once(F* f, int bytes) {
  struct Set {
    const void* f;
    int dev, bytes;
  };
  static std::mutex mu;
  static std::vector<Set> done;
  int dev = 0;
  cudaGetDevice(&dev);  // the attribute is per device
  std::lock_guard<std::mutex> lock(mu);
  for (auto& d : done)
    if (d.f == (const void*)f && d.dev == dev) {
      if (d.bytes >= bytes) return;
      if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess) d.bytes = bytes;
      return;
    }
  if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
    done.push_back({(const void*)f, dev, bytes});
}

}  // namespace

#ifdef MK_TRACE
extern "C" int mk_debug_trace(unsigned long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_trace, sizeof(g_trace));
}
extern "C" int mk_debug_acct(unsigned long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_acct, sizeof(g_acct));
}
extern "C" int mk_debug_cta(unsigned long long* host_out) {
  return (int)cudaMemcpyFromSymbol(host_out, g_cta, sizeof(g_cta));
}
#endif

mk_status launch_conv_bf16(mk_context* ctx, const NbrView& nb, const void* x, int64_t n_src, int c_x, const void* W,
                            int c_in_w, int c_out_w, void* y, int c_y, mk_dtype out_dt, int64_t n_rows, bool trans,
                            cudaStream_t s, const Epilogue& ep) {
  if (n_rows == 0) return MK_OK;
  if (nb.K > kMaxK) MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 conv: more than 128 kernel offsets");
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
  p.off32 = n_src * (int64_t)c_x < INT32_MAX;
  // An epilogue that only adds the fp32 output itself (y = conv + y, the bf16x3 split's running
  // sum) is an in-place accumulate: the plain instance (8 producer warps) instead of the fused
  // one (84 registers, 4 producer warps); the same fp32 additions, so bit-identical.
  p.accum = p.out_f32 && ep.residual == y && !ep.scale && !ep.shift && !ep.relu ? 1 : 0;
  p.ep = p.accum ? Epilogue() : ep;
  static const int dbg = [] {
    const char* e = std::getenv("MK_DEBUG_CONV");
    return e ? std::atoi(e) : 0;
  }();
  p.dbg = dbg;
  p.a_bytes = kTileM * CH * 2;
  p.b_img = (uint32_t)c_y * CH * 2;
  static const int env_fold = [] {  // default: 2 tiles per CTA, folded order (measured best)
    const char* e = std::getenv("MK_FWD_FOLD");
    return e ? std::atoi(e) : 2;
  }();
  static const int env_ctas0 = [] {  // CTAs per SM the smem budget aims at: 3 (default) or 2
    const char* e = std::getenv("MK_FWD_CTAS");
    return e && std::atoi(e) == 2 ? 2 : 3;
  }();
  static const int env_np = [] {
    const char* e = std::getenv("MK_FWD_NP");
    return e ? std::atoi(e) : 0;
  }();
  static const int env_npw = [] {  // producer warps of the two-CTA instance: 8 (default) or 4
    const char* e = std::getenv("MK_FWD_NPW");
    return e && std::atoi(e) == 4 ? 4 : 8;
  }();
  static const int env_samax = [] {  // development: stage slots per two-CTA CTA (default: one per producer warp)
    const char* e = std::getenv("MK_FWD_SAMAX");
    return e ? std::max(2, std::min(16, std::atoi(e))) : 0;
  }();
  p.fold = env_fold > 0 ? 1 : 0;
  // alignment + index buffers (3 per producer warp) + plan + TMEM slot; the barriers (a_full,
  // commit ring, W ring, tfull) are added per plan below
  auto base0 = [&](int npw) { return 1024 + npw * 3 * kTileM * 4 + (int)sizeof(Plan) + 16; };
  // commit-ring size for a plan (an upper bound over sa <= samax, ga >= 1; see kNCB)
  auto ring = [&](int sw, int tb, int samax) {
    int n = kNCB;
    while (n <= (sw / nch) * tb * nch + samax + 4) n *= 2;
    return n;
  };
  // Output columns per CTA.  All of C_out in one CTA when its W ring (2 units of nch chunks of
  // cw x CH) and two A stage slots fit the SM; otherwise the columns are split over
  // blockIdx.y (each CTA gathers the same rows and multiplies by its slice of W_k: e.g. C_in =
  // C_out = 256 needs 2 x 4 x 32 KB of W alone, over the 227 KB of an SM).
  // Producer warps: three CTAs per SM run the 4-warp instance (one stage slot per warp); two
  // CTAs per SM the 8-warp instance with up to 8 slots (16 issuing warps per SM: configs[4]
  // fwd 1239 -> 1113 us, dgrad 1229 -> 1098 us; gathers are latency bound per warp,
  // tools/ubench_ldgsts.cu), except the fused-epilogue instance (84 registers).
  int ysplit = 1, fixed = 0, ctas = 2, npw = kFwdProd, samax = kFwdProd;
  for (;; ++ysplit) {
    p.cw = 16 * (int)ceil_div(ceil_div(c_y, 16), ysplit);
    if (ysplit > 1 && (int64_t)(ysplit - 1) * p.cw >= c_y) continue;  // no empty column slice
    p.b_bytes = (uint32_t)p.cw * CH * 2;
    p.tb = p.fold ? std::max(1, std::min(env_fold, 256 / p.cw)) : std::max(1, std::min(2, 256 / p.cw));
    p.tmem_cols = pow2_cols((uint32_t)(p.tb * p.cw));
    const int base3 = base0(kFwdProd) + 8 * (kFwdProd + ring(nch * 4, p.tb, kFwdProd) + nch * 4 + 2);
    // Three CTAs per SM (configs[1] fwd 65.4 -> 62.9 us, dgrad 64.3 -> 62.2 us) when two stage
    // slots and the W ring fit a third of the SM and the registers allow it (the fused-epilogue
    // instance needs 84 registers: two CTAs).
    ctas = env_ctas0 == 3 && !p.ep.active() && 3 * p.tmem_cols <= 512 &&
                   base3 + nch * 2 * (int)p.b_bytes + 2 * (int)p.a_bytes <= kMaxSmem / 3 - 1024
               ? 3
               : 2;
    // two CTAs: the 8-warp plan when it gets at least 6 slots in half an SM, else the 4-warp one
    for (int w = ctas == 2 && !p.ep.active() ? env_npw : kFwdProd;; w = kFwdProd) {
      npw = w;
      samax = npw == kFwdProd ? kFwdProd : env_samax > 0 ? env_samax : npw;
      const int base = ctas == 3 ? base3 : base0(npw) + 8 * (samax + ring(nch * 4, p.tb, samax) + nch * 4 + 2);
      // per-CTA budget: a third of the SM, half of it (8-warp instance), or the 4-slot cap
      const int budget = ctas == 3 ? kMaxSmem / 3 - 1024 : samax > kFwdProd ? kMaxSmem / 2 - 1024 : kMaxSmem;
      p.sw = nch * 2;
      if (ctas == 2 && samax == kFwdProd &&
          base + p.sw * (int)p.b_bytes + kFwdProd * (int)p.a_bytes <= kMaxSmem / 2 - 1024 - 2 * nch * (int)p.b_bytes)
        p.sw = nch * 4;
      fixed = base + p.sw * (int)p.b_bytes;
      p.sa = std::min(samax, (budget - fixed) / (int)p.a_bytes);
      if (ctas == 2) p.sa -= p.sa % 2;
      if (npw == kFwdProd || p.sa >= 6) break;
    }
    if ((p.sa >= 2 && p.tmem_cols <= 512) || p.cw <= 16) break;
  }
  // one producer warp per slot measured best (fwd 68.6 us vs 73.8 with two slots per warp,
  // configs[1]): more warps issue the gathers faster than fewer warps with deeper queues
  p.np = std::min(npw, env_np > 0 ? std::min(env_np, p.sa) : p.sa);
  p.ga = p.sa % 2 == 0 ? 2 : 1;  // the W ring must hold >= ga units: sw / nch >= 2 >= ga
  // several channel chunks: one MMA step (and commit) per (unit, tile), ga = nch (a commit then
  // never covers steps of a later unit, so the W ring needs no more than two units)
  static const int env_grp = [] {
    const char* e = std::getenv("MK_FWD_GROUP");
    return e ? std::atoi(e) : 1;
  }();
  p.grp = env_grp && nch > 1 && p.sa >= nch ? 1 : 0;
  if (p.grp) p.ga = nch;
  p.ncb = ring(p.sw, p.tb, samax);
  if (p.sa < 2 || p.tmem_cols > 512)
    MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 conv: channel counts too large for the smem pipeline");
  const size_t wbytes = (size_t)nb.K * nch * p.b_img;
  uint8_t* wpack = (uint8_t*)dev_alloc(ctx->alloc, wbytes, s);
  if (!wpack) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "bf16 conv: weight pack allocation failed");
  {
    const int64_t chunks = (int64_t)nb.K * nch * c_y * (CH / 8);
    const int grid = (int)std::min<int64_t>(ceil_div(chunks, 256), 4 * ctx->num_sms);
    pdl_launch(k_pack_w, grid, 256, 0, s, (const __nv_bfloat16*)W, nb.K, c_out_w, c_in_w, trans ? 1 : 0, CH, wpack);
  }
  p.wpack = wpack;
  const int smem = fixed + p.sa * (int)p.a_bytes;
  // one CTA per tb tiles and column slice
  const dim3 grid((unsigned)ceil_div(p.ntiles, p.tb), (unsigned)ysplit);
  cudaError_t e;
  auto go = [&](auto kern, int nw) {
    set_smem_once(kern, smem);
    return pdl_launch(kern, grid, (nw + 6) * 32, smem, s, p);
  };
  const bool epi = p.ep.active();
  if (epi)
    e = CH == 64 ? go(k_conv_umma<64, true, 4>, 4) : CH == 32 ? go(k_conv_umma<32, true, 4>, 4) : go(k_conv_umma<16, true, 4>, 4);
  else if (npw == 8)
    e = CH == 64 ? go(k_conv_umma<64, false, 8>, 8) : CH == 32 ? go(k_conv_umma<32, false, 8>, 8) : go(k_conv_umma<16, false, 8>, 8);
  else
    e = CH == 64 ? go(k_conv_umma<64, false, 4>, 4) : CH == 32 ? go(k_conv_umma<32, false, 4>, 4) : go(k_conv_umma<16, false, 4>, 4);
  if (e == cudaSuccess) e = cudaGetLastError();
  dev_free(ctx->alloc, wpack, s);
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("bf16 conv launch: ") + cudaGetErrorString(e));
  return MK_OK;
}

mk_status launch_wgrad_bf16(mk_context* ctx, const mk_kmap* m, const void* g, int c_out, const void* x, int c_in,
                            float* dW, cudaStream_t s) {
  // K <= 63: the split-K plan is computed by the kernel from the device CSR offsets (no host
  // read-back, fully asynchronous); larger K: the host plan caps the segments per CTA.
  HostTimer ht("wgrad_bf16");
  const bool dev_plan = m->K <= kWgradMaxSegs;
  if (!dev_plan) {
    const mk_status pst = kmap_wplan(m, s);  // built once per map, on first use
    if (pst != MK_OK) return pst;
  }
  const int64_t te = (int64_t)c_out * c_in;
  WgradParams p;
  p.off32 = (int64_t)m->n_out * c_out < INT32_MAX && (int64_t)m->n_in * c_in < INT32_MAX;
  p.gsync = nullptr;  // (epoch throttle off unless the strided plan sets it up below)
  p.sync_b = 1;
  p.sync_s = 0;
  p.sync_emax = 0;
  p.g = (const __nv_bfloat16*)g;
  p.x = (const __nv_bfloat16*)x;
  p.in_idx = m->in_idx;
  p.out_idx = m->out_idx;
  p.segs = dev_plan ? nullptr : m->wseg;
  p.seg_begin = dev_plan ? nullptr : m->wseg_begin;
  p.ptr = m->ptr;
  p.jtab = nullptr;
  p.K = m->K;
  p.c_out = c_out;
  p.c_in = c_in;
  p.pwa = c_out % 64 == 0 ? 64 : c_out % 32 == 0 ? 32 : 16;
  p.pwb = c_in % 64 == 0 ? 64 : c_in % 32 == 0 ? 32 : 16;
  p.halves = c_out > 128 ? 2 : 1;
  p.mrows = c_out <= 64 ? 64 : 128;
  if (c_out > 256) MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 wgrad: C_out above 256");
  static const int env_apad = [] {  // development: MK_WGRAD_APAD=1 zeroed padding panels in every slot
    const char* e = std::getenv("MK_WGRAD_APAD");
    return e ? std::atoi(e) : 0;
  }();
  p.a_pad = env_apad;
  const uint32_t a_padded = (uint32_t)(p.halves * p.mrows) * kPairsPerStage * 2;  // M padded to 64 / 128 per half
  p.a_bytes = p.a_pad ? a_padded : (uint32_t)c_out * kPairsPerStage * 2;
  p.b_bytes = (uint32_t)c_in * kPairsPerStage * 2;
  p.slot_bytes = (p.a_bytes + p.b_bytes + 1023) & ~1023u;
  // producer warps: 4 (three CTAs per SM, default), 8 (two) or 16 (one).  configs[1] wgrad:
  // one CTA 104.5 us; two 85.9 us (82.3 with one commit per slot); three 78.1 us.
  static const int np_env = [] {  // 0: automatic
    const char* v = std::getenv("MK_WGRAD_NP");
    const int x = v ? std::atoi(v) : 0;
    return x == 16 || x == 8 || x == 4 ? x : 0;
  }();
  static const int env_ga = [] {  // development: stage slots released per commit
    const char* e = std::getenv("MK_WGRAD_GA");
    return e ? std::atoi(e) : 0;
  }();
  p.tmem_cols = pow2_cols((uint32_t)(p.halves * c_in));
  // Fewer, larger CTAs when the stage slots of wide channel counts (up to 2 x 32 KB per slot
  // at 256 x 256) or their TMEM accumulators do not fit three CTAs per SM: np = 8 (two CTAs)
  // or 16 (one CTA, up to 3 slots of 64 KB).
  // Automatic: three CTAs unless they get fewer than three stage slots each and two CTAs get
  // at least four (configs[4], C = 96: 2 vs 4 slots, wgrad 1797 -> 1633 us; configs[1], C = 64:
  // 4 vs 8 slots, 74 us with three CTAs vs 82 with two).
  int np = np_env > 0 ? np_env : 4, per_sm = 3, reserve = 0;
  auto plan = [&](int n) {
    per_sm = n == 16 ? 1 : n == 8 ? 2 : 3;
    const int budget = per_sm == 1 ? kMaxSmem : kMaxSmem / per_sm - 1024;
    // (+ room for the last slot's padding rows to read past it, when A has no padding panels)
    reserve = 1024 + 1024 + n * 4 * kPairsPerStage * 4 + (kMaxSegs + 2) * 4 + (int)sizeof(int4) * kMaxSegs + 128 +
              std::max(0, (int)a_padded - (int)p.slot_bytes);
    return std::min(n, (budget - reserve) / (int)p.slot_bytes);
  };
  for (;; np *= 2) {
    p.sa = plan(np);
    if ((p.sa >= 2 && per_sm * p.tmem_cols <= 512) || np >= 16) break;
  }
  if (np_env == 0 && np == 4 && p.sa < 3) {
    const int sa8 = plan(8);
    if (sa8 >= 4 && 2 * p.tmem_cols <= 512) {
      np = 8;
      p.sa = sa8;
    } else {
      p.sa = plan(4);
    }
  }
  if (p.sa >= 8) p.sa -= p.sa % 4;
  static const int env_nacc = [] {  // development: MK_WGRAD_NACC=1 one accumulator
    const char* e = std::getenv("MK_WGRAD_NACC");
    return e ? std::atoi(e) : 2;
  }();
  p.nacc = env_nacc == 2 && per_sm * pow2_cols((uint32_t)(2 * p.halves * c_in)) <= 512 ? 2 : 1;
  p.tmem_cols = pow2_cols((uint32_t)(p.nacc * p.halves * c_in));
  static const int env_wps = [] {  // development: MK_WGRAD_WPS=1 one producer warp per slot
    const char* e = std::getenv("MK_WGRAD_WPS");
    return e ? std::atoi(e) : 0;
  }();
  p.wps = 1;  // producer warps per slot: the spare warps when fewer slots than warps fit
  while (dev_plan && p.sa * p.wps * 2 <= np && p.wps < 4) p.wps *= 2;  // (the host-plan kernel: one)
  if (env_wps == 1) p.wps = 1;
  // stage slots released per commit: grouped at one CTA per SM, one per commit when other CTAs
  // share the SM (wgrad 85.9 -> 82.4 us, configs[1]; grouping at three CTAs: slower)
  p.ga = per_sm >= 2 ? 1 : p.sa % 4 == 0 ? 4 : p.sa % 2 == 0 ? 2 : 1;
  if (env_ga > 0 && p.sa % env_ga == 0) p.ga = env_ga;
  if (p.sa < 2 || p.tmem_cols > 512) MK_FAIL(MK_ERR_UNSUPPORTED, "bf16 wgrad: channel counts too large");
  const int smem = p.sa * (int)p.slot_bytes + reserve;
  float* part = nullptr;
  bool scratch = false;  // part is the context's scratch buffer (held until released below)
  static const int env_mode = [] {  // development: MK_WGRAD_PLAN=0 contiguous ranges, 2 strided
    const char* e = std::getenv("MK_WGRAD_PLAN");
    return e ? std::atoi(e) : 2;
  }();
  p.mode = dev_plan ? (m->K <= 32 && env_mode == 2 ? 2 : 0) : 1;
  if (dev_plan) {
    if (m->n_out > 0 && m->n_in > 0) {
      const int n_cta = ctx->num_sms * per_sm;
      // partial slots: one per CTA (strided plan) or per (CTA, offset) segment; then the
      // (first CTA, CTAs) table of the strided plan
      const int64_t slots = p.mode == 2 ? n_cta : n_cta + m->K;
      const size_t pbytes = ((sizeof(float) * slots * te + 255) & ~size_t(255));
      // epoch throttle of the strided plan (rounds per epoch, slack in epochs): counters for
      // an upper bound of the epochs (rounds <= chunks / spare CTAs + 2)
      static const int env_sync[3] = {
          [] { const char* e = std::getenv("MK_WGRAD_SYNC"); return e ? std::atoi(e) : 1; }(),
          [] { const char* e = std::getenv("MK_WGRAD_SYNCB"); return e ? std::max(1, std::atoi(e)) : 8; }(),
          [] { const char* e = std::getenv("MK_WGRAD_SYNCS"); return e ? std::max(0, std::atoi(e)) : 2; }()};
      const int64_t spare = (int64_t)n_cta - m->K;
      int emax = 0;
      // only when the gathered features exceed L2 (configs[4]: cold-L2 DRAM reads 4.8 -> 2.5 GB
      // per launch, time unchanged; on L2-resident maps it costs a few us)
      const bool big = ((int64_t)m->n_in * c_in + (int64_t)m->n_out * c_out) * 2 > (int64_t)ctx->l2_bytes / 2;
      if (p.mode == 2 && env_sync[0] && spare > 0 && (big || env_sync[0] == 2)) {
        const int64_t chunks = (int64_t)m->K * m->n_out / kPairsPerStage + m->K;
        emax = (int)std::min<int64_t>(1 << 20, (chunks / spare + 2) / env_sync[1] + 2);
      }
      const size_t jbytes = ((sizeof(int32_t) * 2 * m->K + 255) & ~size_t(255));
      ht.mark("plan");
      part = (float*)scratch_acquire(ctx, pbytes + jbytes + sizeof(unsigned) * emax, s);
      ht.mark("alloc");
      if (!part) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "bf16 wgrad: workspace allocation failed");
      scratch = true;
      p.part = part;
      p.jtab = (int32_t*)((uint8_t*)part + pbytes);
      p.gsync = emax > 0 ? (unsigned*)((uint8_t*)part + pbytes + jbytes) : nullptr;
      p.sync_b = env_sync[1];
      p.sync_s = env_sync[2];
      p.sync_emax = emax;
      if (emax > 0) {
        const cudaError_t z = cudaMemsetAsync(p.gsync, 0, sizeof(unsigned) * emax, s);
        if (z != cudaSuccess) {
          scratch_release(ctx, s);
          MK_FAIL(MK_ERR_CUDA, "bf16 wgrad: memset failed");
        }
      }
      auto go = [&](auto kern, int threads) {
        set_smem_once(kern, smem);
        pdl_launch(kern, n_cta, threads, smem, s, p);
      };
      auto per3 = [](int c) { const int c8 = c / 8; return c8 > 0 && 32 % c8 != 0 && 96 % c8 == 0 && (96 / c8) % 8 == 0; };
      const bool p3 = p.off32 && (per3(c_out) || per3(c_in));
      if (np == 16) p3 ? go(k_wgrad_umma<16, true>, (16 + kEpiWarps + 1) * 32) : go(k_wgrad_umma<16, false>, (16 + kEpiWarps + 1) * 32);
      else if (np == 8) p3 ? go(k_wgrad_umma<8, true>, (8 + kEpiWarps + 1) * 32) : go(k_wgrad_umma<8, false>, (8 + kEpiWarps + 1) * 32);
      else p3 ? go(k_wgrad_umma<4, true>, (4 + kEpiWarps + 1) * 32) : go(k_wgrad_umma<4, false>, (4 + kEpiWarps + 1) * 32);
      ht.mark("launch");
      dim3 rg((unsigned)ceil_div(te, 256), (unsigned)m->K);
      if (p.mode == 2)
        pdl_launch(k_reduce_partials_jtab, rg, 256, 0, s, (const int32_t*)p.jtab, m->K, (const float*)part, te, dW);
      else
        pdl_launch(k_reduce_partials_dev, rg, 256, 0, s, (const int64_t*)m->ptr, n_cta, (const float*)part, te, dW);
    } else {
      const cudaError_t z = cudaMemsetAsync(dW, 0, sizeof(float) * m->K * te, s);
      if (z != cudaSuccess) MK_FAIL(MK_ERR_CUDA, "bf16 wgrad: memset failed");
    }
  } else {
    if (m->n_wslots > 0) {
      part = (float*)dev_alloc(ctx->alloc, sizeof(float) * m->n_wslots * te, s);
      if (!part) MK_FAIL(MK_ERR_OUT_OF_MEMORY, "bf16 wgrad: workspace allocation failed");
      p.part = part;
      set_smem_once(k_wgrad_umma<16, false>, smem);
      pdl_launch(k_wgrad_umma<16, false>, m->n_wcta, (16 + kEpiWarps + 1) * 32, smem, s, p);
    }
    dim3 rg((unsigned)ceil_div(te, 256), (unsigned)m->K);
    k_reduce_partials<<<rg, 256, 0, s>>>(m->wslot_begin, part, te, dW);
    g_launches++;
  }
  ht.mark("reduce");
  cudaError_t e = cudaGetLastError();
  if (scratch) scratch_release(ctx, s);
  else if (part) dev_free(ctx->alloc, part, s);
  ht.mark("free");
  if (e != cudaSuccess) MK_FAIL(MK_ERR_CUDA, std::string("bf16 wgrad launch: ") + cudaGetErrorString(e));
  return MK_OK;
}

}  // namespace mk
