// context.cu — device binding, allocator plumbing and the thread-local error channel.
#include <cstring>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "mk_internal.cuh"

namespace mk {

namespace {
thread_local std::string t_msg;
thread_local int64_t t_row = -1;
}  // namespace

std::atomic<int64_t> g_launches{0};

void set_error(mk_status s, const std::string& msg, int64_t row) {
  (void)s;
  t_msg = msg;
  t_row = row;
}
void clear_error() {
  t_msg.clear();
  t_row = -1;
}

void* dev_alloc(const Alloc& a, size_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  if (a.alloc) return a.alloc(bytes, s, a.user);
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void* scratch_acquire(mk_context* ctx, size_t bytes, cudaStream_t s) {
  ctx->scratch_mu.lock();
  if (ctx->scratch_cap < bytes) {
    if (ctx->scratch) dev_free(ctx->alloc, ctx->scratch, ctx->scratch_stream ? ctx->scratch_stream : s);
    const size_t cap = bytes + bytes / 4;
    ctx->scratch = dev_alloc(ctx->alloc, cap, s);
    ctx->scratch_cap = ctx->scratch ? cap : 0;
    ctx->scratch_stream = s;
    if (!ctx->scratch) {
      ctx->scratch_mu.unlock();
      return nullptr;
    }
  } else if (ctx->scratch_stream && ctx->scratch_stream != s) {
    cudaStreamWaitEvent(s, ctx->scratch_ev, 0);  // the previous user's kernels are done with it
  }
  return ctx->scratch;
}

void scratch_release(mk_context* ctx, cudaStream_t s) {
  if (!ctx->scratch_ev) cudaEventCreateWithFlags(&ctx->scratch_ev, cudaEventDisableTiming);
  cudaEventRecord(ctx->scratch_ev, s);
  ctx->scratch_stream = s;
  ctx->scratch_mu.unlock();
}

void dev_free(const Alloc& a, void* p, cudaStream_t s) {
  if (!p) return;
  if (a.free_fn) {
    a.free_fn(p, s, a.user);
    return;
  }
  cudaFreeAsync(p, s);
}

// Thread-local pinned staging buffer for the few small host<->device copies of a call:
// pageable cudaMemcpyAsync is synchronous (and slow); pinned copies are true async DMA.
namespace {
struct PinnedStage {
  void* p = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;
  ~PinnedStage() {
    if (p) cudaFreeHost(p);
    if (ev) cudaEventDestroy(ev);
  }
};
thread_local PinnedStage t_pin;
}  // namespace

void* pinned_stage(size_t bytes) {
  if (t_pin.pending) {  // a previous async copy may still read / write the buffer
    cudaEventSynchronize(t_pin.ev);
    t_pin.pending = false;
  }
  if (!t_pin.ev && cudaEventCreateWithFlags(&t_pin.ev, cudaEventDisableTiming) != cudaSuccess) return nullptr;
  if (bytes > t_pin.cap) {
    if (t_pin.p) cudaFreeHost(t_pin.p);
    t_pin.p = nullptr;
    t_pin.cap = 0;
    size_t c = 4096;
    while (c < bytes) c <<= 1;
    if (cudaMallocHost(&t_pin.p, c) != cudaSuccess) return nullptr;
    t_pin.cap = c;
  }
  return t_pin.p;
}

void pinned_in_flight(cudaStream_t s) {
  if (t_pin.ev && cudaEventRecord(t_pin.ev, s) == cudaSuccess) t_pin.pending = true;
}

namespace {
struct MailboxHolder {
  Mailbox* mb = nullptr;
  unsigned long long seq = 0;
  ~MailboxHolder() {
    if (mb) cudaFreeHost(mb);
  }
};
thread_local MailboxHolder t_mb;
}  // namespace

Mailbox* mailbox(unsigned long long* next_seq) {
  if (!t_mb.mb) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, sizeof(Mailbox), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
    t_mb.mb = (Mailbox*)p;
    std::memset(p, 0, sizeof(Mailbox));
  }
  *next_seq = ++t_mb.seq;
  return t_mb.mb;
}

Mailbox* mailbox_ring_slot(mk_context* ctx, unsigned long long* seq) {
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!ctx->mb_ring) {
      void* p = nullptr;
      if (cudaHostAlloc(&p, sizeof(Mailbox) * mk_context::kMbSlots, cudaHostAllocMapped | cudaHostAllocPortable) !=
          cudaSuccess)
        return nullptr;
      std::memset(p, 0, sizeof(Mailbox) * mk_context::kMbSlots);
      ctx->mb_ring = (Mailbox*)p;
    }
  }
  *seq = ctx->mb_seq.fetch_add(1) + 1;  // never 0 (the slots start zeroed)
  return ctx->mb_ring + (*seq % mk_context::kMbSlots);
}

cudaError_t mailbox_wait(const Mailbox* mb, unsigned long long seq, cudaStream_t s) {
  const volatile unsigned long long* v = &mb->seq;
  for (uint32_t it = 1;; ++it) {
    if (*v == seq) {
      std::atomic_thread_fence(std::memory_order_acquire);
      return cudaSuccess;
    }
    if ((it & 255u) == 0) {  // every ~few us: a failed or finished stream ends the wait
      const cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess) {
        if (*v == seq) continue;
        return cudaErrorUnknown;  // the stream drained without posting
      }
      if (e != cudaErrorNotReady) return e;
    }
  }
}

double HostTimer::now() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("MK_NO_PDL");
    return !(v && v[0] && v[0] != '0');
  }();
  return on;
}

HostTimer::HostTimer(const char* nm) : name(nm) {
  static const bool enabled = std::getenv("MK_HOST_TIMING") != nullptr;
  on = enabled;
  mark("start");
}
HostTimer::~HostTimer() {
  if (!on || n == 0) return;
  mark("end");
  std::fprintf(stderr, "[mk host] %s:", name);
  for (int i = 1; i < n; ++i) std::fprintf(stderr, " %s=%.1f", lab[i], t[i] - t[0]);
  std::fprintf(stderr, "\n");
}

uint32_t next_pow2(uint64_t v) {
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return (uint32_t)p;
}

}  // namespace mk

extern "C" {

mk_status mk_context_create(int device, mk_alloc_fn alloc, mk_free_fn free_fn, void* user,
                            mk_context** out) {
  mk::clear_error();
  if (!out) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_context_create: out is NULL");
  if ((alloc == nullptr) != (free_fn == nullptr))
    MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_context_create: alloc and free must both be set or both NULL");
  int count = 0;
  MK_CUDA_TRY(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_context_create: no such device");
  cudaDeviceProp prop;
  MK_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    MK_FAIL(MK_ERR_UNSUPPORTED, "mk_context_create: libmk is built for sm_100a (B200) only");
  MK_CUDA_TRY(cudaSetDevice(device));
  // Keep freed blocks in the stream-ordered pool (no release to the OS on every sync).
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // Reserve pool memory up front (allocate + free once; the threshold keeps it mapped): the
    // per-call handles and temporaries of a step (tables, maps, partials: ~2-3 GB at configs[4])
    // then never make the pool map new memory inside a step, which stalled the host for
    // 0.3-66 ms when sizes and lifetimes fragmented it.  MK_POOL_RESERVE_MB overrides (0: off).
    const char* e = std::getenv("MK_POOL_RESERVE_MB");
    const size_t mb = e ? (size_t)std::atoll(e) : (size_t)8192;
    if (mb > 0 && (size_t)prop.totalGlobalMem > 4 * (mb << 20)) {
      void* p = nullptr;
      if (cudaMallocAsync(&p, mb << 20, 0) == cudaSuccess) {
        cudaFreeAsync(p, 0);
        cudaStreamSynchronize(0);
      } else {
        cudaGetLastError();
      }
    }
  }
  mk_context* c = new mk_context();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->l2_bytes = prop.l2CacheSize;
  c->alloc.alloc = alloc;
  c->alloc.free_fn = free_fn;
  c->alloc.user = user;
  if (cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    MK_FAIL(MK_ERR_CUDA, "mk_context_create: stream creation failed");
  }
  if (cudaMalloc(&c->d_bar, sizeof(unsigned) * 2 * mk_context::kBarSlots) != cudaSuccess ||
      cudaMemset(c->d_bar, 0, sizeof(unsigned) * 2 * mk_context::kBarSlots) != cudaSuccess) {
    c->d_bar = nullptr;  // the sort falls back to its three-kernel passes
    cudaGetLastError();
  }
  *out = c;
  return MK_OK;
}

void mk_context_destroy(mk_context* ctx) {
  if (!ctx) return;
  for (auto& r : ctx->region_dev) cudaFree(r.second);
  if (ctx->d_bar) cudaFree(ctx->d_bar);
  if (ctx->mb_ring) cudaFreeHost(ctx->mb_ring);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->scratch) {
    cudaDeviceSynchronize();
    mk::dev_free(ctx->alloc, ctx->scratch, nullptr);
  }
  if (ctx->scratch_ev) cudaEventDestroy(ctx->scratch_ev);
  delete ctx;
}

const char* mk_last_error_message(void) { return mk::t_msg.c_str(); }
int64_t mk_last_error_row(void) { return mk::t_row; }
int64_t mk_kernel_launch_count(void) { return mk::g_launches.load(); }

}  // extern "C"
