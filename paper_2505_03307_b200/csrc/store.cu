// a1: the Pauli-term store in HBM, plus library-level plumbing (errors, device info,
// CUDA-event instrumentation).  Replaces SimpleGenerator / GeneratorSet / init_z
// (reference stabilizer.py:83-109, 157-174).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <thread>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#include <unordered_map>

#include "qx_internal.cuh"

// ----------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------
static thread_local char g_error[512] = "";

int qx_fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_error, sizeof(g_error), fmt, ap);
  va_end(ap);
  return status;
}

extern "C" const char* qx_last_error(void) { return g_error; }
extern "C" int qx_abi_version(void) { return QX_ABI_VERSION; }

extern "C" int qx_device_count(int* count) {
  QX_REQUIRE(count != nullptr, "count is NULL");
  QX_CUDA(cudaGetDeviceCount(count));
  return QX_OK;
}

extern "C" int qx_device_info(int device, char* name, int name_cap, int* sm_count,
                              int* cc_major, int* cc_minor, int64_t* total_bytes,
                              int64_t* free_bytes) {
  cudaDeviceProp prop;
  QX_CUDA(cudaGetDeviceProperties(&prop, device));
  if (name && name_cap > 0) {
    strncpy(name, prop.name, name_cap - 1);
    name[name_cap - 1] = 0;
  }
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (total_bytes || free_bytes) {
    size_t f = 0, t = 0;
    QX_CUDA(cudaSetDevice(device));
    QX_CUDA(cudaMemGetInfo(&f, &t));
    if (total_bytes) *total_bytes = (int64_t)t;
    if (free_bytes) *free_bytes = (int64_t)f;
  }
  return QX_OK;
}

extern "C" int qx_host_alloc(int64_t bytes, void** out) {
  QX_REQUIRE(out != nullptr && bytes >= 0, "bad argument");
  *out = nullptr;
  cudaError_t e = cudaMallocHost(out, (size_t)std::max<int64_t>(bytes, 8));
  if (e != cudaSuccess)
    return qx_fail(QX_ERR_RESOURCE, "cannot page-lock %.2f GB of host memory: %s", bytes / 1e9,
                   cudaGetErrorString(e));
  return QX_OK;
}

extern "C" int qx_host_free(void* ptr) {
  if (ptr) QX_CUDA(cudaFreeHost(ptr));
  return QX_OK;
}

// ----------------------------------------------------------------------------
// instrumentation: CUDA events around each kernel class, resolved lazily
// ----------------------------------------------------------------------------
namespace {
struct Pending {
  cudaEvent_t a, b;
};
struct ClassStats {
  int64_t launches = 0;
  double ms = 0.0;
  double bytes = 0.0;
  std::vector<Pending> pending;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
ClassStats g_prof[QX_K_CLASSES];
std::vector<cudaEvent_t> g_event_pool;
std::atomic<int64_t> g_launches{0};

cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void resolve(ClassStats& c) {
  for (Pending& p : c.pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) c.ms += ms;
    g_event_pool.push_back(p.a);
    g_event_pool.push_back(p.b);
  }
  c.pending.clear();
}
}  // namespace

void qx_count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
bool qx_profile_on() { return g_prof_on; }

QxProfileScope::QxProfileScope(int kernel_class, cudaStream_t st, double alg_bytes, int launches)
    : cls(kernel_class), stream(st), start(nullptr), stop(nullptr), active(false) {
  qx_count_launches(launches);
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  active = true;
  start = take_event();
  stop = take_event();
  g_prof[cls].launches += launches;
  g_prof[cls].bytes += alg_bytes;
  cudaEventRecord(start, stream);
}

QxProfileScope::~QxProfileScope() {
  if (!active) return;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  cudaEventRecord(stop, stream);
  g_prof[cls].pending.push_back({start, stop});
  if (g_prof[cls].pending.size() > 4096) resolve(g_prof[cls]);
}

extern "C" int qx_profile_enable(int on) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  g_prof_on = on != 0;
  return QX_OK;
}

extern "C" int qx_profile_reset(void) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (ClassStats& c : g_prof) {
    resolve(c);
    c.launches = 0;
    c.ms = 0.0;
    c.bytes = 0.0;
  }
  return QX_OK;
}

extern "C" int qx_profile_read(int kernel_class, int64_t* launches, double* total_ms,
                               double* alg_bytes) {
  QX_REQUIRE(kernel_class >= 0 && kernel_class < QX_K_CLASSES, "bad kernel class %d", kernel_class);
  std::lock_guard<std::mutex> lock(g_prof_mu);
  ClassStats& c = g_prof[kernel_class];
  resolve(c);
  if (launches) *launches = c.launches;
  if (total_ms) *total_ms = c.ms;
  if (alg_bytes) *alg_bytes = c.bytes;
  return QX_OK;
}

extern "C" int qx_launch_count(int64_t* launches) {
  QX_REQUIRE(launches != nullptr, "launches is NULL");
  *launches = g_launches.load();
  return QX_OK;
}

// ----------------------------------------------------------------------------
// device memory: caching allocator
// ----------------------------------------------------------------------------
// A store is created per circuit run and owns multi-GB buffers; cudaMalloc/cudaFree (and
// the driver's pool when block sizes vary from run to run) cost tens to hundreds of
// milliseconds per run, more than the kernels.  Freed blocks are therefore kept in a
// per-device free list and handed out again for any request they fit within 2x.  Reuse is
// stream-ordered: a block freed on stream S may still be in use by kernels queued on S, so
// it is only handed to the same stream without a wait; any other stream synchronises S first.
namespace {
struct DevBlock {
  void* ptr;
  size_t bytes;
  int device;
  cudaStream_t stream;   // stream of the last user
};
std::mutex g_alloc_mu;
std::unordered_map<void*, DevBlock> g_live;
std::multimap<size_t, DevBlock> g_free[64];

size_t round_block(size_t bytes) {
  const size_t unit = bytes >= (1u << 20) ? (2u << 20) : 512;   // 2 MiB granules for big blocks
  return (bytes + unit - 1) / unit * unit;
}

void release_cached(int device) {
  for (auto& kv : g_free[device]) {
    cudaStreamSynchronize(kv.second.stream);
    cudaFree(kv.second.ptr);
  }
  g_free[device].clear();
}
}  // namespace

int qx_dev_alloc(void** out, int64_t bytes, cudaStream_t stream, int device) {
  *out = nullptr;
  if (device < 0 || device >= 64) return qx_fail(QX_ERR_INVALID, "bad device %d", device);
  const size_t want = round_block((size_t)std::max<int64_t>(bytes, 256));
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  // a cached block of a fitting size whose last user is this stream, or a stream with nothing
  // pending (waiting for a busy stream here would serialise stores that are meant to overlap,
  // e.g. one range's download against the next range's kernels)
  const size_t limit = 2 * want + (64u << 20);
  auto fallback = g_free[device].end();
  for (auto it = g_free[device].lower_bound(want); it != g_free[device].end() && it->first <= limit; ++it) {
    const bool ready = it->second.stream == stream || cudaStreamQuery(it->second.stream) == cudaSuccess;
    if (!ready) {
      cudaGetLastError();                      // cudaErrorNotReady is not an error
      if (fallback == g_free[device].end()) fallback = it;
      continue;
    }
    DevBlock blk = it->second;
    g_free[device].erase(it);
    blk.stream = stream;
    g_live[blk.ptr] = blk;
    *out = blk.ptr;
    return QX_OK;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, want);
  if (e != cudaSuccess && fallback != g_free[device].end()) {   // HBM is tight: wait for the busy block
    cudaGetLastError();
    DevBlock blk = fallback->second;
    g_free[device].erase(fallback);
    cudaStreamSynchronize(blk.stream);
    blk.stream = stream;
    g_live[blk.ptr] = blk;
    *out = blk.ptr;
    return QX_OK;
  }
  if (e != cudaSuccess) {            // give the cache back to the driver and retry once
    cudaGetLastError();
    release_cached(device);
    e = cudaMalloc(&p, want);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    return qx_fail(QX_ERR_RESOURCE, "cannot allocate %.2f GB of HBM on device %d (%.1f GB free): %s",
                   want / 1e9, device, free_b / 1e9, cudaGetErrorString(e));
  }
  g_live[p] = DevBlock{p, want, device, stream};
  *out = p;
  return QX_OK;
}

void qx_dev_free(void* ptr, cudaStream_t stream) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  auto it = g_live.find(ptr);
  if (it == g_live.end()) {
    cudaFree(ptr);
    return;
  }
  DevBlock blk = it->second;
  g_live.erase(it);
  blk.stream = stream;
  g_free[blk.device].emplace(blk.bytes, blk);
}

// A stream is about to be destroyed: wait for it and re-home its cached blocks on the default
// stream so that nobody synchronises a dead handle later.
void qx_dev_forget_stream(cudaStream_t stream) {
  cudaStreamSynchronize(stream);
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  for (int d = 0; d < 64; ++d)
    for (auto& kv : g_free[d])
      if (kv.second.stream == stream) kv.second.stream = 0;
  for (auto& kv : g_live)
    if (kv.second.stream == stream) kv.second.stream = 0;
}

// small page-locked staging blocks (offset mirrors): same idea, cudaMallocHost is ~0.3 ms a call
namespace {
std::multimap<size_t, void*> g_pinned_free;
std::unordered_map<void*, size_t> g_pinned_live;
}  // namespace

int qx_pinned_alloc(void** out, int64_t bytes) {
  const size_t want = ((size_t)std::max<int64_t>(bytes, 64) + 4095) / 4096 * 4096;
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  auto it = g_pinned_free.lower_bound(want);
  if (it != g_pinned_free.end() && it->first <= 4 * want) {
    *out = it->second;
    g_pinned_live[*out] = it->first;
    g_pinned_free.erase(it);
    return QX_OK;
  }
  QX_CUDA(cudaMallocHost(out, want));
  g_pinned_live[*out] = want;
  return QX_OK;
}

void qx_pinned_free(void* ptr) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  auto it = g_pinned_live.find(ptr);
  if (it == g_pinned_live.end()) {
    cudaFreeHost(ptr);
    return;
  }
  g_pinned_free.emplace(it->second, ptr);
  g_pinned_live.erase(it);
}

extern "C" int qx_trim(void) {
  std::lock_guard<std::mutex> lock(g_alloc_mu);
  for (int d = 0; d < 64; ++d)
    if (!g_free[d].empty()) {
      cudaSetDevice(d);
      release_cached(d);
    }
  return QX_OK;
}

// ----------------------------------------------------------------------------
// store lifetime and capacity
// ----------------------------------------------------------------------------
static int alloc_buffers(qx_store* s, int64_t cap, u64** keys, double** lam) {
  for (int b = 0; b < 2; ++b) {
    QX_TRY(qx_dev_alloc_t(&keys[b], cap, s->stream, s->device));
    QX_TRY(qx_dev_alloc_t(&lam[b], cap, s->stream, s->device));
  }
  return QX_OK;
}

extern "C" int qx_store_create(int device, int n_qubits, int n_segments, int64_t capacity_terms,
                               qx_store** out) {
  QX_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  if (n_qubits < 1) return qx_fail(QX_ERR_INVALID, "qubit count must be positive, got %d", n_qubits);
  if (n_qubits > QX_MAX_QUBITS_WIDE)
    return qx_fail(QX_ERR_UNSUPPORTED, "n_qubits=%d: keys hold at most %d words (n <= %d)", n_qubits,
                   QX_MAX_WORDS, QX_MAX_QUBITS_WIDE);
  QX_REQUIRE(n_segments >= 1 && n_segments <= (1 << 20), "bad segment count %d", n_segments);
  qx_store* s = new qx_store();
  {
    const int st0 = qx_arena_init(s, device, n_qubits, (int64_t)n_segments + 16);
    if (st0 != QX_OK) {
      delete s;
      return st0;
    }
  }
  s->n_seg = n_segments;
  s->n_words = n_qubits <= QX_MAX_QUBITS ? 1 : (2 * n_qubits + 63) / 64;
  s->cap = std::max<int64_t>(capacity_terms, std::max<int64_t>(4096, 2 * (int64_t)n_segments));
  int st = alloc_buffers(s, s->cap, s->keys, s->lam);
  for (int b = 0; b < 2 && st == QX_OK && s->n_words > 1; ++b)
    st = qx_dev_alloc_t(&s->hi[b], s->cap * (s->n_words - 1), s->stream, s->device);
  if (st == QX_OK) {
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < 2 && st == QX_OK; ++b)
      st = qx_dev_alloc_t(&s->seg[b], (int64_t)n_segments + 1, s->stream, s->device);
    if (st == QX_OK)
      st = qx_pinned_alloc(reinterpret_cast<void**>(&s->h_seg), 8 * ((int64_t)n_segments + 1));
    if (st == QX_OK && e == cudaSuccess)
      e = cudaMemsetAsync(s->seg[0], 0, sizeof(int64_t) * (size_t)(n_segments + 1), s->stream);
    if (st == QX_OK && e != cudaSuccess) st = qx_fail(QX_ERR_CUDA, "store allocation failed: %s", cudaGetErrorString(e));
  }
  if (st != QX_OK) {
    qx_store_destroy(s);
    return st;
  }
  memset(s->h_seg, 0, sizeof(int64_t) * (size_t)(n_segments + 1));
  s->exact = true;
  *out = s;
  return QX_OK;
}

namespace {
void join_workers(qx_store* s);      // host threads of a narrow download (below)

// CUDA events of the phase timers are kept per device across stores: creating one costs more than
// recording it, and a store lives for one circuit run
constexpr int kEventDevices = 64;
std::mutex g_event_mu;
std::vector<cudaEvent_t> g_timer_events[kEventDevices];
bool event_pool_take(int device, cudaEvent_t* e) {
  if (device < 0 || device >= kEventDevices) return false;
  std::lock_guard<std::mutex> lock(g_event_mu);
  if (g_timer_events[device].empty()) return false;
  *e = g_timer_events[device].back();
  g_timer_events[device].pop_back();
  return true;
}
void event_pool_put(int device, const std::vector<cudaEvent_t>& events) {
  if (device < 0 || device >= kEventDevices) {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    return;
  }
  std::lock_guard<std::mutex> lock(g_event_mu);
  for (cudaEvent_t e : events) {
    if (g_timer_events[device].size() < 4096) g_timer_events[device].push_back(e);
    else cudaEventDestroy(e);
  }
}
}

extern "C" int qx_store_destroy(qx_store* s) {
  if (!s) return QX_OK;
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  join_workers(s);
  for (int b = 0; b < 2; ++b) {
    qx_dev_free(s->keys[b], s->stream);
    qx_dev_free(s->lam[b], s->stream);
    qx_dev_free(s->seg[b], s->stream);
    qx_dev_free(s->hi[b], s->stream);
  }
  qx_pinned_free(s->h_seg);
  qx_arena_release(s);
  if (s->events) {
    event_pool_put(s->device, *s->events);
    delete s->events;
  }
  if (s->own_stream) {
    // blocks handed back above carry this stream as their last user: forget it before it dies
    qx_dev_forget_stream(s->stream);
    cudaStreamDestroy(s->stream);
  }
  delete s;
  return QX_OK;
}

extern "C" int qx_store_slice(qx_store* src, int32_t seg_lo, int32_t seg_hi, int64_t capacity_terms,
                              qx_store** out) {
  QX_REQUIRE(src && out, "NULL argument");
  QX_REQUIRE(seg_lo >= 0 && seg_lo < seg_hi && seg_hi <= src->n_seg, "bad segment range [%d, %d) of %d",
             seg_lo, seg_hi, src->n_seg);
  QX_NARROW_ONLY(src, "qx_store_slice");
  *out = nullptr;
  QX_CUDA(cudaSetDevice(src->device));
  if (!src->exact) QX_TRY(qx_store_refresh(src));
  QX_CUDA(cudaStreamSynchronize(src->stream));          // the source terms are final
  const int64_t first = src->h_seg[seg_lo], count = src->h_seg[seg_hi] - first;
  qx_store* s = nullptr;
  QX_TRY(qx_store_create(src->device, src->n_qubits, seg_hi - seg_lo, std::max(capacity_terms, count), &s));
  cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    s->stream = 0;
    qx_store_destroy(s);
    return qx_fail(QX_ERR_CUDA, "cudaStreamCreate failed: %s", cudaGetErrorString(e));
  }
  s->own_stream = true;
  for (int g = 0; g <= s->n_seg; ++g) s->h_seg[g] = src->h_seg[seg_lo + g] - first;
  const int c = s->cur;
  if (count > 0) {
    e = cudaMemcpyAsync(s->keys[c], src->keys[src->cur] + first, sizeof(u64) * (size_t)count,
                        cudaMemcpyDeviceToDevice, s->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(s->lam[c], src->lam[src->cur] + first, sizeof(double) * (size_t)count,
                          cudaMemcpyDeviceToDevice, s->stream);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(s->seg[c], s->h_seg, sizeof(int64_t) * (size_t)(s->n_seg + 1), cudaMemcpyHostToDevice,
                        s->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);   // src may change once we return
  if (e != cudaSuccess) {
    qx_store_destroy(s);
    return qx_fail(QX_ERR_CUDA, "slice copy failed: %s", cudaGetErrorString(e));
  }
  s->exact = true;
  s->ub_total = count;
  s->ub_seg = 0;
  for (int g = 0; g < s->n_seg; ++g) s->ub_seg = std::max(s->ub_seg, s->h_seg[g + 1] - s->h_seg[g]);
  *out = s;
  return QX_OK;
}

extern "C" int qx_store_set_stream(qx_store* s, void* cuda_stream) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  QX_CUDA(cudaStreamSynchronize(s->stream));
  s->stream = (cudaStream_t)cuda_stream;
  return QX_OK;
}

// Make room for `terms` per buffer.  keep_live copies the live terms across.
int qx_store_reserve(qx_store* s, int64_t terms, bool keep_live) {
  if (terms <= s->cap) return QX_OK;
  QX_CUDA(cudaSetDevice(s->device));
  if (keep_live && !s->exact) QX_TRY(qx_store_refresh(s));
  const int64_t live = keep_live ? s->h_seg[s->n_seg] : 0;
  const int64_t old_cap = s->cap;
  const int old_cur = s->cur;
  // One buffer pair at a time so the peak is old + new, not 2x new.  Try generous growth
  // first, fall back to the exact need when HBM is tight.
  const int dead = s->cur ^ 1, old = s->cur;
  int64_t want = std::max<int64_t>(terms + terms / 8, s->cap * 2);
  qx_dev_free(s->keys[dead], s->stream);
  qx_dev_free(s->lam[dead], s->stream);
  s->keys[dead] = nullptr;
  s->lam[dead] = nullptr;
  int st = qx_dev_alloc_t(&s->keys[dead], want, s->stream, s->device);
  if (st == QX_OK) st = qx_dev_alloc_t(&s->lam[dead], want, s->stream, s->device);
  if (st != QX_OK && want > terms) {
    qx_dev_free(s->keys[dead], s->stream);
    qx_dev_free(s->lam[dead], s->stream);
    s->keys[dead] = nullptr;
    s->lam[dead] = nullptr;
    want = terms;
    st = qx_dev_alloc_t(&s->keys[dead], want, s->stream, s->device);
    if (st == QX_OK) st = qx_dev_alloc_t(&s->lam[dead], want, s->stream, s->device);
  }
  if (st != QX_OK) {
    s->cap = 0;      // the store is unusable now; the caller surfaces ResourceLimitError
    return qx_fail(QX_ERR_RESOURCE, "term store would need %.1f GB of HBM for %lld terms on device %d",
                   32.0 * (double)terms / 1e9, (long long)terms, s->device);
  }
  if (live > 0) {
    QX_CUDA(cudaMemcpyAsync(s->keys[dead], s->keys[old], sizeof(u64) * (size_t)live,
                            cudaMemcpyDeviceToDevice, s->stream));
    QX_CUDA(cudaMemcpyAsync(s->lam[dead], s->lam[old], sizeof(double) * (size_t)live,
                            cudaMemcpyDeviceToDevice, s->stream));
  }
  QX_CUDA(cudaMemcpyAsync(s->seg[dead], s->seg[old], sizeof(int64_t) * (size_t)(s->n_seg + 1),
                          cudaMemcpyDeviceToDevice, s->stream));
  qx_dev_free(s->keys[old], s->stream);
  qx_dev_free(s->lam[old], s->stream);
  s->keys[old] = nullptr;
  s->lam[old] = nullptr;
  st = qx_dev_alloc_t(&s->keys[old], want, s->stream, s->device);
  if (st == QX_OK) st = qx_dev_alloc_t(&s->lam[old], want, s->stream, s->device);
  if (st != QX_OK) {
    s->cap = 0;
    return qx_fail(QX_ERR_RESOURCE, "term store would need %.1f GB of HBM for %lld terms on device %d",
                   32.0 * (double)want / 1e9, (long long)want, s->device);
  }
  s->cur = dead;
  s->cap = want;
  if (s->n_words > 1) {
    // the upper words: new planes of the new capacity, live part of every plane copied across
    u64* fresh[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b) QX_TRY(qx_dev_alloc_t(&fresh[b], want * (s->n_words - 1), s->stream, s->device));
    for (int w = 1; w < s->n_words && live > 0; ++w)
      QX_CUDA(cudaMemcpyAsync(fresh[s->cur] + (size_t)(w - 1) * (size_t)want,
                              s->hi[old_cur] + (size_t)(w - 1) * (size_t)old_cap, sizeof(u64) * (size_t)live,
                              cudaMemcpyDeviceToDevice, s->stream));
    for (int b = 0; b < 2; ++b) {
      qx_dev_free(s->hi[b], s->stream);
      s->hi[b] = fresh[b];
    }
  }
  return QX_OK;
}

int qx_arena_init(QxArena* a, int device, int n_qubits, int64_t pinned_words) {
  int count = 0;
  QX_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    return qx_fail(QX_ERR_CUDA, "CUDA device %d not available (%d visible)", device, count);
  QX_CUDA(cudaSetDevice(device));
  static int cached_sm[64] = {0}, cached_major[64] = {0};
  if (device < 64 && cached_sm[device] == 0) {      // cudaGetDeviceProperties costs ~1 ms
    int sm = 0, major = 0;
    QX_CUDA(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, device));
    QX_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    cached_sm[device] = sm;
    cached_major[device] = major;
  }
  if (cached_major[device] < 10)
    return qx_fail(QX_ERR_CUDA, "device %d is sm_%dx; this library is built for sm_100a only",
                   device, cached_major[device]);
  a->device = device;
  a->n_qubits = n_qubits;
  a->sm_count = cached_sm[device];
  a->h_pinned_words = pinned_words;
  QX_TRY(qx_pinned_alloc(reinterpret_cast<void**>(&a->h_pinned), 8 * pinned_words));
  return QX_OK;
}

void qx_arena_release(QxArena* a) {
  qx_dev_free(a->scratch, a->stream);
  qx_dev_free(a->status, a->stream);
  qx_pinned_free(a->h_pinned);
  a->scratch = nullptr;
  a->status = nullptr;
  a->h_pinned = nullptr;
}

int qx_arena_scratch(QxArena* s, int64_t bytes) {
  if (bytes <= s->scratch_bytes) return QX_OK;
  qx_dev_free(s->scratch, s->stream);     // stream-ordered: earlier kernels still see it
  s->scratch = nullptr;
  s->scratch_bytes = 0;
  const int64_t want = bytes + bytes / 4 + 4096;
  QX_TRY(qx_dev_alloc(&s->scratch, want, s->stream, s->device));
  s->scratch_bytes = want;
  return QX_OK;
}

int qx_arena_status(QxArena* s, int64_t words) {
  if (words <= s->status_words) return QX_OK;
  qx_dev_free(s->status, s->stream);
  s->status = nullptr;
  s->status_words = 0;
  const int64_t want = words + words / 4 + 1024;
  QX_TRY(qx_dev_alloc_t(&s->status, want, s->stream, s->device));
  s->status_words = want;
  return QX_OK;
}

// Small device -> host read-backs (offsets, counts) go through a kernel that stores into
// page-locked host memory (directly addressable under UVA) instead of cudaMemcpyAsync: a copy
// would queue on the device-to-host copy engine behind whatever bulk download another store
// has in flight there, and stall this store's host thread for the length of that download.
static __global__ void k_readback(int64_t* __restrict__ host_dst, const int64_t* __restrict__ src, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    host_dst[i] = src[i];
}

int qx_readback(cudaStream_t stream, int64_t* pinned_dst, const int64_t* d_src, int64_t n_words) {
  if (n_words <= 0) return QX_OK;
  const int grid = (int)std::min<int64_t>((n_words + 255) / 256, 64);
  k_readback<<<grid, 256, 0, stream>>>(pinned_dst, d_src, n_words);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  return QX_OK;
}

int qx_store_refresh(qx_store* s) {
  QX_CUDA(cudaSetDevice(s->device));
  QX_TRY(qx_readback(s->stream, s->h_seg, s->seg[s->cur], (int64_t)s->n_seg + 1));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  s->exact = true;
  s->ub_total = s->h_seg[s->n_seg];
  int64_t m = 0;
  for (int g = 0; g < s->n_seg; ++g) m = std::max(m, s->h_seg[g + 1] - s->h_seg[g]);
  s->ub_seg = m;
  return QX_OK;
}

// ----------------------------------------------------------------------------
// content in / out
// ----------------------------------------------------------------------------
extern "C" int qx_store_upload(qx_store* s, const int64_t* offsets, const uint64_t* keys,
                               const double* lambdas) {
  QX_REQUIRE(s && offsets, "NULL argument");
  QX_NARROW_ONLY(s, "qx_store_upload");
  QX_REQUIRE(offsets[0] == 0, "offsets[0] must be 0");
  for (int g = 0; g < s->n_seg; ++g)
    QX_REQUIRE(offsets[g + 1] >= offsets[g], "offsets must be non-decreasing (segment %d)", g);
  const int64_t total = offsets[s->n_seg];
  QX_REQUIRE(total == 0 || (keys && lambdas), "keys/lambdas are NULL");
  if (s->n_qubits < 32) {
    const uint64_t limit = 1ull << (2 * s->n_qubits);
    for (int64_t i = 0; i < total; ++i)
      QX_REQUIRE(keys[i] < limit, "word index %llu out of range [0, 4**%d)",
                 (unsigned long long)keys[i], s->n_qubits);
  }
  QX_CUDA(cudaSetDevice(s->device));
  QX_TRY(qx_store_reserve(s, total, false));
  const int c = s->cur;
  if (total > 0) {
    QX_CUDA(cudaMemcpyAsync(s->keys[c], keys, sizeof(u64) * (size_t)total, cudaMemcpyHostToDevice,
                            s->stream));
    QX_CUDA(cudaMemcpyAsync(s->lam[c], lambdas, sizeof(double) * (size_t)total,
                            cudaMemcpyHostToDevice, s->stream));
  }
  memcpy(s->h_seg, offsets, sizeof(int64_t) * (size_t)(s->n_seg + 1));
  QX_CUDA(cudaMemcpyAsync(s->seg[c], s->h_seg, sizeof(int64_t) * (size_t)(s->n_seg + 1),
                          cudaMemcpyHostToDevice, s->stream));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  s->exact = true;
  s->ub_total = total;
  s->ub_seg = 0;
  for (int g = 0; g < s->n_seg; ++g) s->ub_seg = std::max(s->ub_seg, offsets[g + 1] - offsets[g]);
  return QX_OK;
}

extern "C" int qx_store_upload_wide(qx_store* s, const int64_t* offsets, const uint64_t* words,
                                    const double* lambdas);

extern "C" int qx_store_init_z(qx_store* s, const int32_t* qubits) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  if (s->n_words > 1) {
    const int W = s->n_words;
    std::vector<int64_t> off(s->n_seg + 1);
    std::vector<uint64_t> words((size_t)s->n_seg * W, 0ull);
    std::vector<double> lam(s->n_seg, 1.0);
    for (int g = 0; g < s->n_seg; ++g) {
      const int q = qubits ? qubits[g] : g;
      QX_REQUIRE(q >= 0 && q < s->n_qubits, "qubit %d out of range for n=%d", q, s->n_qubits);
      const int pos = 2 * (s->n_qubits - 1 - q);
      off[g] = g;
      words[(size_t)g * W + (pos >> 6)] = 3ull << (pos & 63);
    }
    off[s->n_seg] = s->n_seg;
    return qx_store_upload_wide(s, off.data(), words.data(), lam.data());
  }
  std::vector<int64_t> off(s->n_seg + 1);
  std::vector<uint64_t> keys(s->n_seg);
  std::vector<double> lam(s->n_seg, 1.0);
  for (int g = 0; g < s->n_seg; ++g) {
    const int q = qubits ? qubits[g] : g;
    QX_REQUIRE(q >= 0 && q < s->n_qubits, "qubit %d out of range for n=%d", q, s->n_qubits);
    off[g] = g;
    keys[g] = 3ull << (2 * (s->n_qubits - 1 - q));
  }
  off[s->n_seg] = s->n_seg;
  return qx_store_upload(s, off.data(), keys.data(), lam.data());
}

extern "C" int qx_store_ranks(qx_store* s, int64_t* ranks) {
  QX_REQUIRE(s && ranks, "NULL argument");
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  for (int g = 0; g < s->n_seg; ++g) ranks[g] = s->h_seg[g + 1] - s->h_seg[g];
  return QX_OK;
}

extern "C" int qx_store_download(qx_store* s, int64_t* offsets, uint64_t* keys, double* lambdas,
                                 int64_t cap_terms) {
  QX_REQUIRE(s && offsets, "NULL argument");
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  memcpy(offsets, s->h_seg, sizeof(int64_t) * (size_t)(s->n_seg + 1));
  const int64_t total = s->h_seg[s->n_seg];
  if (keys == nullptr && lambdas == nullptr) return QX_OK;
  QX_NARROW_ONLY(s, "qx_store_download");
  QX_REQUIRE(cap_terms >= total, "download buffer holds %lld terms, store has %lld",
             (long long)cap_terms, (long long)total);
  QX_CUDA(cudaSetDevice(s->device));
  if (total > 0) {
    if (keys)
      QX_CUDA(cudaMemcpyAsync(keys, s->keys[s->cur], sizeof(u64) * (size_t)total,
                              cudaMemcpyDeviceToHost, s->stream));
    if (lambdas)
      QX_CUDA(cudaMemcpyAsync(lambdas, s->lam[s->cur], sizeof(double) * (size_t)total,
                              cudaMemcpyDeviceToHost, s->stream));
  }
  QX_CUDA(cudaStreamSynchronize(s->stream));
  return QX_OK;
}

extern "C" int qx_store_download_async(qx_store* s, int64_t* offsets, uint64_t* keys, double* lambdas,
                                       int64_t cap_terms) {
  QX_REQUIRE(s && offsets && keys && lambdas, "NULL argument");
  QX_NARROW_ONLY(s, "qx_store_download_async");
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  memcpy(offsets, s->h_seg, sizeof(int64_t) * (size_t)(s->n_seg + 1));
  const int64_t total = s->h_seg[s->n_seg];
  QX_REQUIRE(cap_terms >= total, "download buffer holds %lld terms, store has %lld",
             (long long)cap_terms, (long long)total);
  QX_CUDA(cudaSetDevice(s->device));
  if (total > 0) {
    QX_CUDA(cudaMemcpyAsync(keys, s->keys[s->cur], sizeof(u64) * (size_t)total, cudaMemcpyDeviceToHost,
                            s->stream));
    QX_CUDA(cudaMemcpyAsync(lambdas, s->lam[s->cur], sizeof(double) * (size_t)total, cudaMemcpyDeviceToHost,
                            s->stream));
  }
  return QX_OK;
}

extern "C" int qx_store_device_view(qx_store* s, const uint64_t** d_keys, const double** d_lambdas,
                                    const int64_t** d_offsets) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  QX_NARROW_ONLY(s, "qx_store_device_view");
  if (d_keys) *d_keys = (const uint64_t*)s->keys[s->cur];
  if (d_lambdas) *d_lambdas = s->lam[s->cur];
  if (d_offsets) *d_offsets = s->seg[s->cur];
  return QX_OK;
}

extern "C" int qx_store_capacity(qx_store* s, int64_t* capacity_terms, int64_t* hbm_bytes) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  if (capacity_terms) *capacity_terms = s->cap;
  if (hbm_bytes) *hbm_bytes = (32 + 16 * (s->n_words - 1)) * s->cap + s->scratch_bytes + 4 * s->status_words;
  return QX_OK;
}

// ---- narrow download: 32-bit keys over PCIe, widened on the host while the copy runs ----------
namespace {
struct HostWorkers {
  std::vector<std::thread> threads;
  std::vector<cudaEvent_t> events;
};

void join_workers(qx_store* s) {
  HostWorkers* hw = static_cast<HostWorkers*>(s->host_workers);
  if (!hw) return;
  for (std::thread& t : hw->threads) t.join();
  for (cudaEvent_t e : hw->events)
    if (e) cudaEventDestroy(e);
  delete hw;
  s->host_workers = nullptr;
}
}  // namespace

extern "C" int qx_store_set_keep_narrow(qx_store* s, int on) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  s->want_narrow = on < 0 ? 0 : (on > 2 ? 2 : on);
  return QX_OK;
}

extern "C" int qx_store_download_narrow_async(qx_store* s, int64_t* offsets, uint64_t* keys, double* lambdas,
                                              int64_t cap_terms, uint32_t* staging, int32_t threads) {
  QX_REQUIRE(s && offsets && keys && lambdas, "NULL argument");
  if (!s->narrow_keys) return qx_store_download_async(s, offsets, keys, lambdas, cap_terms);
  QX_REQUIRE(staging != nullptr, "staging is NULL");
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  memcpy(offsets, s->h_seg, sizeof(int64_t) * (size_t)(s->n_seg + 1));
  const int64_t total = s->h_seg[s->n_seg];
  QX_REQUIRE(cap_terms >= total, "download buffer holds %lld terms, store has %lld", (long long)cap_terms,
             (long long)total);
  QX_CUDA(cudaSetDevice(s->device));
  join_workers(s);
  if (total == 0) return QX_OK;
  // the keys first, in a few chunks with an event behind each, then the coefficients in one
  // copy: the host threads widen chunk c while the later chunks and the (twice as large)
  // coefficient copy are still on the wire.  Few, large copies: every cudaMemcpyAsync costs the
  // copy engine tens of microseconds of set-up.
  static const int max_chunks = getenv("QX_WIDEN_CHUNKS") ? atoi(getenv("QX_WIDEN_CHUNKS")) : 2;
  const int n_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(max_chunks, total / (1 << 20)));
  const int64_t chunk = (total + n_chunks - 1) / n_chunks;
  HostWorkers* hw = new HostWorkers();
  hw->events.resize(n_chunks, nullptr);
  s->host_workers = hw;             // owned by the store from here on: an error below cannot leak it
  const u32* d_keys = reinterpret_cast<const u32*>(s->keys[s->cur]);
  for (int c = 0; c < n_chunks; ++c) {
    const int64_t lo = c * chunk, len = std::min(chunk, total - lo);
    cudaEventCreateWithFlags(&hw->events[c], cudaEventDisableTiming);
    if (len > 0)
      QX_CUDA(cudaMemcpyAsync(staging + lo, d_keys + lo, sizeof(u32) * (size_t)len, cudaMemcpyDeviceToHost, s->stream));
    QX_CUDA(cudaEventRecord(hw->events[c], s->stream));
  }
  QX_CUDA(cudaMemcpyAsync(lambdas, s->lam[s->cur], sizeof(double) * (size_t)total, cudaMemcpyDeviceToHost, s->stream));
  const int T = std::max(1, std::min<int>(threads, 64));
  const int device = s->device;
  static const bool skip_widen = getenv("QX_WIDEN_SKIP") != nullptr;      // timing experiments only
  for (int t = 0; t < T; ++t)
    hw->threads.emplace_back([=]() {
      cudaSetDevice(device);
      for (int c = 0; c < n_chunks; ++c) {
        cudaEventSynchronize(hw->events[c]);
        const int64_t lo = c * chunk, len = std::min(chunk, total - lo);
        const int64_t a = lo + len * t / T, b = lo + len * (t + 1) / T;
        // streaming stores: the destination is written once and not read here -- no
        // read-for-ownership traffic competing with the DMA for host memory bandwidth
#if defined(__x86_64__)
        for (int64_t i = a; i < b; ++i) _mm_stream_si64(reinterpret_cast<long long*>(keys + i), (long long)staging[i]);
        _mm_sfence();
#else
        for (int64_t i = a; i < b; ++i) keys[i] = staging[i];
#endif
      }
    });
  s->host_workers = hw;
  return QX_OK;
}

// Packed form (qx_store_set_keep_narrow(s, 2) and a large result): per term the low 16 bits of
// its key, per generator a table first[h] = position of its first key with high half >= h.
// Ten bytes per term cross PCIe; the host threads rebuild the 64-bit keys bucket by bucket.
extern "C" int qx_store_download_packed_async(qx_store* s, int64_t* offsets, uint64_t* keys, double* lambdas,
                                              int64_t cap_terms, uint32_t* staging, int64_t staging_words,
                                              int32_t threads, int64_t* d2h_bytes) {
  QX_REQUIRE(s && offsets && keys && lambdas, "NULL argument");
  if (!s->narrow_keys || !s->pack_bnd) {
    QX_REQUIRE(!s->narrow_keys || staging_words >= cap_terms, "staging holds %lld words, need %lld",
               (long long)staging_words, (long long)cap_terms);
    QX_TRY(qx_store_download_narrow_async(s, offsets, keys, lambdas, cap_terms, staging, threads));
    if (d2h_bytes) *d2h_bytes = (s->narrow_keys ? 12 : 16) * s->h_seg[s->n_seg];
    return QX_OK;
  }
  QX_REQUIRE(staging != nullptr, "staging is NULL");
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  memcpy(offsets, s->h_seg, sizeof(int64_t) * (size_t)(s->n_seg + 1));
  const int64_t total = s->h_seg[s->n_seg];
  const int n_seg = s->n_seg;
  const int64_t bnd_words = (int64_t)n_seg * (QX_PACK_BUCKETS + 1);
  const int64_t lo_words = (total + 1) / 2;
  QX_REQUIRE(cap_terms >= total, "download buffer holds %lld terms, store has %lld", (long long)cap_terms,
             (long long)total);
  QX_REQUIRE(staging_words >= bnd_words + lo_words, "staging holds %lld words, the packed form needs %lld",
             (long long)staging_words, (long long)(bnd_words + lo_words));
  QX_CUDA(cudaSetDevice(s->device));
  join_workers(s);
  if (d2h_bytes) *d2h_bytes = 10 * total + 4 * bnd_words;
  if (total == 0) return QX_OK;
  // staging: [bucket tables][low halves]; the tables first (every chunk needs them), then the
  // halves in a few chunks with an event behind each, then the coefficients in one copy
  u32* h_bnd = staging;
  unsigned short* h_lo = reinterpret_cast<unsigned short*>(staging + bnd_words);
  static const int max_chunks = getenv("QX_WIDEN_CHUNKS") ? atoi(getenv("QX_WIDEN_CHUNKS")) : 2;
  const int n_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(max_chunks, total / (1 << 20)));
  const int64_t chunk = (total + n_chunks - 1) / n_chunks;
  HostWorkers* hw = new HostWorkers();
  hw->events.resize(n_chunks, nullptr);
  s->host_workers = hw;             // owned by the store from here on: an error below cannot leak it
  QX_CUDA(cudaMemcpyAsync(h_bnd, s->pack_bnd, sizeof(u32) * (size_t)bnd_words, cudaMemcpyDeviceToHost, s->stream));
  const unsigned short* d_lo = reinterpret_cast<const unsigned short*>(s->keys[s->cur]);
  for (int c = 0; c < n_chunks; ++c) {
    const int64_t lo = c * chunk, len = std::min(chunk, total - lo);
    cudaEventCreateWithFlags(&hw->events[c], cudaEventDisableTiming);
    if (len > 0)
      QX_CUDA(cudaMemcpyAsync(h_lo + lo, d_lo + lo, sizeof(unsigned short) * (size_t)len, cudaMemcpyDeviceToHost, s->stream));
    QX_CUDA(cudaEventRecord(hw->events[c], s->stream));
  }
  QX_CUDA(cudaMemcpyAsync(lambdas, s->lam[s->cur], sizeof(double) * (size_t)total, cudaMemcpyDeviceToHost, s->stream));
  const int T = std::max(1, std::min<int>(threads, 64));
  const int device = s->device;
  std::vector<int64_t> off(offsets, offsets + n_seg + 1);
  for (int t = 0; t < T; ++t)
    hw->threads.emplace_back([=]() {
      cudaSetDevice(device);
      for (int c = 0; c < n_chunks; ++c) {
        cudaEventSynchronize(hw->events[c]);
        const int64_t lo = c * chunk, len = std::min(chunk, total - lo);
        const int64_t a = lo + len * t / T, b = lo + len * (t + 1) / T;     // my global positions
        int g = (int)(std::upper_bound(off.begin(), off.end(), a) - off.begin()) - 1;
        for (int64_t p = a; p < b; ++g) {
          const int64_t g0 = off[g], g1 = std::min<int64_t>(off[g + 1], b);
          if (g1 <= p) continue;                                             // empty generator
          const u32* first = h_bnd + (size_t)g * (QX_PACK_BUCKETS + 1);
          const u32 lp = (u32)(p - g0), le = (u32)(g1 - g0);
          // bucket of local position lp: first[h] <= lp < first[h + 1]
          u32 h = (u32)(std::upper_bound(first, first + QX_PACK_BUCKETS + 1, lp) - first) - 1u;
          u32 q = lp;
          while (q < le) {
            const u32 end = std::min(first[h + 1], le);
            const u64 hi = (u64)h << 16;
#if defined(__x86_64__)
            for (u32 i = q; i < end; ++i)
              _mm_stream_si64(reinterpret_cast<long long*>(keys + g0 + i), (long long)(hi | h_lo[g0 + i]));
#else
            for (u32 i = q; i < end; ++i) keys[g0 + i] = hi | h_lo[g0 + i];
#endif
            if (end > q) q = end;
            ++h;
          }
          p = g1;
        }
#if defined(__x86_64__)
        _mm_sfence();
#endif
      }
    });
  s->host_workers = hw;
  return QX_OK;
}

// ---- phase timers (the reference's four timing keys, measured on the device) ----
extern "C" int qx_store_event_record(qx_store* s, int32_t* index) {
  QX_REQUIRE(s && index, "NULL argument");
  QX_CUDA(cudaSetDevice(s->device));
  if (!s->events) s->events = new std::vector<cudaEvent_t>();
  cudaEvent_t e;
  if (!event_pool_take(s->device, &e)) QX_CUDA(cudaEventCreate(&e));
  s->events->push_back(e);
  QX_CUDA(cudaEventRecord(e, s->stream));
  *index = (int32_t)s->events->size() - 1;
  return QX_OK;
}

extern "C" int qx_store_event_elapsed(qx_store* s, int32_t first, int32_t second, double* ms) {
  QX_REQUIRE(s && ms, "NULL argument");
  const int32_t n = s->events ? (int32_t)s->events->size() : 0;
  QX_REQUIRE(first >= 0 && first < n && second >= 0 && second < n, "event index out of range (%d, %d of %d)", first,
             second, n);
  QX_CUDA(cudaSetDevice(s->device));
  QX_CUDA(cudaEventSynchronize((*s->events)[second]));
  float f = 0.f;
  QX_CUDA(cudaEventElapsedTime(&f, (*s->events)[first], (*s->events)[second]));
  *ms = (double)f;
  return QX_OK;
}

extern "C" int qx_store_synchronize(qx_store* s) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  QX_CUDA(cudaSetDevice(s->device));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  join_workers(s);
  return QX_OK;
}
