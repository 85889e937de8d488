// a1: the Pauli-term store in HBM, plus library-level plumbing (errors, device info,
// CUDA-event instrumentation).  Replaces SimpleGenerator / GeneratorSet / init_z
// (reference stabilizer.py:83-109, 157-174).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>

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
// store lifetime and capacity
// ----------------------------------------------------------------------------
static int alloc_buffers(qx_store* s, int64_t cap, u64** keys, double** lam) {
  size_t free_b = 0, total_b = 0;
  QX_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double need = 2.0 * 16.0 * (double)cap;
  if (need > 0.92 * (double)free_b)
    return qx_fail(QX_ERR_RESOURCE,
                   "term store of %lld terms needs %.1f GB of HBM, %.1f GB free on device %d",
                   (long long)cap, need / 1e9, free_b / 1e9, s->device);
  for (int b = 0; b < 2; ++b) {
    QX_CUDA(cudaMalloc(&keys[b], sizeof(u64) * (size_t)cap));
    QX_CUDA(cudaMalloc(&lam[b], sizeof(double) * (size_t)cap));
  }
  return QX_OK;
}

extern "C" int qx_store_create(int device, int n_qubits, int n_segments, int64_t capacity_terms,
                               qx_store** out) {
  QX_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  if (n_qubits < 1) return qx_fail(QX_ERR_INVALID, "qubit count must be positive, got %d", n_qubits);
  if (n_qubits > QX_MAX_QUBITS)
    return qx_fail(QX_ERR_UNSUPPORTED, "n_qubits=%d: keys are one 64-bit word (n <= %d)", n_qubits,
                   QX_MAX_QUBITS);
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
  s->cap = std::max<int64_t>(capacity_terms, std::max<int64_t>(4096, 2 * (int64_t)n_segments));
  int st = alloc_buffers(s, s->cap, s->keys, s->lam);
  if (st == QX_OK) {
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < 2 && e == cudaSuccess; ++b)
      e = cudaMalloc(&s->seg[b], sizeof(int64_t) * (size_t)(n_segments + 1));
    if (e == cudaSuccess) e = cudaMallocHost(&s->h_seg, sizeof(int64_t) * (size_t)(n_segments + 1));
    if (e == cudaSuccess) e = cudaMemset(s->seg[0], 0, sizeof(int64_t) * (size_t)(n_segments + 1));
    if (e != cudaSuccess) st = qx_fail(QX_ERR_CUDA, "store allocation failed: %s", cudaGetErrorString(e));
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

extern "C" int qx_store_destroy(qx_store* s) {
  if (!s) return QX_OK;
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  for (int b = 0; b < 2; ++b) {
    cudaFree(s->keys[b]);
    cudaFree(s->lam[b]);
    cudaFree(s->seg[b]);
  }
  cudaFreeHost(s->h_seg);
  qx_arena_release(s);
  delete s;
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
  QX_CUDA(cudaStreamSynchronize(s->stream));
  // Growth is done one buffer pair at a time so the peak is old + new, not 2x new.
  int64_t want = std::max<int64_t>(terms + terms / 8, s->cap * 2);
  size_t free_b = 0, total_b = 0;
  QX_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double avail = 0.94 * ((double)free_b + 32.0 * (double)s->cap);
  if (32.0 * (double)want > avail) want = terms;
  if (32.0 * (double)want > avail)
    return qx_fail(QX_ERR_RESOURCE,
                   "term store would need %.1f GB of HBM for %lld terms (%.1f GB usable on device %d)",
                   32.0 * (double)want / 1e9, (long long)want, avail / 1e9, s->device);
  const int dead = s->cur ^ 1;
  QX_CUDA(cudaFree(s->keys[dead]));
  QX_CUDA(cudaFree(s->lam[dead]));
  s->keys[dead] = nullptr;
  s->lam[dead] = nullptr;
  QX_CUDA(cudaMalloc(&s->keys[dead], sizeof(u64) * (size_t)want));
  QX_CUDA(cudaMalloc(&s->lam[dead], sizeof(double) * (size_t)want));
  if (live > 0) {
    QX_CUDA(cudaMemcpyAsync(s->keys[dead], s->keys[s->cur], sizeof(u64) * (size_t)live,
                            cudaMemcpyDeviceToDevice, s->stream));
    QX_CUDA(cudaMemcpyAsync(s->lam[dead], s->lam[s->cur], sizeof(double) * (size_t)live,
                            cudaMemcpyDeviceToDevice, s->stream));
    QX_CUDA(cudaStreamSynchronize(s->stream));
  }
  const int old = s->cur;
  QX_CUDA(cudaFree(s->keys[old]));
  QX_CUDA(cudaFree(s->lam[old]));
  s->keys[old] = nullptr;
  s->lam[old] = nullptr;
  QX_CUDA(cudaMalloc(&s->keys[old], sizeof(u64) * (size_t)want));
  QX_CUDA(cudaMalloc(&s->lam[old], sizeof(double) * (size_t)want));
  // live data now sits in `dead`; the offsets follow the live index
  if (s->cur != dead) {
    QX_CUDA(cudaMemcpyAsync(s->seg[dead], s->seg[s->cur], sizeof(int64_t) * (size_t)(s->n_seg + 1),
                            cudaMemcpyDeviceToDevice, s->stream));
    QX_CUDA(cudaStreamSynchronize(s->stream));
    s->cur = dead;
  }
  s->cap = want;
  return QX_OK;
}

int qx_arena_init(QxArena* a, int device, int n_qubits, int64_t pinned_words) {
  int count = 0;
  QX_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    return qx_fail(QX_ERR_CUDA, "CUDA device %d not available (%d visible)", device, count);
  QX_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  QX_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return qx_fail(QX_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a only",
                   device, prop.major, prop.minor);
  a->device = device;
  a->n_qubits = n_qubits;
  a->sm_count = prop.multiProcessorCount;
  a->h_pinned_words = pinned_words;
  QX_CUDA(cudaMallocHost(&a->h_pinned, sizeof(int64_t) * (size_t)pinned_words));
  return QX_OK;
}

void qx_arena_release(QxArena* a) {
  cudaFree(a->scratch);
  cudaFree(a->status);
  cudaFreeHost(a->h_pinned);
  a->scratch = nullptr;
  a->status = nullptr;
  a->h_pinned = nullptr;
}

int qx_arena_scratch(QxArena* s, int64_t bytes) {
  if (bytes <= s->scratch_bytes) return QX_OK;
  QX_CUDA(cudaStreamSynchronize(s->stream));
  if (s->scratch) QX_CUDA(cudaFree(s->scratch));
  s->scratch = nullptr;
  s->scratch_bytes = 0;
  const int64_t want = bytes + bytes / 4 + 4096;
  cudaError_t e = cudaMalloc(&s->scratch, (size_t)want);
  if (e != cudaSuccess)
    return qx_fail(QX_ERR_RESOURCE, "scratch of %.2f GB not available: %s", want / 1e9,
                   cudaGetErrorString(e));
  s->scratch_bytes = want;
  return QX_OK;
}

int qx_arena_status(QxArena* s, int64_t words) {
  if (words <= s->status_words) return QX_OK;
  QX_CUDA(cudaStreamSynchronize(s->stream));
  if (s->status) QX_CUDA(cudaFree(s->status));
  s->status = nullptr;
  s->status_words = 0;
  const int64_t want = words + words / 4 + 1024;
  cudaError_t e = cudaMalloc(&s->status, sizeof(u32) * (size_t)want);
  if (e != cudaSuccess)
    return qx_fail(QX_ERR_RESOURCE, "look-back table of %.2f GB not available: %s",
                   4.0 * want / 1e9, cudaGetErrorString(e));
  s->status_words = want;
  return QX_OK;
}

int qx_store_refresh(qx_store* s) {
  QX_CUDA(cudaSetDevice(s->device));
  QX_CUDA(cudaMemcpyAsync(s->h_seg, s->seg[s->cur], sizeof(int64_t) * (size_t)(s->n_seg + 1),
                          cudaMemcpyDeviceToHost, s->stream));
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

extern "C" int qx_store_init_z(qx_store* s, const int32_t* qubits) {
  QX_REQUIRE(s != nullptr, "store is NULL");
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

extern "C" int qx_store_device_view(qx_store* s, const uint64_t** d_keys, const double** d_lambdas,
                                    const int64_t** d_offsets) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  if (d_keys) *d_keys = (const uint64_t*)s->keys[s->cur];
  if (d_lambdas) *d_lambdas = s->lam[s->cur];
  if (d_offsets) *d_offsets = s->seg[s->cur];
  return QX_OK;
}

extern "C" int qx_store_capacity(qx_store* s, int64_t* capacity_terms, int64_t* hbm_bytes) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  if (capacity_terms) *capacity_terms = s->cap;
  if (hbm_bytes) *hbm_bytes = 32 * s->cap + s->scratch_bytes + 4 * s->status_words;
  return QX_OK;
}

extern "C" int qx_store_synchronize(qx_store* s) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  QX_CUDA(cudaSetDevice(s->device));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  return QX_OK;
}
