// Internal declarations shared by the translation units of libqimax_b200.so.
// sm_100a only; no CPU fallback anywhere in this library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/qimax_b200.h"

typedef unsigned long long u64;
typedef unsigned int u32;

// ----------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------
int qx_fail(int status, const char* fmt, ...);

#define QX_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      return qx_fail(QX_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,                  \
                     cudaGetErrorString(_e), __FILE__, __LINE__);                  \
  } while (0)

#define QX_TRY(expr)                 \
  do {                               \
    int _s = (expr);                 \
    if (_s != QX_OK) return _s;      \
  } while (0)

#define QX_REQUIRE(cond, ...)                              \
  do {                                                     \
    if (!(cond)) return qx_fail(QX_ERR_INVALID, __VA_ARGS__); \
  } while (0)

// ----------------------------------------------------------------------------
// instrumentation (profile.cu)
// ----------------------------------------------------------------------------
struct QxProfileScope {
  int cls;
  cudaStream_t stream;
  cudaEvent_t start, stop;
  bool active;
  QxProfileScope(int kernel_class, cudaStream_t st, double alg_bytes, int launches = 1);
  ~QxProfileScope();
};
void qx_count_launches(int n);
bool qx_profile_on();

// ----------------------------------------------------------------------------
// geometry of the device-wide passes
// ----------------------------------------------------------------------------
constexpr int QX_MAX_QUBITS = 32;         // one-word keys: every kernel
constexpr int QX_MAX_WORDS = 16;          // multi-word keys (wide.cu), n <= 512
constexpr int QX_MAX_QUBITS_WIDE = 32 * QX_MAX_WORDS;
constexpr int QX_RADIX_BITS = 8;
constexpr int QX_RADIX = 1 << QX_RADIX_BITS;
constexpr int QX_PACK_BUCKETS = 1 << 16;  // packed download: one bucket per value of a key's high 16 bits
constexpr int QX_SORT_THREADS = 384;     // 12 warps
constexpr int QX_SORT_ITEMS = 12;        // keys per thread, warp-striped
constexpr int QX_SORT_TILE = QX_SORT_THREADS * QX_SORT_ITEMS;   // 4608 terms
constexpr int QX_SMALL_MAX = 8192;       // largest segment the one-CTA merge takes
constexpr int QX_SCAN_THREADS = 256;
constexpr int QX_SCAN_ITEMS = 8;
constexpr int QX_SCAN_TILE = QX_SCAN_THREADS * QX_SCAN_ITEMS;   // 2048 terms

// ----------------------------------------------------------------------------
// per-handle device context + scratch, shared by the store and the expansion
// ----------------------------------------------------------------------------
struct QxArena {
  int device = 0;
  int n_qubits = 0;
  int sm_count = 148;
  cudaStream_t stream = 0;
  bool own_stream = false;      // created by the library (qx_store_slice): destroyed with the handle
  void* scratch = nullptr;      // generic byte scratch (tables, histograms, offsets)
  int64_t scratch_bytes = 0;
  u32* status = nullptr;        // look-back words of the sort passes
  int64_t status_words = 0;
  int64_t* h_pinned = nullptr;  // small pinned staging
  int64_t h_pinned_words = 0;
};
// Device allocations through the library's caching allocator (store.cu): a store created
// per circuit run gets its multi-GB buffers back in microseconds instead of paying
// cudaMalloc/cudaFree (tens of ms) every run.
int qx_dev_alloc(void** out, int64_t bytes, cudaStream_t stream, int device);
void qx_dev_free(void* ptr, cudaStream_t stream);
void qx_dev_forget_stream(cudaStream_t stream);
int qx_pinned_alloc(void** out, int64_t bytes);
void qx_pinned_free(void* ptr);
template <typename T>
inline int qx_dev_alloc_t(T** out, int64_t count, cudaStream_t stream, int device) {
  return qx_dev_alloc(reinterpret_cast<void**>(out), (int64_t)sizeof(T) * count, stream, device);
}

int qx_arena_init(QxArena* a, int device, int n_qubits, int64_t pinned_words);
void qx_arena_release(QxArena* a);
int qx_arena_scratch(QxArena* a, int64_t bytes);
int qx_arena_status(QxArena* a, int64_t words);

// ----------------------------------------------------------------------------
// the term store (a1)
// ----------------------------------------------------------------------------
struct qx_store : QxArena {
  int n_seg = 0;
  int64_t cap = 0;              // terms per buffer
  u64* keys[2] = {nullptr, nullptr};
  double* lam[2] = {nullptr, nullptr};
  int64_t* seg[2] = {nullptr, nullptr};   // device offsets, n_seg+1 each
  int want_narrow = 0;          // the caller only downloads next: the grouped step may leave 32-bit keys (1)
                                // or 16-bit low halves + a bucket table (2)
  bool narrow_keys = false;     // keys[cur] holds 32-bit keys (n <= 16); only the narrow download reads them
  u32* pack_bnd = nullptr;      // != nullptr: keys[cur] holds 16-bit low halves and this is the bucket table
                                // (n_seg x (QX_PACK_BUCKETS + 1), inside the keys[cur] block behind the halves)
  void* host_workers = nullptr; // threads widening downloaded keys on the host (store.cu), joined by synchronize
  int n_words = 1;              // 64-bit words per key; > 1 = wide store (wide.cu)
  u64* hi[2] = {nullptr, nullptr};        // words 1..n_words-1, plane-major, `cap` words per plane
  int cur = 0;                  // which of the two buffers is live
  int64_t* h_seg = nullptr;     // pinned host mirror of the live offsets
  bool exact = false;           // h_seg matches the device
  int64_t ub_total = 0;         // host upper bound on the live term count
  int64_t ub_seg = 0;           // host upper bound on the largest live segment
  std::vector<cudaEvent_t>* events = nullptr;   // phase timers of the caller (qx_store_event_record)
};

int qx_store_reserve(qx_store* s, int64_t terms, bool keep_live);
int qx_store_refresh(qx_store* s);          // D2H of the live offsets, sets exact
// n_words int64 from device memory into PAGE-LOCKED host memory, by a kernel on `stream` (no copy engine)
int qx_readback(cudaStream_t stream, int64_t* pinned_dst, const int64_t* d_src, int64_t n_words);
inline void qx_store_flip(qx_store* s) { s->cur ^= 1; }
inline int qx_store_scratch(qx_store* s, int64_t bytes) { return qx_arena_scratch(s, bytes); }

// clifford.cu: validate a sign-permutation program against the store's qubit count
int qx_check_program(const qx_store* s, const uint32_t* program, int32_t n_ops);
// the reference's CX tables (lut.py:108-134) in the packed form of qx_apply_clifford
void qx_standard_cx(u32* cx_c, u32* cx_t, u32* cx_s);
// merge.cu: canonicalize (or only sort) the live buffer; narrow = it holds 32-bit raw keys
int qx_run_merge(qx_store* s, double eps, bool sort_only, bool narrow);
// wide.cu: the merge of a multi-word store
int qx_wide_merge(qx_store* s, double eps);
// merge.cu: stable segmented sort of (64-bit key, opaque 8-byte payload) pairs by the low `bits`
// bits of the key with the onesweep passes; buffers ping-pong, *cur names the live pair
int qx_sort_pairs(qx_store* s, u64* keys[2], double* vals[2], int64_t* seg[2], int* cur, int64_t total,
                  int64_t largest_seg, int bits);
// entry points that only exist for one-word keys refuse wide stores with this
#define QX_NARROW_ONLY(s, what)                                                                      \
  do {                                                                                               \
    if ((s)->n_words > 1)                                                                            \
      return qx_fail(QX_ERR_UNSUPPORTED, "%s needs one-word keys (n <= %d); this store has n = %d", \
                     what, QX_MAX_QUBITS, (s)->n_qubits);                                            \
    if ((s)->narrow_keys)                                                                            \
      return qx_fail(QX_ERR_INVALID, "%s: the store was left with 32-bit keys for download "         \
                     "(qx_store_set_keep_narrow); only qx_store_download_narrow_async reads it", what); \
  } while (0)
