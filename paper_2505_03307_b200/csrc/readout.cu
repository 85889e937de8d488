// a9 + a10: density expansion 2^-n * prod_j (I + P_j) and coefficient look-up
// (reference measure.py:40-123, product tables pauli.py:37-49).
//
// The accumulator is a one-segment store with complex128 coefficients (double2).
// One generator round is:
//   product  out = acc  U  { acc_a * g_b }: word = XOR of the two keys (the base-4
//            codes multiply by XOR), phase = i^(sum of PHASE_EXP over digits), which on
//            the packed key is two popcounts of bit-plane masks -- no per-digit loop;
//   merge    the same sort + run-sum machinery as the evolution store, complex sums,
//            dropping exact zeros only (measure.py:86).
// The term budget is checked on the raw length before anything is written, like the
// reference does (measure.py:59-62).
#include "merge.cuh"

struct qx_expansion : QxArena {
  int64_t cap = 0;
  u64* keys[2] = {nullptr, nullptr};
  double2* vals[2] = {nullptr, nullptr};
  int64_t* seg[2] = {nullptr, nullptr};   // {0, count}
  int cur = 0;
  int64_t count = 0;                       // exact, host side
  u64* g_keys = nullptr;                   // staging for a generator passed from the host
  double* g_lam = nullptr;
  int64_t g_cap = 0;
};

namespace {

constexpr int kThreads = 256;
constexpr u64 kPlane = 0x5555555555555555ull;

// exponent k of a.b = i^k (a xor b), digits packed 2 bits each (pauli.py:38-46)
__device__ __forceinline__ u32 product_phase(u64 a, u64 b) {
  const u64 ah = (a >> 1) & kPlane, al = a & kPlane, bh = (b >> 1) & kPlane, bl = b & kPlane;
  const u64 plus = ((~ah & al & bh & ~bl) | (ah & ~al & bh & bl) | (ah & al & ~bh & bl)) & kPlane;
  const u64 active = (ah | al) & (bh | bl) & ((ah ^ bh) | (al ^ bl));
  const u64 minus = active & ~plus;
  return (u32)(__popcll(plus) - __popcll(minus)) & 3u;
}

__global__ void __launch_bounds__(kThreads)
k_pair_product(const u64* __restrict__ acc_keys, const double2* __restrict__ acc_vals, int64_t na,
               const u64* __restrict__ g_keys, const double* __restrict__ g_lam, int64_t ng,
               u64* __restrict__ out_keys, double2* __restrict__ out_vals, int64_t* seg_out) {
  const int64_t raw = na * (1 + ng);
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < raw; r += stride) {
    if (r < na) {
      out_keys[r] = acc_keys[r];
      out_vals[r] = acc_vals[r];
      continue;
    }
    const int64_t p = r - na;
    const int64_t a = p / ng, b = p - a * ng;
    const u64 ka = acc_keys[a], kb = g_keys[b];
    const double2 c = acc_vals[a];
    const double l = g_lam[b];
    const double re = c.x * l, im = c.y * l;
    double2 v;
    switch (product_phase(ka, kb)) {
      case 0: v = make_double2(re, im); break;
      case 1: v = make_double2(-im, re); break;
      case 2: v = make_double2(-re, -im); break;
      default: v = make_double2(im, -re); break;
    }
    st_stream(out_keys + r, ka ^ kb);
    st_stream(out_vals + r, v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    seg_out[0] = 0;
    seg_out[1] = raw;
  }
}

__global__ void k_set_identity(u64* keys, double2* vals, int64_t* seg) {
  keys[0] = 0ull;
  vals[0] = make_double2(1.0, 0.0);
  seg[0] = 0;
  seg[1] = 1;
}

__global__ void __launch_bounds__(kThreads)
k_max_abs_imag(const double2* __restrict__ vals, int64_t n, double* __restrict__ out) {
  // single CTA per launch slice; max is order-independent, so the result is deterministic
  __shared__ double s_warp[kThreads / 32];
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    m = fmax(m, fabs(vals[i].y));
  for (int d = 16; d > 0; d >>= 1) m = fmax(m, __shfl_xor_sync(QX_FULL_MASK, m, d));
  if (lane_id() == 0) s_warp[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) m = fmax(m, s_warp[w]);
    out[blockIdx.x] = m;
  }
}

// coefficient of each queried word: binary search in the ascending unique keys
__global__ void k_lookup(const u64* __restrict__ keys, const double2* __restrict__ vals, int64_t n,
                         const u64* __restrict__ words, int64_t nw, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nw) return;
  const u64 w = words[i];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < w) lo = mid + 1; else hi = mid;
  }
  out[i] = (lo < n && keys[lo] == w) ? vals[lo].x : 0.0;
}

int reserve(qx_expansion* e, int64_t terms) {
  if (terms <= e->cap) return QX_OK;
  const int64_t want = std::max<int64_t>(terms + terms / 8, 2 * e->cap);
  const int dead = e->cur ^ 1, old = e->cur;
  qx_dev_free(e->keys[dead], e->stream);
  qx_dev_free(e->vals[dead], e->stream);
  e->keys[dead] = nullptr;
  e->vals[dead] = nullptr;
  QX_TRY(qx_dev_alloc_t(&e->keys[dead], want, e->stream, e->device));
  QX_TRY(qx_dev_alloc_t(&e->vals[dead], want, e->stream, e->device));
  if (e->count > 0) {
    QX_CUDA(cudaMemcpyAsync(e->keys[dead], e->keys[old], sizeof(u64) * (size_t)e->count,
                            cudaMemcpyDeviceToDevice, e->stream));
    QX_CUDA(cudaMemcpyAsync(e->vals[dead], e->vals[old], sizeof(double2) * (size_t)e->count,
                            cudaMemcpyDeviceToDevice, e->stream));
  }
  QX_CUDA(cudaMemcpyAsync(e->seg[dead], e->seg[old], sizeof(int64_t) * 2, cudaMemcpyDeviceToDevice,
                          e->stream));
  qx_dev_free(e->keys[old], e->stream);
  qx_dev_free(e->vals[old], e->stream);
  e->keys[old] = nullptr;
  e->vals[old] = nullptr;
  QX_TRY(qx_dev_alloc_t(&e->keys[old], want, e->stream, e->device));
  QX_TRY(qx_dev_alloc_t(&e->vals[old], want, e->stream, e->device));
  e->cur = dead;
  e->cap = want;
  return QX_OK;
}

int multiply_device(qx_expansion* e, const u64* d_keys, const double* d_lam, int64_t ng,
                    int64_t term_budget) {
  const int64_t raw = e->count * (1 + ng);
  if (term_budget >= 0 && raw > term_budget)      // negative: no budget (the reference has no such value)
    return qx_fail(QX_ERR_RESOURCE, "density expansion exceeded the term budget (%lld)",
                   (long long)term_budget);
  QX_TRY(reserve(e, raw));
  const int in = e->cur, out = e->cur ^ 1;
  {
    const int64_t want = (raw + kThreads - 1) / kThreads;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)e->sm_count * 8));
    QxProfileScope prof(QX_K_READOUT_PRODUCT, e->stream, 24.0 * (double)(e->count + raw));
    k_pair_product<<<grid, kThreads, 0, e->stream>>>(e->keys[in], e->vals[in], e->count, d_keys, d_lam,
                                                     ng, e->keys[out], e->vals[out], e->seg[out]);
    QX_CUDA(cudaGetLastError());
  }
  qxm::MergeBuffers<double2> mb;
  for (int b = 0; b < 2; ++b) {
    mb.keys[b] = e->keys[b];
    mb.vals[b] = e->vals[b];
    mb.seg[b] = e->seg[b];
  }
  mb.cur = out;
  mb.n_seg = 1;
  mb.ub_total = raw;
  mb.ub_seg = raw;
  const bool small = raw <= QX_SMALL_MAX;
  if (small) {
    QX_TRY(qxm::merge_small<double2>(e, mb, 0.0, QX_K_SMALL_MERGE));
  } else {
    QX_TRY(qxm::merge_large<double2>(e, mb, 0.0, QX_K_READOUT_REDUCE));
  }
  e->cur = mb.cur;
  QX_CUDA(cudaMemcpyAsync(e->h_pinned + 2, e->seg[e->cur], sizeof(int64_t) * 2, cudaMemcpyDeviceToHost,
                          e->stream));
  QX_CUDA(cudaStreamSynchronize(e->stream));
  if (small && *reinterpret_cast<int*>(e->h_pinned) != 0)
    return qx_fail(QX_ERR_CONSISTENCY, "small-merge segment bound violated (internal error)");
  e->count = e->h_pinned[3];
  return QX_OK;
}

}  // namespace

extern "C" int qx_expansion_create(int device, int n_qubits, int64_t capacity_terms,
                                   qx_expansion** out) {
  QX_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  if (n_qubits < 1) return qx_fail(QX_ERR_INVALID, "qubit count must be positive, got %d", n_qubits);
  if (n_qubits > QX_MAX_QUBITS)
    return qx_fail(QX_ERR_UNSUPPORTED, "n_qubits=%d: keys are one 64-bit word (n <= %d)", n_qubits,
                   QX_MAX_QUBITS);
  qx_expansion* e = new qx_expansion();
  int st = qx_arena_init(e, device, n_qubits, 16);
  if (st != QX_OK) {
    delete e;
    return st;
  }
  e->cap = std::max<int64_t>(capacity_terms, 4096);
  for (int b = 0; b < 2 && st == QX_OK; ++b) {
    st = qx_dev_alloc_t(&e->keys[b], e->cap, e->stream, e->device);
    if (st == QX_OK) st = qx_dev_alloc_t(&e->vals[b], e->cap, e->stream, e->device);
    if (st == QX_OK) st = qx_dev_alloc_t(&e->seg[b], 2, e->stream, e->device);
  }
  if (st != QX_OK) {
    qx_expansion_destroy(e);
    return st;
  }
  st = qx_expansion_reset(e);
  if (st != QX_OK) {
    qx_expansion_destroy(e);
    return st;
  }
  *out = e;
  return QX_OK;
}

extern "C" int qx_expansion_destroy(qx_expansion* e) {
  if (!e) return QX_OK;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->stream);
  for (int b = 0; b < 2; ++b) {
    qx_dev_free(e->keys[b], e->stream);
    qx_dev_free(e->vals[b], e->stream);
    qx_dev_free(e->seg[b], e->stream);
  }
  qx_dev_free(e->g_keys, e->stream);
  qx_dev_free(e->g_lam, e->stream);
  qx_arena_release(e);
  delete e;
  return QX_OK;
}

extern "C" int qx_expansion_reset(qx_expansion* e) {
  QX_REQUIRE(e != nullptr, "expansion is NULL");
  QX_CUDA(cudaSetDevice(e->device));
  k_set_identity<<<1, 1, 0, e->stream>>>(e->keys[e->cur], e->vals[e->cur], e->seg[e->cur]);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  e->count = 1;
  return QX_OK;
}

extern "C" int qx_expansion_multiply(qx_expansion* e, const uint64_t* keys, const double* lambdas,
                                     int64_t count, int64_t term_budget) {
  QX_REQUIRE(e != nullptr && count >= 0, "bad argument");
  QX_REQUIRE(count == 0 || (keys && lambdas), "keys/lambdas are NULL");
  QX_CUDA(cudaSetDevice(e->device));
  if (count > e->g_cap) {
    qx_dev_free(e->g_keys, e->stream);
    qx_dev_free(e->g_lam, e->stream);
    e->g_keys = nullptr;
    e->g_lam = nullptr;
    e->g_cap = 0;
    const int64_t want = std::max<int64_t>(count, 1024);
    QX_TRY(qx_dev_alloc_t(&e->g_keys, want, e->stream, e->device));
    QX_TRY(qx_dev_alloc_t(&e->g_lam, want, e->stream, e->device));
    e->g_cap = want;
  }
  if (count > 0) {
    QX_CUDA(cudaMemcpyAsync(e->g_keys, keys, sizeof(u64) * (size_t)count, cudaMemcpyHostToDevice, e->stream));
    QX_CUDA(cudaMemcpyAsync(e->g_lam, lambdas, sizeof(double) * (size_t)count, cudaMemcpyHostToDevice,
                            e->stream));
  }
  return multiply_device(e, e->g_keys, e->g_lam, count, term_budget);
}

extern "C" int qx_expansion_multiply_segment(qx_expansion* e, qx_store* s, int32_t segment,
                                             int64_t term_budget) {
  QX_REQUIRE(e && s, "NULL argument");
  QX_NARROW_ONLY(s, "qx_expansion_multiply_segment");
  QX_REQUIRE(segment >= 0 && segment < s->n_seg, "segment %d out of range", segment);
  QX_REQUIRE(e->device == s->device, "store and expansion live on different devices");
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  QX_CUDA(cudaSetDevice(e->device));
  if (e->stream != s->stream) QX_CUDA(cudaStreamSynchronize(s->stream));
  const int64_t lo = s->h_seg[segment], n = s->h_seg[segment + 1] - lo;
  return multiply_device(e, s->keys[s->cur] + lo, s->lam[s->cur] + lo, n, term_budget);
}

extern "C" int qx_expansion_size(qx_expansion* e, int64_t* terms) {
  QX_REQUIRE(e && terms, "NULL argument");
  *terms = e->count;
  return QX_OK;
}

extern "C" int qx_expansion_max_abs_imag(qx_expansion* e, double* worst) {
  QX_REQUIRE(e && worst, "NULL argument");
  QX_CUDA(cudaSetDevice(e->device));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((e->count + kThreads - 1) / kThreads, 1024));
  QX_TRY(qx_arena_scratch(e, 8 * 1024));
  double* d_out = reinterpret_cast<double*>(e->scratch);
  {
    QxProfileScope prof(QX_K_READOUT_REDUCE, e->stream, 16.0 * (double)e->count);
    k_max_abs_imag<<<grid, kThreads, 0, e->stream>>>(e->vals[e->cur], e->count, d_out);
    QX_CUDA(cudaGetLastError());
  }
  std::vector<double> host(grid);
  QX_CUDA(cudaMemcpyAsync(host.data(), d_out, sizeof(double) * (size_t)grid, cudaMemcpyDeviceToHost,
                          e->stream));
  QX_CUDA(cudaStreamSynchronize(e->stream));
  double m = 0.0;
  for (double v : host) m = std::max(m, v);
  *worst = m;
  return QX_OK;
}

extern "C" int qx_expansion_download(qx_expansion* e, uint64_t* keys, double* re, double* im,
                                     int64_t cap_terms) {
  QX_REQUIRE(e != nullptr, "expansion is NULL");
  QX_REQUIRE(cap_terms >= e->count, "download buffer holds %lld terms, expansion has %lld",
             (long long)cap_terms, (long long)e->count);
  QX_CUDA(cudaSetDevice(e->device));
  const int64_t n = e->count;
  if (n == 0) return QX_OK;
  if (keys)
    QX_CUDA(cudaMemcpyAsync(keys, e->keys[e->cur], sizeof(u64) * (size_t)n, cudaMemcpyDeviceToHost,
                            e->stream));
  if (re)
    QX_CUDA(cudaMemcpy2DAsync(re, sizeof(double), e->vals[e->cur], sizeof(double2), sizeof(double),
                              (size_t)n, cudaMemcpyDeviceToHost, e->stream));
  if (im)
    QX_CUDA(cudaMemcpy2DAsync(im, sizeof(double), reinterpret_cast<double*>(e->vals[e->cur]) + 1,
                              sizeof(double2), sizeof(double), (size_t)n, cudaMemcpyDeviceToHost,
                              e->stream));
  QX_CUDA(cudaStreamSynchronize(e->stream));
  return QX_OK;
}

extern "C" int qx_expansion_lookup(qx_expansion* e, const uint64_t* words, int64_t n_words,
                                   double* re) {
  QX_REQUIRE(e && n_words >= 0, "bad argument");
  if (n_words == 0) return QX_OK;
  QX_REQUIRE(words && re, "words/re are NULL");
  QX_CUDA(cudaSetDevice(e->device));
  QX_TRY(qx_arena_scratch(e, 16 * n_words));
  u64* d_words = reinterpret_cast<u64*>(e->scratch);
  double* d_out = reinterpret_cast<double*>(d_words + n_words);
  QX_CUDA(cudaMemcpyAsync(d_words, words, sizeof(u64) * (size_t)n_words, cudaMemcpyHostToDevice, e->stream));
  k_lookup<<<(unsigned)((n_words + 255) / 256), 256, 0, e->stream>>>(e->keys[e->cur], e->vals[e->cur],
                                                                     e->count, d_words, n_words, d_out);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  QX_CUDA(cudaMemcpyAsync(re, d_out, sizeof(double) * (size_t)n_words, cudaMemcpyDeviceToHost, e->stream));
  QX_CUDA(cudaStreamSynchronize(e->stream));
  return QX_OK;
}
