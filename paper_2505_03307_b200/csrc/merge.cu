// a6 for the evolution store: qx_merge (canonicalize, reference stabilizer.py:325-337),
// plus the per-segment reductions of the read-out side: Z/I-only sums (north-star
// kernel 4) and sum of squares (the P^2 = I self-check).
#include "merge.cuh"

int qx_run_merge(qx_store* s, double eps, bool sort_only, bool narrow) {
  // multi-word keys: one CTA per generator (wide.cu); a sort is a merge that drops nothing
  if (s->n_words > 1) return qx_wide_merge(s, sort_only ? 0.0 : eps);
  QX_NARROW_ONLY(s, "merge");
  if (s->ub_seg > QX_SMALL_MAX && !s->exact) QX_TRY(qx_store_refresh(s));
  // both paths write into the other buffer; make sure it can hold the raw terms
  qxm::MergeBuffers<double> mb;
  for (int b = 0; b < 2; ++b) {
    mb.keys[b] = s->keys[b];
    mb.vals[b] = s->lam[b];
    mb.seg[b] = s->seg[b];
  }
  mb.cur = s->cur;
  mb.n_seg = s->n_seg;
  mb.ub_total = s->ub_total;
  mb.ub_seg = s->ub_seg;
  bool small = s->ub_seg <= QX_SMALL_MAX;
  if (narrow) {
    if (small || sort_only) return qx_fail(QX_ERR_CONSISTENCY, "narrow keys outside the large merge (internal error)");
    QX_TRY((qxm::merge_large<double, u32>(s, mb, eps, QX_K_REDUCE, true)));
  } else if (small) {
    QX_TRY(qxm::merge_small<double>(s, mb, eps, QX_K_SMALL_MERGE));
  } else {
    QX_TRY(qxm::merge_large<double>(s, mb, eps, QX_K_REDUCE, !sort_only));
    if (sort_only) {            // a permutation inside each segment: sizes are what they were
      s->cur = mb.cur;
      return QX_OK;
    }
  }
  s->cur = mb.cur;
  s->exact = false;
  QX_TRY(qx_store_refresh(s));                     // one small D2H: the new ranks
  if (small && *reinterpret_cast<int*>(s->h_pinned) != 0)
    return qx_fail(QX_ERR_CONSISTENCY, "small-merge segment bound violated (internal error)");
  return QX_OK;
}

int qx_sort_pairs(qx_store* s, u64* keys[2], double* vals[2], int64_t* seg[2], int* cur, int64_t total,
                  int64_t largest_seg, int bits) {
  qxm::MergeBuffers<double> mb;
  for (int b = 0; b < 2; ++b) {
    mb.keys[b] = keys[b];
    mb.vals[b] = vals[b];
    mb.seg[b] = seg[b];
  }
  mb.cur = *cur;
  mb.n_seg = s->n_seg;
  mb.ub_total = total;
  mb.ub_seg = largest_seg;
  QX_TRY((qxm::merge_large<double, u64>(s, mb, 0.0, QX_K_REDUCE, false, QX_K_SORT_PASS, QX_K_SORT_HIST, nullptr,
                                        nullptr, true, nullptr, bits)));
  *cur = mb.cur;
  return QX_OK;
}

namespace {

// ---- per-segment deterministic reductions -------------------------------------------
constexpr int kRedThreads = 256;
constexpr int kChunks = 64;          // fixed split of every segment: the sum order never changes

// hi / n_words / cap: the upper key words of a multi-word store (n > 32), plane-major (csrc/wide.cu)
template <int MODE>                  // 0: sum over Z/I-only words, 1: sum of squares
__global__ void __launch_bounds__(kRedThreads)
k_segment_partial(const u64* __restrict__ keys, const u64* __restrict__ hi, int n_words, int64_t cap,
                  const double* __restrict__ lam, const int64_t* __restrict__ seg,
                  double* __restrict__ partial) {
  __shared__ double s_warp[kRedThreads / 32];
  const int g = blockIdx.y, c = blockIdx.x;
  const int64_t lo = seg[g], n = seg[g + 1] - lo;
  const int64_t per = (n + kChunks - 1) / kChunks;
  const int64_t a = lo + c * per, b = min(lo + n, a + per);
  double acc = 0.0;
  for (int64_t i = a + threadIdx.x; i < b; i += kRedThreads) {
    const double v = lam[i];
    if (MODE == 0) {
      bool zi = zi_only(keys[i]);
      for (int w = 1; w < n_words; ++w) zi = zi && zi_only(hi[(size_t)(w - 1) * (size_t)cap + i]);
      if (zi) acc += v;
    } else {
      acc += v * v;
    }
  }
  acc = warp_sum(acc);                         // xor butterfly: fixed tree
  if (lane_id() == 0) s_warp[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) t += s_warp[w];
    partial[(size_t)g * kChunks + c] = t;
  }
}

__global__ void k_segment_final(const double* __restrict__ partial, double* __restrict__ out,
                                int n_seg) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_seg) return;
  double t = 0.0;
  for (int c = 0; c < kChunks; ++c) t += partial[(size_t)g * kChunks + c];
  out[g] = t;
}

template <int MODE>
int segment_reduce(qx_store* s, double* host_out) {
  QX_REQUIRE(s && host_out, "NULL argument");
  QX_CUDA(cudaSetDevice(s->device));
  const int64_t bytes = 8ll * s->n_seg * (kChunks + 1);
  QX_TRY(qx_store_scratch(s, bytes));
  double* partial = reinterpret_cast<double*>(s->scratch);
  double* out = partial + (size_t)s->n_seg * kChunks;
  {
    QxProfileScope prof(QX_K_READOUT_REDUCE, s->stream, 16.0 * (double)s->ub_total, 2);
    dim3 grid(kChunks, s->n_seg);
    k_segment_partial<MODE><<<grid, kRedThreads, 0, s->stream>>>(
        s->keys[s->cur], s->n_words > 1 ? s->hi[s->cur] : nullptr, s->n_words, (int64_t)s->cap,
        s->lam[s->cur], s->seg[s->cur], partial);
    QX_CUDA(cudaGetLastError());
    k_segment_final<<<(s->n_seg + 127) / 128, 128, 0, s->stream>>>(partial, out, s->n_seg);
    QX_CUDA(cudaGetLastError());
  }
  QX_CUDA(cudaMemcpyAsync(host_out, out, sizeof(double) * (size_t)s->n_seg, cudaMemcpyDeviceToHost,
                          s->stream));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  return QX_OK;
}

}  // namespace

extern "C" int qx_merge(qx_store* s, double eps, int64_t* ranks) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  QX_REQUIRE(eps >= 0.0, "eps must be non-negative");
  QX_CUDA(cudaSetDevice(s->device));
  QX_TRY(qx_run_merge(s, eps, false, false));
  if (ranks)
    for (int g = 0; g < s->n_seg; ++g) ranks[g] = s->h_seg[g + 1] - s->h_seg[g];
  return QX_OK;
}

extern "C" int qx_sort(qx_store* s) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  QX_CUDA(cudaSetDevice(s->device));
  return qx_run_merge(s, 0.0, true, false);
}

extern "C" int qx_store_zi_sums(qx_store* s, double* sums) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  return segment_reduce<0>(s, sums);     // any key width: the upper words are tested plane by plane
}
extern "C" int qx_store_norms(qx_store* s, double* sum_sq) { return segment_reduce<1>(s, sum_sq); }
