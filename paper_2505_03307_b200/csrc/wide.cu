// More than 32 qubits: multi-word keys.
//
// The reference switches to Python big-int indices above 31 qubits (stabilizer.py:40-59) so that
// Clifford and near-Clifford circuits run at any width -- their stabilizer rank stays tiny.  On
// the device a wide store keeps W = ceil(2n / 64) words per term as W planes (word 0, the least
// significant one, in the ordinary key array; words 1..W-1 plane-major in `hi`), n <= 512.
//
// What runs on wide stores is the part of the path such circuits use:
//   qx_apply_clifford_wide  fused run of sign-permutation gates (apply_cx stabilizer.py:340-363,
//                           H/S/X/SX of engine.py:183-218): one thread per term, words in local
//                           memory, the whole program applied before the term is written back;
//   qx_apply_split_wide     v1 rotation (engine.py:190-217): two entries per term, the second
//                           one (second branch weight 0) a zero-weight copy of the first, which
//                           the merge adds into the same key without changing the sum;
//   merge / sort            generators up to 16384 / W raw terms: one CTA per generator, bitonic
//                           sort on (words, input position) in shared memory, in-order run sums,
//                           drop rule, compaction across generators by look-back.  Larger ones:
//                           a permutation sorted word by word with the one-word onesweep passes
//                           (stable LSD over the W words), then one reduce + compaction pass.
// Branching operators of v2/v3 are applied gate by gate with these kernels (engine.py); the
// grouped operator step (run on the generators' support: qx_store_compact / qx_store_expand), the
// density-expansion read-out and partitioning stay one-word (QX_ERR_UNSUPPORTED); the Heisenberg
// read-out (qx_store_zi_sums, merge.cu) takes any width.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "qx_device.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxWords = QX_MAX_WORDS;

struct Planes {
  u64* p[kMaxWords];
};

Planes planes_of(qx_store* s, int buf) {
  Planes pl;
  for (int w = 0; w < kMaxWords; ++w) pl.p[w] = nullptr;
  pl.p[0] = s->keys[buf];
  for (int w = 1; w < s->n_words; ++w) pl.p[w] = s->hi[buf] + (size_t)(w - 1) * (size_t)s->cap;
  return pl;
}

// ---- Clifford run ----------------------------------------------------------------------------
// op: bits 0-1 kind (0 = 1q permutation, 1 = CX); bits 16-23 image axes, 24-27 signs (as in
// qx_apply_clifford); bits 32-47 bit position of the (control) digit; bits 48-63 of the target.
__global__ void __launch_bounds__(kThreads)
k_clifford_wide(Planes pl, double* __restrict__ lam, const int64_t* __restrict__ seg, int n_seg, int n_words,
                const u64* __restrict__ ops, int n_ops, u32 cx_c, u32 cx_t, u32 cx_s) {
  const int64_t total = seg[n_seg];
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < total; i += (int64_t)gridDim.x * kThreads) {
    u64 k[kMaxWords];
    for (int w = 0; w < n_words; ++w) k[w] = pl.p[w][i];
    u32 neg = 0;
    for (int j = 0; j < n_ops; ++j) {
      const u64 op = ops[j];
      const u32 lo = (u32)op;
      const u32 p0 = (u32)(op >> 32) & 0xffffu;
      const u32 d0 = (u32)(k[p0 >> 6] >> (p0 & 63u)) & 3u;
      if ((lo & 3u) == 0u) {
        const u32 nd = (lo >> (16u + 2u * d0)) & 3u;
        neg ^= (lo >> (24u + d0)) & 1u;
        k[p0 >> 6] ^= (u64)(d0 ^ nd) << (p0 & 63u);
      } else {
        const u32 p1 = (u32)(op >> 48) & 0xffffu;
        const u32 d1 = (u32)(k[p1 >> 6] >> (p1 & 63u)) & 3u;
        const u32 e = d0 * 4u + d1;
        neg ^= (cx_s >> e) & 1u;
        k[p0 >> 6] ^= (u64)(d0 ^ ((cx_c >> (2u * e)) & 3u)) << (p0 & 63u);
        k[p1 >> 6] ^= (u64)(d1 ^ ((cx_t >> (2u * e)) & 3u)) << (p1 & 63u);
      }
    }
    for (int w = 0; w < n_words; ++w) pl.p[w][i] = k[w];
    if (neg) lam[i] = -lam[i];
  }
}

// ---- v1 split --------------------------------------------------------------------------------
struct SplitTableW {
  double w1[4], w2[4];
  u32 a1[4], a2[4];
  u32 pos;
};

__global__ void __launch_bounds__(kThreads)
k_split_wide(Planes in, const double* __restrict__ lam_in, const int64_t* __restrict__ seg_in, int n_seg,
             int n_words, Planes out, double* __restrict__ lam_out, int64_t* __restrict__ seg_out,
             const SplitTableW tb) {
  const int64_t total = seg_in[n_seg];
  const int word = (int)(tb.pos >> 6), sh = (int)(tb.pos & 63u);
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < total; i += (int64_t)gridDim.x * kThreads) {
    const double l = lam_in[i];
    const u64 kw = in.p[word][i];
    const u32 d = (u32)(kw >> sh) & 3u;
    const u64 cleared = kw & ~(3ull << sh);
    const bool second = tb.w2[d] != 0.0;
    for (int w = 0; w < n_words; ++w) {
      const u64 v = in.p[w][i];
      out.p[w][2 * i] = w == word ? (cleared | ((u64)tb.a1[d] << sh)) : v;
      // no second branch: a zero-weight copy of the first one (the merge adds 0.0 into its key)
      out.p[w][2 * i + 1] = w == word ? (cleared | ((u64)(second ? tb.a2[d] : tb.a1[d]) << sh)) : v;
    }
    lam_out[2 * i] = l * tb.w1[d];
    lam_out[2 * i + 1] = second ? l * tb.w2[d] : 0.0;
  }
  for (int g = blockIdx.x * kThreads + threadIdx.x; g <= n_seg; g += gridDim.x * kThreads) seg_out[g] = 2 * seg_in[g];
}

// ---- merge: one CTA per generator ----------------------------------------------------------------
constexpr int kMergeThreads = 512;

__device__ __forceinline__ bool wide_greater(const u64* sk, int cap, int n_words, int a, int b,
                                             unsigned short ia, unsigned short ib) {
  for (int w = n_words - 1; w >= 0; --w) {
    const u64 ka = sk[(size_t)w * cap + a], kb = sk[(size_t)w * cap + b];
    if (ka != kb) return ka > kb;
  }
  return ia > ib;
}
__device__ __forceinline__ bool wide_equal(const u64* sk, int cap, int n_words, int a, int b) {
  for (int w = 0; w < n_words; ++w)
    if (sk[(size_t)w * cap + a] != sk[(size_t)w * cap + b]) return false;
  return true;
}

__global__ void __launch_bounds__(kMergeThreads)
k_small_merge_wide(Planes in, const double* __restrict__ lam_in, const int64_t* __restrict__ seg_in, int n_seg,
                   int n_words, Planes out, double* __restrict__ lam_out, int64_t* __restrict__ seg_out,
                   u64* status, u32* ticket, int* error, int cap, double eps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* sk = reinterpret_cast<u64*>(smem_raw);                                   // [n_words][cap]
  unsigned short* sidx = reinterpret_cast<unsigned short*>(sk + (size_t)n_words * cap);
  __shared__ int s_g;
  __shared__ u64 s_scan[kMergeThreads / 32 + 1];
  __shared__ u64 s_base;
  if (threadIdx.x == 0) s_g = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int g = s_g;
  if (g >= n_seg) return;
  const int64_t start = seg_in[g];
  int len = (int)min((int64_t)0x7fffffff, seg_in[g + 1] - start);
  if (len > cap) {
    if (threadIdx.x == 0) atomicExch(error, 1);
    len = 0;
  }
  int m = 32;
  while (m < len) m <<= 1;
  for (int e = threadIdx.x; e < m; e += kMergeThreads) {
    for (int w = 0; w < n_words; ++w) sk[(size_t)w * cap + e] = e < len ? in.p[w][start + e] : ~0ull;
    sidx[e] = (unsigned short)e;
  }
  __syncthreads();
  // padding: all-ones words and position >= len, so it ends up behind every live term
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (m >> 1); t += kMergeThreads) {
        const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int hi = lo | j;
        const unsigned short ia = sidx[lo], ib = sidx[hi];
        const bool greater = wide_greater(sk, cap, n_words, lo, hi, ia, ib);
        if (greater == ((lo & k) == 0)) {
          for (int w = 0; w < n_words; ++w) {
            const u64 a = sk[(size_t)w * cap + lo];
            sk[(size_t)w * cap + lo] = sk[(size_t)w * cap + hi];
            sk[(size_t)w * cap + hi] = a;
          }
          sidx[lo] = ib;
          sidx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  const int rows = (len + kMergeThreads - 1) / kMergeThreads;
  u64 my_count = 0;
  for (int r = 0; r < rows; ++r) {
    const int e = r * kMergeThreads + threadIdx.x;
    if (e < len && (e == 0 || !wide_equal(sk, cap, n_words, e - 1, e))) {
      double sum = lam_in[start + sidx[e]];
      for (int j = e + 1; j < len && wide_equal(sk, cap, n_words, e, j); ++j) sum += lam_in[start + sidx[j]];
      if (fabs(sum) >= eps) ++my_count;
    }
  }
  u64 seg_total;
  block_exclusive_sum<u64>(my_count, s_scan, seg_total);
  if ((threadIdx.x >> 5) == 0) {
    const u64 excl = lookback_exclusive(status, g, seg_total);
    if (lane_id() == 0) s_base = excl;
  }
  __syncthreads();
  const int64_t base = (int64_t)s_base;
  u64 kept_before = 0;
  for (int r = 0; r < rows; ++r) {
    const int e = r * kMergeThreads + threadIdx.x;
    bool kept = false;
    double sum = 0.0;
    if (e < len && (e == 0 || !wide_equal(sk, cap, n_words, e - 1, e))) {
      sum = lam_in[start + sidx[e]];
      for (int j = e + 1; j < len && wide_equal(sk, cap, n_words, e, j); ++j) sum += lam_in[start + sidx[j]];
      kept = fabs(sum) >= eps;
    }
    u64 row_total;
    const u64 excl = block_exclusive_sum<u64>(kept ? 1ull : 0ull, s_scan, row_total);
    if (kept) {
      const int64_t pos = base + (int64_t)(kept_before + excl);
      for (int w = 0; w < n_words; ++w) out.p[w][pos] = sk[(size_t)w * cap + e];
      lam_out[pos] = sum;
    }
    kept_before += row_total;
  }
  if (threadIdx.x == 0) {
    seg_out[g] = base;
    if (g == n_seg - 1) seg_out[n_seg] = base + (int64_t)seg_total;
  }
}

int merge_cap(int n_words) {
  int cap = 32;
  while (cap * 2 * n_words <= 16384) cap <<= 1;
  return cap;                                    // W = 2: 8192, 3-4: 4096, 5-8: 2048 raw terms per generator
}


// ---- merge of generators beyond one CTA's shared memory ----------------------------------------
// LSD over the W words: a permutation (input positions, carried as the 8-byte payload of the
// one-word onesweep passes of merge.cuh) is sorted stably by word 0, then word 1, ... word W-1,
// each time on the plane gathered through the permutation so far.  Stable passes leave equal
// words in input order, so the runs below are summed in the order np.add.at uses
// (stabilizer.py:333-335).  The terms themselves move once, in k_wide_reduce.
__global__ void k_wide_iota(double* __restrict__ perm, int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    perm[i] = __longlong_as_double((long long)i);
}

__global__ void k_wide_gather(const u64* __restrict__ plane, const double* __restrict__ perm, u64* __restrict__ out,
                              int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = plane[__double_as_longlong(perm[i])];
}

constexpr int kWrThreads = 256;
constexpr int kWrRows = 4;
constexpr int kWrTile = kWrThreads * kWrRows;

__device__ __forceinline__ bool wide_same(const Planes& pl, int n_words, int64_t a, int64_t b) {
  for (int w = 0; w < n_words; ++w)
    if (pl.p[w][a] != pl.p[w][b]) return false;
  return true;
}

// One thread per sorted position: heads (first of a run of equal words inside the generator) sum
// their run in order, apply the drop rule (stabilizer.py:336) and are compacted by a block scan +
// decoupled look-back over tiles (tile = blockIdx.x, see qx_device.cuh).
__global__ void __launch_bounds__(kWrThreads)
k_wide_reduce(Planes in, const double* __restrict__ lam_in, const double* __restrict__ perm,
              const int64_t* __restrict__ seg_in, int n_seg, int n_words, Planes out, double* __restrict__ lam_out,
              int64_t* __restrict__ seg_out, u64* status, double eps) {
  __shared__ u64 s_scan[kWrThreads / 32 + 1];
  __shared__ u64 s_base;
  const int tile = qx_tile_id(reinterpret_cast<u32*>(status + gridDim.x));   // see qx_device.cuh
  const int64_t total = seg_in[n_seg];
  const int64_t tbase = (int64_t)tile * kWrTile;
  bool kept[kWrRows], opens[kWrRows];
  double sum[kWrRows];
  int seg_id[kWrRows];
  u64 mine = 0;
#pragma unroll
  for (int r = 0; r < kWrRows; ++r) {
    const int64_t i = tbase + r * kWrThreads + threadIdx.x;
    kept[r] = opens[r] = false;
    sum[r] = 0.0;
    seg_id[r] = 0;
    if (i < total) {
      const int g = segment_of(seg_in, n_seg, i);
      const int64_t lo = seg_in[g], hi = seg_in[g + 1];
      const int64_t pi = __double_as_longlong(perm[i]);
      seg_id[r] = g;
      opens[r] = i == lo;
      if (i == lo || !wide_same(in, n_words, pi, __double_as_longlong(perm[i - 1]))) {
        double acc = lam_in[pi];
        for (int64_t j = i + 1; j < hi; ++j) {
          const int64_t pj = __double_as_longlong(perm[j]);
          if (!wide_same(in, n_words, pi, pj)) break;
          acc += lam_in[pj];
        }
        sum[r] = acc;
        kept[r] = fabs(acc) >= eps;
      }
    }
    mine += kept[r] ? 1ull : 0ull;
  }
  u64 tile_total;
  block_exclusive_sum<u64>(mine, s_scan, tile_total);
  if ((threadIdx.x >> 5) == 0) {
    const u64 excl = lookback_exclusive(status, tile, tile_total);
    if (lane_id() == 0) s_base = excl;
  }
  __syncthreads();
  const int64_t base = (int64_t)s_base;
  u64 before = 0;
#pragma unroll
  for (int r = 0; r < kWrRows; ++r) {
    const int64_t i = tbase + r * kWrThreads + threadIdx.x;
    u64 row_total;
    const u64 excl = block_exclusive_sum<u64>(kept[r] ? 1ull : 0ull, s_scan, row_total);
    const int64_t pos = base + (int64_t)(before + excl);
    if (opens[r]) open_offsets(seg_in, seg_out, seg_id[r], i, pos);
    if (kept[r]) {
      const int64_t pi = __double_as_longlong(perm[i]);
      for (int w = 0; w < n_words; ++w) out.p[w][pos] = in.p[w][pi];
      lam_out[pos] = sum[r];
    }
    before += row_total;
  }
  if (threadIdx.x == 0 && tbase + kWrTile >= total) close_offsets(seg_in, seg_out, n_seg, total, base + (int64_t)tile_total);
}

struct DevBlock {
  void* p = nullptr;
  cudaStream_t st = 0;
  ~DevBlock() {
    if (p) qx_dev_free(p, st);
  }
};

int wide_merge_large(qx_store* s, double eps) {
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  const int64_t total = s->h_seg[s->n_seg];
  int64_t largest = 0;
  for (int g = 0; g < s->n_seg; ++g) largest = std::max(largest, s->h_seg[g + 1] - s->h_seg[g]);
  const int in = s->cur, out = s->cur ^ 1;
  const int64_t tiles = std::max<int64_t>(1, (total + kWrTile - 1) / kWrTile);
  // one block: two key buffers, two permutation buffers, the spare offsets, the look-back words
  const int64_t n_al = (total + 31) & ~31ll;
  const int64_t seg_words = ((int64_t)s->n_seg + 1 + 31) & ~31ll;
  DevBlock blk;
  blk.st = s->stream;
  QX_TRY(qx_dev_alloc(&blk.p, 8 * (4 * n_al + seg_words + tiles + 1), s->stream, s->device));   // + the ticket word of QX_TICKETED_LOOKBACK builds
  u64* kbuf[2] = {reinterpret_cast<u64*>(blk.p), reinterpret_cast<u64*>(blk.p) + n_al};
  double* pbuf[2] = {reinterpret_cast<double*>(kbuf[1] + n_al), reinterpret_cast<double*>(kbuf[1] + 2 * n_al)};
  int64_t* seg_spare = reinterpret_cast<int64_t*>(kbuf[1] + 3 * n_al);
  u64* status = reinterpret_cast<u64*>(seg_spare + seg_words);
  int64_t* segs[2] = {s->seg[in], seg_spare};
  const Planes pin = planes_of(s, in);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)s->sm_count * 8));
  int cur = 0;
  k_wide_iota<<<grid, 256, 0, s->stream>>>(pbuf[cur], total);
  QX_CUDA(cudaGetLastError());
  for (int w = 0; w < s->n_words; ++w) {
    k_wide_gather<<<grid, 256, 0, s->stream>>>(pin.p[w], pbuf[cur], kbuf[cur], total);
    QX_CUDA(cudaGetLastError());
    // bits of this word that can be set: the top word of the key holds 2n - 64 (W - 1) of them
    const int bits = std::min(64, 2 * s->n_qubits - 64 * w);
    QX_TRY(qx_sort_pairs(s, kbuf, pbuf, segs, &cur, total, largest, bits));
  }
  QX_CUDA(cudaMemsetAsync(status, 0, sizeof(u64) * (size_t)(tiles + 1), s->stream));
  {
    QxProfileScope prof(QX_K_REDUCE, s->stream, (8.0 * s->n_words + 8.0) * 2.0 * (double)total);
    k_wide_reduce<<<(unsigned)tiles, kWrThreads, 0, s->stream>>>(pin, s->lam[in], pbuf[cur], segs[cur], s->n_seg,
                                                                s->n_words, planes_of(s, out), s->lam[out],
                                                                s->seg[out], status, eps);
    QX_CUDA(cudaGetLastError());
  }
  s->cur = out;
  s->exact = false;
  return qx_store_refresh(s);      // synchronises: the scratch block may go back to the allocator
}

}  // namespace

int qx_wide_merge(qx_store* s, double eps) {
  if (!s->exact && s->ub_seg > merge_cap(s->n_words)) QX_TRY(qx_store_refresh(s));
  if (s->ub_seg > merge_cap(s->n_words)) return wide_merge_large(s, eps);
  int cap = 32;
  while (cap < s->ub_seg) cap <<= 1;
  const size_t smem = (size_t)cap * (8 * (size_t)s->n_words + 2);
  const int64_t bytes = 16 + 8 * ((int64_t)s->n_seg + 1);
  QX_TRY(qx_arena_scratch(s, bytes));
  QX_CUDA(cudaMemsetAsync(s->scratch, 0, (size_t)bytes, s->stream));
  u32* ticket = reinterpret_cast<u32*>(s->scratch);
  int* error = reinterpret_cast<int*>(reinterpret_cast<char*>(s->scratch) + 8);
  u64* status = reinterpret_cast<u64*>(reinterpret_cast<char*>(s->scratch) + 16);
  static bool attr_set = false;
  if (!attr_set) {
    QX_CUDA(cudaFuncSetAttribute(k_small_merge_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8 + 8192 * 2 + 64));
    attr_set = true;
  }
  const int in = s->cur, out = s->cur ^ 1;
  {
    QxProfileScope prof(QX_K_SMALL_MERGE, s->stream, (8.0 * s->n_words + 8.0) * 2.0 * (double)s->ub_total);
    k_small_merge_wide<<<s->n_seg, kMergeThreads, smem, s->stream>>>(
        planes_of(s, in), s->lam[in], s->seg[in], s->n_seg, s->n_words, planes_of(s, out), s->lam[out],
        s->seg[out], status, ticket, error, cap, eps);
    QX_CUDA(cudaGetLastError());
  }
  QX_TRY(qx_readback(s->stream, s->h_pinned, reinterpret_cast<const int64_t*>(reinterpret_cast<char*>(s->scratch) + 8), 1));
  s->cur = out;
  s->exact = false;
  QX_TRY(qx_store_refresh(s));
  if ((int)(s->h_pinned[0] & 0xffffffff) != 0)
    return qx_fail(QX_ERR_CONSISTENCY, "multi-word merge: segment bound violated (internal error)");
  return QX_OK;
}

extern "C" int qx_apply_clifford_wide(qx_store* s, const uint64_t* ops, int32_t n_ops, uint32_t cx_c,
                                      uint32_t cx_t, uint32_t cx_s) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  QX_REQUIRE(n_ops >= 0 && (n_ops == 0 || ops), "bad program");
  QX_REQUIRE(s->n_words > 1, "store has one-word keys: use qx_apply_clifford");
  if (n_ops == 0) return QX_OK;
  const u32 limit = 2u * (u32)s->n_qubits;
  for (int i = 0; i < n_ops; ++i) {
    const u32 kind = (u32)ops[i] & 3u, p0 = (u32)(ops[i] >> 32) & 0xffffu, p1 = (u32)(ops[i] >> 48) & 0xffffu;
    QX_REQUIRE(kind <= 1u, "op %d: unknown kind %u", i, kind);
    QX_REQUIRE(p0 < limit && (p0 & 1u) == 0u, "op %d: digit position %u out of range", i, p0);
    if (kind == 1u) QX_REQUIRE(p1 < limit && (p1 & 1u) == 0u && p1 != p0, "op %d: bad CX target position %u", i, p1);
  }
  QX_CUDA(cudaSetDevice(s->device));
  QX_TRY(qx_arena_scratch(s, 8ll * n_ops));
  QX_CUDA(cudaMemcpyAsync(s->scratch, ops, sizeof(u64) * (size_t)n_ops, cudaMemcpyHostToDevice, s->stream));
  const int64_t total = std::max<int64_t>(s->ub_total, 1);
  const int grid = (int)std::min<int64_t>((total + kThreads - 1) / kThreads, (int64_t)s->sm_count * 8);
  {
    QxProfileScope prof(QX_K_CLIFFORD, s->stream, 2.0 * (8.0 * s->n_words + 8.0) * (double)s->ub_total);
    k_clifford_wide<<<grid, kThreads, 0, s->stream>>>(planes_of(s, s->cur), s->lam[s->cur], s->seg[s->cur], s->n_seg,
                                                      s->n_words, reinterpret_cast<const u64*>(s->scratch), n_ops,
                                                      cx_c, cx_t, cx_s);
    QX_CUDA(cudaGetLastError());
  }
  QX_CUDA(cudaStreamSynchronize(s->stream));     // the program was copied from caller memory
  return QX_OK;
}

extern "C" int qx_apply_split_wide(qx_store* s, int32_t qubit, const int32_t a1[4], const double w1[4],
                                   const int32_t a2[4], const double w2[4]) {
  QX_REQUIRE(s && a1 && w1 && a2 && w2, "NULL argument");
  QX_REQUIRE(s->n_words > 1, "store has one-word keys: use qx_apply_split");
  QX_REQUIRE(qubit >= 0 && qubit < s->n_qubits, "qubit %d out of range for n=%d", qubit, s->n_qubits);
  SplitTableW tb;
  tb.pos = 2u * (u32)(s->n_qubits - 1 - qubit);
  for (int d = 0; d < 4; ++d) {
    QX_REQUIRE(a1[d] >= 0 && a1[d] <= 3 && a2[d] >= 0 && a2[d] <= 3, "axis code out of range");
    tb.a1[d] = (u32)a1[d];
    tb.a2[d] = (u32)a2[d];
    tb.w1[d] = w1[d];
    tb.w2[d] = w2[d];
  }
  QX_CUDA(cudaSetDevice(s->device));
  const int64_t ub_in = s->ub_total;
  QX_TRY(qx_store_reserve(s, 2 * ub_in + 2, true));
  const int in = s->cur, out = s->cur ^ 1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((ub_in + kThreads - 1) / kThreads, (int64_t)s->sm_count * 8));
  {
    QxProfileScope prof(QX_K_SPLIT, s->stream, 3.0 * (8.0 * s->n_words + 8.0) * (double)ub_in);
    k_split_wide<<<grid, kThreads, 0, s->stream>>>(planes_of(s, in), s->lam[in], s->seg[in], s->n_seg, s->n_words,
                                                   planes_of(s, out), s->lam[out], s->seg[out], tb);
    QX_CUDA(cudaGetLastError());
  }
  qx_store_flip(s);
  s->exact = false;
  s->ub_total = 2 * ub_in;
  s->ub_seg = 2 * s->ub_seg;
  return QX_OK;
}

// content in / out: words are term-major on the host ([term][word], word 0 least significant)
extern "C" int qx_store_upload_wide(qx_store* s, const int64_t* offsets, const uint64_t* words,
                                    const double* lambdas) {
  QX_REQUIRE(s && offsets, "NULL argument");
  QX_REQUIRE(s->n_words > 1, "store has one-word keys: use qx_store_upload");
  QX_REQUIRE(offsets[0] == 0, "offsets[0] must be 0");
  for (int g = 0; g < s->n_seg; ++g)
    QX_REQUIRE(offsets[g + 1] >= offsets[g], "offsets must be non-decreasing (segment %d)", g);
  const int64_t total = offsets[s->n_seg];
  QX_REQUIRE(total == 0 || (words && lambdas), "words/lambdas are NULL");
  const int W = s->n_words;
  const int top_bits = 2 * s->n_qubits - 64 * (W - 1);
  if (top_bits < 64)
    for (int64_t i = 0; i < total; ++i)
      QX_REQUIRE((words[(size_t)i * W + (W - 1)] >> top_bits) == 0, "word index of term %lld out of range [0, 4**%d)",
                 (long long)i, s->n_qubits);
  QX_CUDA(cudaSetDevice(s->device));
  QX_TRY(qx_store_reserve(s, total, false));
  const int c = s->cur;
  std::vector<u64> plane((size_t)std::max<int64_t>(total, 1));
  const Planes pl = planes_of(s, c);
  for (int w = 0; w < W; ++w) {
    for (int64_t i = 0; i < total; ++i) plane[(size_t)i] = words[(size_t)i * W + w];
    if (total > 0) QX_CUDA(cudaMemcpy(pl.p[w], plane.data(), sizeof(u64) * (size_t)total, cudaMemcpyHostToDevice));
  }
  if (total > 0)
    QX_CUDA(cudaMemcpyAsync(s->lam[c], lambdas, sizeof(double) * (size_t)total, cudaMemcpyHostToDevice, s->stream));
  memcpy(s->h_seg, offsets, sizeof(int64_t) * (size_t)(s->n_seg + 1));
  QX_CUDA(cudaMemcpyAsync(s->seg[c], s->h_seg, sizeof(int64_t) * (size_t)(s->n_seg + 1), cudaMemcpyHostToDevice,
                          s->stream));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  s->exact = true;
  s->ub_total = total;
  s->ub_seg = 0;
  for (int g = 0; g < s->n_seg; ++g) s->ub_seg = std::max(s->ub_seg, offsets[g + 1] - offsets[g]);
  return QX_OK;
}

extern "C" int qx_store_download_wide(qx_store* s, int64_t* offsets, uint64_t* words, double* lambdas,
                                      int64_t cap_terms) {
  QX_REQUIRE(s && offsets, "NULL argument");
  QX_REQUIRE(s->n_words > 1, "store has one-word keys: use qx_store_download");
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  memcpy(offsets, s->h_seg, sizeof(int64_t) * (size_t)(s->n_seg + 1));
  const int64_t total = s->h_seg[s->n_seg];
  if (words == nullptr && lambdas == nullptr) return QX_OK;
  QX_REQUIRE(cap_terms >= total, "download buffer holds %lld terms, store has %lld", (long long)cap_terms,
             (long long)total);
  QX_CUDA(cudaSetDevice(s->device));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  const int W = s->n_words;
  const Planes pl = planes_of(s, s->cur);
  if (total > 0 && words) {
    std::vector<u64> plane((size_t)total);
    for (int w = 0; w < W; ++w) {
      QX_CUDA(cudaMemcpy(plane.data(), pl.p[w], sizeof(u64) * (size_t)total, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < total; ++i) words[(size_t)i * W + w] = plane[(size_t)i];
    }
  }
  if (total > 0 && lambdas)
    QX_CUDA(cudaMemcpy(lambdas, s->lam[s->cur], sizeof(double) * (size_t)total, cudaMemcpyDeviceToHost));
  return QX_OK;
}

extern "C" int qx_store_words(qx_store* s, int32_t* n_words) {
  QX_REQUIRE(s && n_words, "NULL argument");
  *n_words = s->n_words;
  return QX_OK;
}

// ---- compaction onto the support (the grouped operator step above 32 qubits) ---------------------
// The reference runs v2/v3 operators at any width with big-int indices (stabilizer.py:40-59,
// 289-322).  A branching operator only ever acts on the digits a term HAS, and the circuits that
// are feasible above 32 qubits keep their generators on few qubits.  A generator none of whose
// terms has a digit on a qubit the operator touches is not changed by it at all; when the support
// of the OTHER generators is at most 32 qubits wide, their terms are packed into one-word keys over
// those qubits -- ascending qubit order, so the order of the words is kept -- the one-word
// operator step runs on them (grouped / bucketed / one-launch paths, all of it), and the result is
// spread back between the untouched generators.  Identity digits contribute a factor of exactly 1
// and no branch, so the coefficients are the reference's bit for bit.
namespace {

struct QubitMap {
  int n_sel;
  int wide_pos[QX_MAX_QUBITS];     // bit position of selected qubit j in the wide key (j ascending = qubit ascending)
};

// one CTA per segment: OR of the support masks of its terms, n_words words
__global__ void __launch_bounds__(kThreads)
k_wide_support(Planes pl, const int64_t* __restrict__ seg, int n_words, u64* __restrict__ out) {
  __shared__ u64 s_acc[kThreads / 32];
  const int g = blockIdx.x;
  const int64_t lo = seg[g], hi = seg[g + 1];
  for (int w = 0; w < n_words; ++w) {
    u64 acc = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) acc |= support_mask(pl.p[w][i]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc |= __shfl_xor_sync(QX_FULL_MASK, acc, d);
    if (lane_id() == 0) s_acc[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      u64 all = 0;
      for (int i = 0; i < kThreads / 32; ++i) all |= s_acc[i];
      out[(size_t)g * n_words + w] = all;
    }
    __syncthreads();
  }
}

// index of the segment that holds term i (offsets ascending, empty segments allowed)
__device__ __forceinline__ int segment_holding(const int64_t* off, int n_seg, int64_t i) {
  int lo = 0, hi = n_seg;                       // off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// narrow term i (offsets n_off: taken segments only, the others empty) <- wide term
__global__ void __launch_bounds__(kThreads)
k_wide_compact(Planes in, const double* __restrict__ lam_in, const int64_t* __restrict__ w_off,
               const int64_t* __restrict__ n_off, int n_seg, int n_words, u64* __restrict__ keys_out,
               double* __restrict__ lam_out, int* __restrict__ error, const __grid_constant__ QubitMap map) {
  const int64_t total = n_off[n_seg];
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < total; i += (int64_t)gridDim.x * kThreads) {
    const int g = segment_holding(n_off, n_seg, i);
    const int64_t src = w_off[g] + (i - n_off[g]);
    u64 k[kMaxWords];
    for (int w = 0; w < n_words; ++w) k[w] = in.p[w][src];
    u64 out = 0;
    for (int j = 0; j < map.n_sel; ++j) {
      const int pos = map.wide_pos[j];
      const u64 d = (k[pos >> 6] >> (pos & 63)) & 3ull;
      k[pos >> 6] &= ~(3ull << (pos & 63));
      out |= d << (2 * (map.n_sel - 1 - j));
    }
    u64 rest = 0;
    for (int w = 0; w < n_words; ++w) rest |= k[w];
    if (rest) atomicExch(error, 1);                 // a digit outside the selection
    keys_out[i] = out;
    lam_out[i] = lam_in[src];
  }
}

// new wide term i (offsets o_off) <- the one-word store's term (taken segments) or the old wide term
__global__ void __launch_bounds__(kThreads)
k_wide_expand(const u64* __restrict__ keys_in, const double* __restrict__ lam_in, const int64_t* __restrict__ n_off,
              Planes old, const double* __restrict__ lam_old, const int64_t* __restrict__ w_off,
              const int64_t* __restrict__ o_off, const unsigned char* __restrict__ take, int n_seg, int n_words,
              Planes out, double* __restrict__ lam_out, const __grid_constant__ QubitMap map) {
  const int64_t total = o_off[n_seg];
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < total; i += (int64_t)gridDim.x * kThreads) {
    const int g = segment_holding(o_off, n_seg, i);
    const int64_t r = i - o_off[g];
    if (take[g]) {
      u64 k[kMaxWords];
      for (int w = 0; w < n_words; ++w) k[w] = 0;
      const u64 key = keys_in[n_off[g] + r];
      for (int j = 0; j < map.n_sel; ++j) {
        const int pos = map.wide_pos[j];
        k[pos >> 6] |= ((key >> (2 * (map.n_sel - 1 - j))) & 3ull) << (pos & 63);
      }
      for (int w = 0; w < n_words; ++w) out.p[w][i] = k[w];
      lam_out[i] = lam_in[n_off[g] + r];
    } else {
      for (int w = 0; w < n_words; ++w) out.p[w][i] = old.p[w][w_off[g] + r];
      lam_out[i] = lam_old[w_off[g] + r];
    }
  }
}

int fill_map(const qx_store* wide, const int32_t* qubits, int32_t n_sel, QubitMap* map) {
  QX_REQUIRE(qubits && n_sel >= 1 && n_sel <= QX_MAX_QUBITS, "need 1..%d selected qubits, got %d", QX_MAX_QUBITS, n_sel);
  map->n_sel = n_sel;
  for (int j = 0; j < n_sel; ++j) {
    QX_REQUIRE(qubits[j] >= 0 && qubits[j] < wide->n_qubits && (j == 0 || qubits[j] > qubits[j - 1]),
               "selected qubits must ascend within [0, %d)", wide->n_qubits);
    map->wide_pos[j] = 2 * (wide->n_qubits - 1 - qubits[j]);
  }
  return QX_OK;
}

int grid_for(const qx_store* s, int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((total + kThreads - 1) / kThreads, (int64_t)s->sm_count * 8));
}

int check_pair(const qx_store* wide, const qx_store* narrow, int32_t n_sel, const uint8_t* take) {
  QX_REQUIRE(wide && narrow && take, "NULL argument");
  QX_REQUIRE(narrow->n_words == 1 && narrow->n_qubits == n_sel && narrow->n_seg == wide->n_seg &&
                 narrow->device == wide->device,
             "the one-word store must have %d qubits and %d segments on device %d", n_sel, wide->n_seg, wide->device);
  QX_REQUIRE(!wide->narrow_keys && !narrow->narrow_keys, "a store was left with narrow keys for download");
  return QX_OK;
}

}  // namespace

extern "C" int qx_store_support(qx_store* s, uint64_t* words) {
  QX_REQUIRE(s && words, "NULL argument");
  QX_REQUIRE(!s->narrow_keys, "qx_store_support: the store was left with narrow keys for download");
  QX_CUDA(cudaSetDevice(s->device));
  const size_t bytes = 8 * (size_t)s->n_words * (size_t)s->n_seg;
  QX_TRY(qx_store_scratch(s, (int64_t)bytes));
  k_wide_support<<<s->n_seg, kThreads, 0, s->stream>>>(planes_of(s, s->cur), s->seg[s->cur], s->n_words,
                                                      reinterpret_cast<u64*>(s->scratch));
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  QX_CUDA(cudaMemcpyAsync(words, s->scratch, bytes, cudaMemcpyDeviceToHost, s->stream));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  return QX_OK;
}

extern "C" int qx_store_compact(qx_store* wide, const int32_t* qubits, int32_t n_sel, const uint8_t* take,
                                qx_store* narrow) {
  QX_TRY(check_pair(wide, narrow, n_sel, take));
  QubitMap map;
  QX_TRY(fill_map(wide, qubits, n_sel, &map));
  QX_CUDA(cudaSetDevice(wide->device));
  if (!wide->exact) QX_TRY(qx_store_refresh(wide));
  const int n_seg = wide->n_seg;
  std::vector<int64_t> n_off((size_t)n_seg + 1, 0);
  int64_t largest = 0;
  for (int g = 0; g < n_seg; ++g) {
    const int64_t len = take[g] ? wide->h_seg[g + 1] - wide->h_seg[g] : 0;
    n_off[g + 1] = n_off[g] + len;
    largest = std::max(largest, len);
  }
  const int64_t total = n_off[n_seg];
  QX_TRY(qx_store_reserve(narrow, total, false));
  QX_TRY(qx_store_scratch(wide, 16));
  int* error = reinterpret_cast<int*>(wide->scratch);
  QX_CUDA(cudaMemsetAsync(error, 0, 16, wide->stream));
  const int c = narrow->cur;
  QX_CUDA(cudaMemcpyAsync(narrow->seg[c], n_off.data(), sizeof(int64_t) * (size_t)(n_seg + 1), cudaMemcpyHostToDevice,
                          wide->stream));
  if (total > 0) {
    k_wide_compact<<<grid_for(wide, total), kThreads, 0, wide->stream>>>(
        planes_of(wide, wide->cur), wide->lam[wide->cur], wide->seg[wide->cur], narrow->seg[c], n_seg, wide->n_words,
        narrow->keys[c], narrow->lam[c], error, map);
    qx_count_launches(1);
    QX_CUDA(cudaGetLastError());
  }
  int h_error = 0;
  QX_CUDA(cudaMemcpyAsync(&h_error, error, sizeof(int), cudaMemcpyDeviceToHost, wide->stream));
  QX_CUDA(cudaStreamSynchronize(wide->stream));      // n_off is read by the copy above; the one-word store runs on its own stream
  QX_REQUIRE(h_error == 0, "qx_store_compact: a taken term has a non-identity digit outside the selected qubits");
  memcpy(narrow->h_seg, n_off.data(), sizeof(int64_t) * (size_t)(n_seg + 1));
  narrow->exact = true;
  narrow->pack_bnd = nullptr;
  narrow->ub_total = total;
  narrow->ub_seg = largest;
  return QX_OK;
}

extern "C" int qx_store_expand(qx_store* narrow, const int32_t* qubits, int32_t n_sel, const uint8_t* take,
                               qx_store* wide) {
  QX_TRY(check_pair(wide, narrow, n_sel, take));
  QubitMap map;
  QX_TRY(fill_map(wide, qubits, n_sel, &map));
  QX_CUDA(cudaSetDevice(wide->device));
  if (!narrow->exact) QX_TRY(qx_store_refresh(narrow));
  if (!wide->exact) QX_TRY(qx_store_refresh(wide));
  QX_CUDA(cudaStreamSynchronize(narrow->stream));
  const int n_seg = wide->n_seg;
  std::vector<int64_t> o_off((size_t)n_seg + 1, 0);
  int64_t largest = 0;
  for (int g = 0; g < n_seg; ++g) {
    const int64_t len = take[g] ? narrow->h_seg[g + 1] - narrow->h_seg[g] : wide->h_seg[g + 1] - wide->h_seg[g];
    o_off[g + 1] = o_off[g] + len;
    largest = std::max(largest, len);
  }
  const int64_t total = o_off[n_seg];
  QX_TRY(qx_store_reserve(wide, std::max(total, wide->h_seg[n_seg]), true));   // both buffers: old content stays live
  const int in = wide->cur, out = wide->cur ^ 1;
  QX_TRY(qx_store_scratch(wide, (int64_t)n_seg + 64));
  unsigned char* d_take = reinterpret_cast<unsigned char*>(wide->scratch);
  QX_CUDA(cudaMemcpyAsync(d_take, take, (size_t)n_seg, cudaMemcpyHostToDevice, wide->stream));
  QX_CUDA(cudaMemcpyAsync(wide->seg[out], o_off.data(), sizeof(int64_t) * (size_t)(n_seg + 1), cudaMemcpyHostToDevice,
                          wide->stream));
  if (total > 0) {
    k_wide_expand<<<grid_for(wide, total), kThreads, 0, wide->stream>>>(
        narrow->keys[narrow->cur], narrow->lam[narrow->cur], narrow->seg[narrow->cur], planes_of(wide, in),
        wide->lam[in], wide->seg[in], wide->seg[out], d_take, n_seg, wide->n_words, planes_of(wide, out), wide->lam[out],
        map);
    qx_count_launches(1);
    QX_CUDA(cudaGetLastError());
  }
  QX_CUDA(cudaStreamSynchronize(wide->stream));       // host arrays above; the one-word store may be destroyed right away
  wide->cur = out;
  memcpy(wide->h_seg, o_off.data(), sizeof(int64_t) * (size_t)(n_seg + 1));
  wide->exact = true;
  wide->ub_total = total;
  wide->ub_seg = largest;
  return QX_OK;
}
