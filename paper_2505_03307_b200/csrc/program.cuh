// N1: the WHOLE circuit in one launch for stores that stay small.
//
// Configs 1, 2, 3, 5 never hold more than a few thousand terms per generator: their cost is
// launches and host round trips (C5 in v3: 61 launches, one read-back per branching operator).
// The steps a circuit plan replays on the device do not depend on the terms, only on the gate
// list (engine._compile_operators / _compile_v1): a Clifford run, a branching operator with the
// run behind it folded in (+ the reference's source order in v3), a final re-sort.  So the plan
// is compiled ONCE into a device-resident step list (qx_program_create: operator tables and the
// images of the single-digit words under every run) and one kernel walks it: one CTA per
// generator -- generators never interact (reference engine.py:113-116) -- with the generator's
// terms in shared memory from init_z to the canonical result:
//   clifford  image composition of every term's digits (expand.cuh), in place;
//   oprun     [v3: sources into the reference's string order, pattern word then word,
//             stabilizer.py:294-296]  branch counts + scan, raw terms (products qubit 0 first,
//             stabilizer.py:311-319; images of the run composed in), bitonic sort on (key, raw
//             position), in-order run sums, drop rule |sum| >= eps (stabilizer.py:336), compaction;
//             the generator's rank after the merge goes into one row of a device table;
//   sort      canonical order after a run that is not behind a branching operator.
// The ranks table, the offsets and one status word are read back ONCE at the end; the host
// replays its own bookkeeping (rank trace, update counts, collapse message with generator and
// step, engine.py:148-152) against the recorded ranks.  Everything is the same arithmetic in the
// same order as the step-by-step kernels (k_small_operator, k_order_by_pattern, k_clifford_run),
// so results are bit-identical to them.  A generator that outgrows shared memory at any step
// (more than kPgSrcCap terms, more than kPgRawCap raw branches) flags the run as "did not fit":
// the store is untouched (the kernel reads one buffer and writes the other) and the caller takes
// the step-by-step path.
#pragma once

constexpr int kPgThreads = 512;
constexpr int kPgWarps = kPgThreads / 32;
constexpr int kPgSrcCap = 4096;                  // terms of a generator between steps
constexpr int kPgRawCap = QX_SMALL_MAX;          // raw branches of one operator step (8192)
constexpr int kPgOrdCap = kOrdCap;               // k_order_by_pattern leaves longer segments alone

enum { PG_CLIFFORD = 0, PG_OPRUN = 1, PG_SORT = 2 };

struct __align__(16) PgStep {
  int kind;
  int order;            // oprun: 1 = sources into (pattern, word) order first (v3)
  int rank_row;         // oprun: row of the ranks table
  int pad;
  OperatorTable tb;     // oprun
  ImageTable<u64> im;   // clifford, oprun (identity images: no run behind the operator)
};

template <int kSrc, int kRaw>
struct PgSmemT {
  static constexpr int kSrcCap = kSrc, kRawCap = kRaw;
  u64 rkey[kRaw];
  double rlam[kRaw];
  u64 ckey[kSrc];
  double clam[kSrc];
  unsigned short ridx[kRaw];
  unsigned short soff[kSrc + 8];
  PgStep st;                   // the step being executed (header, operator table, images)
  u64 scan[kPgWarps + 1];
  u64 base;
  u32 kept_tab[(kRaw + kPgThreads - 1) / kPgThreads * kPgWarps];
  u32 kept_total;
  u64 bmask;
  int fast;
};

// Two sizes: the full one fills an SM's shared memory (one CTA per SM, and the launch switches the
// SM's shared-memory carve-out: ~10 us on an otherwise idle GPU); circuits whose generators stay
// below 256 terms (configs 1, 2, 3) take the small one.
typedef PgSmemT<kPgSrcCap, kPgRawCap> PgSmem;
typedef PgSmemT<256, 512> PgSmemSmall;
static_assert(sizeof(PgSmem) <= 227 * 1024, "one CTA's shared memory");

template <typename T>
__device__ __forceinline__ T pg_block_exclusive_sum(T v, u64* scan, T& total) {
  const int warp = threadIdx.x >> 5;
  T incl = warp_inclusive_sum(v);
  if (lane_id() == 31) scan[warp] = (u64)incl;
  __syncthreads();
  if (warp == 0) {
    u64 w = lane_id() < (u32)kPgWarps ? scan[lane_id()] : 0ull;
    const u64 wi = warp_inclusive_sum(w);
    if (lane_id() < (u32)kPgWarps) scan[lane_id()] = wi - w;
    if (lane_id() == 31) scan[kPgWarps] = wi;
  }
  __syncthreads();
  const T out = (T)scan[warp] + incl - v;
  total = (T)scan[kPgWarps];
  __syncthreads();
  return out;
}

// Bitonic network over the m = 2^x >= 32 pairs (rkey[e], ridx[e]) in shared memory, ascending by
// key, ties by index (a stable sort of whatever the indices stand for).  All three orderings of
// the kernel go through it; the payloads are gathered through the sorted indices afterwards.
//   * pairs at distance <= 32 lie inside one 64-element chunk, and a chunk always belongs to the
//     same warp: those substeps (all of the phases k <= 64, the last six of every later phase) run
//     warp by warp with __syncwarp only -- m = 8192 costs 36 CTA barriers instead of 91;
//   * a thread's compare-exchanges of one substep are independent: their loads are issued in
//     batches before the first compare (the network is latency-bound: one CTA per SM, 16 warps).
constexpr int kPgBatch = 4;

// compare-exchange of the pairs t, t + stride, ... (kPgBatch of them, those below `limit`) of the
// substep (k, j); pair t of a substep touches lo = t with a zero inserted at bit log2(j), hi = lo | j
template <typename SM>
__device__ __forceinline__ void pg_cmpxchg_batch(SM& sm, int t0, int stride, int limit, int k, int j) {
  u64 ka[kPgBatch], kb[kPgBatch];
  unsigned short ia[kPgBatch], ib[kPgBatch];
#pragma unroll
  for (int i = 0; i < kPgBatch; ++i) {
    const int t = t0 + i * stride;
    if (t < limit) {
      const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
      ka[i] = sm.rkey[lo];
      kb[i] = sm.rkey[lo | j];
      ia[i] = sm.ridx[lo];
      ib[i] = sm.ridx[lo | j];
    }
  }
#pragma unroll
  for (int i = 0; i < kPgBatch; ++i) {
    const int t = t0 + i * stride;
    if (t < limit) {
      const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
      const bool greater = ka[i] > kb[i] || (ka[i] == kb[i] && ia[i] > ib[i]);
      if (greater == ((lo & k) == 0)) {
        sm.rkey[lo] = kb[i];
        sm.rkey[lo | j] = ka[i];
        sm.ridx[lo] = ib[i];
        sm.ridx[lo | j] = ia[i];
      }
    }
  }
}

// Stable LSD radix sort of the first `count` pairs (rkey[e], ridx[e] == e) for the large cases: the
// bitonic network does m/2 * log2(m) * (log2(m) + 1) / 2 compare-exchanges (3.7e5 at 8192 elements,
// 37 us on one SM), a byte-wise LSD pass touches every element twice and only the bytes that differ
// need a pass.  Only the 16-bit indices move between the passes (keys are read through them); the
// keys are brought into the sorted order once at the end, so the state left behind is the
// network's: rkey ascending, ridx = where each pair came from, ties in input order (LSD is stable).
// A pass: every warp owns a contiguous block of the list and walks it 32 elements at a time --
// MATCH.ANY gives each element its rank among the equal digits of its round, the round's leader of
// a digit bumps the warp's private count -- then the counts are scanned over (digit, warp) and a
// second walk scatters.  `scratch`: 64 KB that is dead during the sort (the generator's own arrays
// while its raw list is sorted, the raw coefficients while its terms are).
template <typename SM>
__device__ __noinline__ void pg_radix_sort(SM& sm, int count, void* scratch, int key_bits) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned short* idx2 = reinterpret_cast<unsigned short*>(scratch);               // count
  unsigned short* off = idx2 + SM::kRawCap;                                        // count
  u32* whist = reinterpret_cast<u32*>(off + SM::kRawCap);                          // [kPgWarps][256]
  u32* flag = whist + kPgWarps * 256;
  const int per_warp = ((count + kPgWarps - 1) / kPgWarps + 31) & ~31;
  const int w_lo = warp * per_warp, w_hi = min(count, w_lo + per_warp);
  unsigned short* cur = sm.ridx;
  unsigned short* nxt = idx2;
  for (int shift = 0; shift < key_bits; shift += 8) {
    for (int i = tid; i < kPgWarps * 256; i += kPgThreads) whist[i] = 0u;
    if (tid == 0) *flag = 0u;
    __syncthreads();
    u32* mine = whist + warp * 256;
    for (int e0 = w_lo; e0 < w_hi; e0 += 32) {
      const int e = e0 + lane;
      const bool valid = e < w_hi;
      const u32 d = valid ? (u32)(sm.rkey[cur[e]] >> shift) & 255u : 256u + (u32)lane;
      const u32 peers = __match_any_sync(QX_FULL_MASK, d);
      const int leader = __ffs(peers) - 1;
      u32 old = 0;
      if (valid && lane == leader) {
        old = mine[d];
        mine[d] = old + __popc(peers);
      }
      old = __shfl_sync(QX_FULL_MASK, old, leader);
      if (valid) off[e] = (unsigned short)(old + __popc(peers & lanemask_lt()));
      __syncwarp();
    }
    __syncthreads();
    // digit totals -> exclusive start of every (digit, warp) bin; a pass whose digit is the same
    // for every element moves nothing and is skipped
    u32 tot = 0;
    if (tid < 256)
      for (int w = 0; w < kPgWarps; ++w) tot += whist[w * 256 + tid];
    if (tid < 256 && tot == (u32)count) *flag = 1u;
    u32 total_all;
    u32 run = pg_block_exclusive_sum<u32>(tid < 256 ? tot : 0u, sm.scan, total_all);
    const bool skip = *flag != 0u;                // uniform: read behind the scan's barriers ...
    __syncthreads();                              // ... and in front of the next pass, which clears it
    if (skip) continue;
    if (tid < 256) {
      for (int w = 0; w < kPgWarps; ++w) {
        const u32 c = whist[w * 256 + tid];
        whist[w * 256 + tid] = run;
        run += c;
      }
    }
    __syncthreads();
    for (int e0 = w_lo; e0 < w_hi; e0 += 32) {
      const int e = e0 + lane;
      if (e < w_hi) {
        const unsigned short from = cur[e];
        const u32 d = (u32)(sm.rkey[from] >> shift) & 255u;
        nxt[mine[d] + off[e]] = from;
      }
    }
    __syncthreads();
    unsigned short* t = cur;
    cur = nxt;
    nxt = t;
  }
  // keys into the sorted order through the scratch block, indices into their home
  u64* tmp = reinterpret_cast<u64*>(scratch);
  if (cur != sm.ridx) {
    // the scratch block is about to hold the keys: move the indices first
    unsigned short hold[(SM::kRawCap + kPgThreads - 1) / kPgThreads];
#pragma unroll
    for (int i = 0; i < (SM::kRawCap + kPgThreads - 1) / kPgThreads; ++i) {
      const int e = tid + i * kPgThreads;
      hold[i] = e < count ? cur[e] : (unsigned short)0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < (SM::kRawCap + kPgThreads - 1) / kPgThreads; ++i) {
      const int e = tid + i * kPgThreads;
      if (e < count) sm.ridx[e] = hold[i];
    }
    __syncthreads();
  }
  for (int e = tid; e < count; e += kPgThreads) tmp[e] = sm.rkey[sm.ridx[e]];
  __syncthreads();
  for (int e = tid; e < count; e += kPgThreads) sm.rkey[e] = tmp[e];
  __syncthreads();
}

// count: the real pairs (the rest up to m, a power of two, is padding that sorts last);
// scratch / key_bits: see pg_radix_sort (scratch may be NULL: network only)
template <typename SM>
__device__ __noinline__ void pg_sort_pairs(SM& sm, int m, int count, void* scratch, int key_bits) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if constexpr (SM::kRawCap >= 8192) {
    if (m >= 1024 && scratch != nullptr) {
      pg_radix_sort(sm, count, scratch, key_bits);
      return;
    }
  }
  if (m <= 128) {
    // a handful of terms (configs 1, 2, 3 never leave this branch): every element counts the
    // elements in front of it -- m broadcast reads, two barriers, no network.  Callers hand the
    // pairs over with ridx[e] == e, so ties go by position.
    u64 mine = 0;
    int rank = 0;
    if (tid < m) {
      mine = sm.rkey[tid];
#pragma unroll 8
      for (int j = 0; j < m; ++j) {
        const u64 kj = sm.rkey[j];
        rank += (kj < mine || (kj == mine && j < tid)) ? 1 : 0;
      }
    }
    __syncthreads();
    if (tid < m) {
      sm.rkey[rank] = mine;
      sm.ridx[rank] = (unsigned short)tid;
    }
    __syncthreads();
    return;
  }
  const int pairs = m >> 1;
  // pair index t = 32 * chunk + lane covers chunk `chunk` of 64 elements (m >= 64); for m = 32 the
  // first half-warp covers the only chunk
  auto warp_part = [&](int k_lo, int k_hi) {
    for (int k = k_lo; k <= k_hi; k <<= 1) {
      for (int j = min(k >> 1, 32); j > 0; j >>= 1) {
        for (int t0 = warp * 32 + lane; t0 < pairs; t0 += 32 * kPgWarps * kPgBatch)
          pg_cmpxchg_batch(sm, t0, 32 * kPgWarps, pairs, k, j);
        __syncwarp();
      }
    }
  };
  warp_part(2, min(m, 64));
  __syncthreads();
  for (int k = 128; k <= m; k <<= 1) {
    for (int j = k >> 1; j >= 64; j >>= 1) {
      for (int t0 = tid; t0 < pairs; t0 += kPgThreads * kPgBatch) pg_cmpxchg_batch(sm, t0, kPgThreads, pairs, k, j);
      __syncthreads();
    }
    warp_part(k, k);
    __syncthreads();
  }
}

// the generator's terms into the order of the sorted indices (payload gather behind pg_sort_pairs);
// take_keys: the sorted rkey ARE the new keys, otherwise they are gathered like the coefficients
template <typename SM>
__device__ __forceinline__ void pg_gather_terms(SM& sm, int len, bool take_keys) {
  const int tid = threadIdx.x;
  for (int e = tid; e < len; e += kPgThreads) {
    const int from = sm.ridx[e];
    sm.rlam[e] = sm.clam[from];
    if (!take_keys) sm.rkey[e] = sm.ckey[from];
  }
  __syncthreads();
  for (int e = tid; e < len; e += kPgThreads) {
    sm.ckey[e] = sm.rkey[e];
    sm.clam[e] = sm.rlam[e];
  }
  __syncthreads();
}

// canonical order of the generator's terms (keys are unique)
template <typename SM>
__device__ __forceinline__ void pg_sort_terms(SM& sm, int len, int key_bits) {
  const int tid = threadIdx.x;
  int m = 32;
  while (m < len) m <<= 1;
  for (int e = tid; e < m; e += kPgThreads) {
    sm.rkey[e] = e < len ? sm.ckey[e] : ~0ull;
    sm.ridx[e] = (unsigned short)e;
  }
  __syncthreads();
  pg_sort_pairs(sm, m, len, sm.rlam, key_bits);        // the raw coefficients are dead here
  pg_gather_terms(sm, len, true);
}

// image of one term under the step's run: digits composed qubit 0 first; returns the sign flip
__device__ __forceinline__ u32 pg_image(const ImageTable<u64>& im, u64 key, u64& out) {
  u64 w = 0;
  u32 ex = 0;
  for (u64 mask = support_mask(key); mask;) {
    const int bit = 63 - __clzll((long long)mask);
    mask ^= 1ull << bit;
    const int p = bit >> 1;
    const u32 ax = (u32)((key >> bit) & 3ull);
    compose<u64>(w, ex, im.img[p][ax - 1], im.imx[p][ax - 1], im.e[p][ax - 1]);
  }
  out = w;
  return composed_sign<u64>(w, ex);
}

// Generators that start as single Z words (init_z, stabilizer.py:169-174) are made in the kernel:
// no upload in front of the launch.
struct PgInit {
  int on;                      // 0: evolve the store's content
  int n_qubits;
  int qubit[QX_MAX_QUBITS];    // generator g = Z on qubit[g]
};

// What the host reads, written by the kernel straight into page-locked host memory (UVA): no
// read-back launch, no copy-engine round trip -- the stream synchronize is the only wait.
struct PgHost {
  int64_t* flags;              // [n_seg] bit 0: did not fit, bit 1: result did not fit the host buffers, bits 8..: the step that did not fit
  int64_t* raw;                // [n_seg] raw branches of the generator's branching steps
  int64_t* seg;                // [n_seg + 1] offsets of the result
  int64_t* ranks;              // [rows][n_seg]
  int64_t* clock;              // [2][n_seg] %globaltimer at the start and the end of the generator's CTA
  u64* keys;                   // result terms (may be NULL): same layout as the store's
  double* lam;
  int64_t cap;
};

template <typename SM>
__global__ void __launch_bounds__(kPgThreads, 1)
k_small_circuit(const u64* __restrict__ keys_in, const double* __restrict__ lam_in,
                const int64_t* __restrict__ seg_in, int n_seg, const PgStep* __restrict__ steps, int n_steps,
                u64* __restrict__ keys_out, double* __restrict__ lam_out, int64_t* __restrict__ seg_out,
                u64* status, double eps, const __grid_constant__ PgInit init, const __grid_constant__ PgHost host) {
  extern __shared__ __align__(16) unsigned char pg_raw[];
  SM& sm = *reinterpret_cast<SM*>(pg_raw);
  constexpr int kSrcCap = SM::kSrcCap, kRawCap = SM::kRawCap;
  const int g = qx_tile_id(reinterpret_cast<u32*>(status + n_seg));   // in-order dispatch, see qx_device.cuh (status[n_seg]: a zeroed spare word)
  const int tid = threadIdx.x;
  long long t_start = 0;
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int key_bits = 2 * init.n_qubits;    // bits of a word that can be set
  int len;
  bool bad = false;
  int bad_step = 0;                          // the step that did not fit (reported to the host)
  bool sorted = init.on != 0;                // the terms are in word order (a single Z word is)
  u64 raw_sum = 0;
  if (init.on) {
    len = 1;
    if (tid == 0) {
      sm.ckey[0] = 3ull << (2 * (init.n_qubits - 1 - init.qubit[g]));
      sm.clam[0] = 1.0;
    }
  } else {
    const int64_t start = seg_in[g];
    len = (int)min((int64_t)0x7fffffff, seg_in[g + 1] - start);
    bad = len > kSrcCap;
    if (bad) len = 0;
    for (int e = tid; e < len; e += kPgThreads) {
      sm.ckey[e] = keys_in[start + e];
      sm.clam[e] = lam_in[start + e];
    }
  }
  __syncthreads();

  // The record of a step (16-byte header, operator table, images: 4.3 KB) is loaded into
  // registers one step AHEAD and only stored to shared memory when its step begins: the global
  // round trip hides behind the previous step instead of standing in front of every step.
  constexpr int kStepWords = (int)(sizeof(PgStep) / 4);
  constexpr int kPre = (kStepWords + kPgThreads - 1) / kPgThreads;
  u32 pre[kPre];
  auto prefetch = [&](int si) {
    const u32* src = reinterpret_cast<const u32*>(steps + si);
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      const int at = tid + i * kPgThreads;
      pre[i] = at < kStepWords ? __ldg(src + at) : 0u;
    }
  };
  if (n_steps > 0) prefetch(0);
  __syncthreads();

  for (int si = 0; si < n_steps && !bad && len > 0; ++si) {
    {
      u32* dst = reinterpret_cast<u32*>(&sm.st);
#pragma unroll
      for (int i = 0; i < kPre; ++i) {
        const int at = tid + i * kPgThreads;
        if (at < kStepWords) dst[at] = pre[i];
      }
    }
    __syncthreads();
    if (si + 1 < n_steps) prefetch(si + 1);
    const PgStep* st = &sm.st;
    const int kind = st->kind;
    if (kind == PG_SORT) {
      pg_sort_terms(sm, len, key_bits);
      sorted = true;
      continue;
    }
    if (kind == PG_CLIFFORD) {
      for (int e = tid; e < len; e += kPgThreads) {
        u64 out;
        if (pg_image(sm.st.im, sm.ckey[e], out)) sm.clam[e] = -sm.clam[e];
        sm.ckey[e] = out;
      }
      __syncthreads();
      sorted = false;
      continue;
    }
    // ---- oprun
    if (st->order && len >= 3 && len <= kPgOrdCap) {   // (the small variant never reaches the cap)
      // the reference's string order: pattern word (branch count minus one of every digit), then
      // word -- a stable sort by pattern of terms that are in word order
      if (!sorted) pg_sort_terms(sm, len, key_bits);
      int m = 32;
      while (m < len) m <<= 1;
      for (int e = tid; e < m; e += kPgThreads) {
        u64 p = ~0ull;
        if (e < len) {
          const u64 key = sm.ckey[e];
          p = 0;
          for (u64 sup = support_mask(key); sup;) {
            const int b = __ffsll((long long)sup) - 1;
            sup &= sup - 1;
            p |= (u64)(sm.st.tb.cnt[b >> 1][((key >> b) & 3ull) - 1] - 1) << b;
          }
        }
        sm.rkey[e] = p;
        sm.ridx[e] = (unsigned short)e;
      }
      __syncthreads();
      pg_sort_pairs(sm, m, len, sm.rlam, key_bits);
      pg_gather_terms(sm, len, false);
    }
    // qubits on which the operator branches at all; on the others every cell has one output axis.
    // fast: all those single weights are exactly +-1 (Clifford cells), so they only flip signs
    if (tid < 32) {
      bool br = false, unit = true;
      for (int a = 0; a < 3; ++a) {
        if (sm.st.tb.cnt[tid][a] > 1) br = true;
        else unit = unit && fabs(sm.st.tb.w[tid][a][0]) == 1.0;
      }
      u64 mine = br ? 1ull << (2 * tid) : 0ull;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) mine |= __shfl_xor_sync(QX_FULL_MASK, mine, d);
      const u32 oks = __ballot_sync(QX_FULL_MASK, br || unit);
      if (tid == 0) {
        sm.bmask = mine;
        sm.fast = oks == 0xffffffffu ? 1 : 0;
      }
    }
    __syncthreads();
    const u64 bmask = sm.bmask;
    // branch counts -> exclusive raw offsets (consecutive sources per thread)
    auto branches = [&](u64 key) {
      u32 c = 1;
      for (u64 mk = support_mask(key) & bmask; mk;) {
        const int bit = __ffsll((long long)mk) - 1;
        mk &= mk - 1;
        c *= sm.st.tb.cnt[bit >> 1][((key >> bit) & 3ull) - 1];
      }
      return c;
    };
    const int per = (len + kPgThreads - 1) / kPgThreads;
    const int e0 = tid * per, e1 = min(len, e0 + per);
    u64 mine = 0;
    for (int e = e0; e < e1; ++e) mine += branches(sm.ckey[e]);
    u64 total;
    u64 run = pg_block_exclusive_sum<u64>(mine, sm.scan, total);
    if (total > (u64)kRawCap) {
      bad = true;
      bad_step = si;
      break;
    }
    for (int e = e0; e < e1; ++e) {
      sm.soff[e] = (unsigned short)run;
      run += branches(sm.ckey[e]);
    }
    if (tid == 0) sm.soff[len] = (unsigned short)total;
    raw_sum += total;
    __syncthreads();
    const int raw = (int)total;
    int m = 32;
    while (m < raw) m <<= 1;
    if (sm.fast && raw <= 4 * len) {
      // Few branches per source (near-Clifford circuits: one rotation in the operator): one thread
      // per SOURCE.  The digits the operator does not branch on contribute a fixed image and a
      // sign -- composed once per source, not once per raw term; factors on different qubits
      // commute, and multiplying by +-1 is exact wherever it happens in the product, so the
      // coefficient is bitwise lambda * w_q0 * w_q1 * ... in qubit order (stabilizer.py:311-319).
      for (int e = tid; e < len; e += kPgThreads) {
        const u64 key = sm.ckey[e];
        const double lam = sm.clam[e];
        u64 wb = 0;
        u32 eb = 0, neg = 0;
        for (u64 mk = support_mask(key) & ~bmask; mk;) {
          const int bit = 63 - __clzll((long long)mk);
          mk ^= 1ull << bit;
          const int p = bit >> 1;
          const u32 d = (u32)((key >> bit) & 3ull) - 1u;
          neg ^= sm.st.tb.w[p][d][0] < 0.0 ? 1u : 0u;
          const u32 ax = sm.st.tb.axis[p][d][0];
          compose<u64>(wb, eb, sm.st.im.img[p][ax - 1], sm.st.im.imx[p][ax - 1], sm.st.im.e[p][ax - 1]);
        }
        const u64 bm = support_mask(key) & bmask;
        const u32 r0 = sm.soff[e], r1 = sm.soff[e + 1];
        for (u32 r = r0; r < r1; ++r) {
          u32 b = r - r0;
          u64 picks = 0;
          for (u64 mk = bm; mk;) {
            const int bit = __ffsll((long long)mk) - 1;
            mk &= mk - 1;
            u32 q, pick;
            divmod_small<u32>(b, sm.st.tb.cnt[bit >> 1][(u32)((key >> bit) & 3ull) - 1u], q, pick);
            picks |= (u64)pick << bit;
            b = q;
          }
          double v = lam;
          u64 out = wb;
          u32 ex = eb;
          for (u64 mk = bm; mk;) {
            const int bit = 63 - __clzll((long long)mk);
            mk ^= 1ull << bit;
            const int p = bit >> 1;
            const u32 d = (u32)((key >> bit) & 3ull) - 1u, pick = (u32)(picks >> bit) & 3u;
            v = __dmul_rn(v, sm.st.tb.w[p][d][pick]);
            const u32 ax = sm.st.tb.axis[p][d][pick];
            compose<u64>(out, ex, sm.st.im.img[p][ax - 1], sm.st.im.imx[p][ax - 1], sm.st.im.e[p][ax - 1]);
          }
          if (composed_sign<u64>(out, ex) ^ neg) v = -v;     // sign flips are exact
          sm.rkey[r] = out;
          sm.rlam[r] = v;
          sm.ridx[r] = (unsigned short)r;
        }
      }
      for (int r = raw + tid; r < m; r += kPgThreads) {
        sm.rkey[r] = ~0ull;
        sm.rlam[r] = 0.0;
        sm.ridx[r] = (unsigned short)r;
      }
    } else {
      // raw terms: source by bisection of the offsets, picks by mixed-radix decode (lowest digit
      // fastest), product and image composition qubit 0 first (stabilizer.py:311-319)
      for (int r = tid; r < m; r += kPgThreads) {
        u64 out = ~0ull;
        double v = 0.0;
        if (r < raw) {
          int lo = 0, hi = len;                // soff[lo] <= r < soff[hi]
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if ((int)sm.soff[mid] <= r) lo = mid; else hi = mid;
          }
          const u64 key = sm.ckey[lo];
          u32 b = (u32)r - (u32)sm.soff[lo];
          u64 picks = 0;
          for (u64 mask = support_mask(key) & bmask; mask;) {
            const int bit = __ffsll((long long)mask) - 1;
            mask &= mask - 1;
            u32 q, pick;
            divmod_small<u32>(b, sm.st.tb.cnt[bit >> 1][(u32)((key >> bit) & 3ull) - 1u], q, pick);
            picks |= (u64)pick << bit;
            b = q;
          }
          v = sm.clam[lo];
          out = 0;
          u32 ex = 0;
          for (u64 mask = support_mask(key); mask;) {
            const int bit = 63 - __clzll((long long)mask);
            mask ^= 1ull << bit;
            const int p = bit >> 1;
            const u32 d = (u32)((key >> bit) & 3ull) - 1u, pick = (u32)(picks >> bit) & 3u;
            v = __dmul_rn(v, sm.st.tb.w[p][d][pick]);
            const u32 ax = sm.st.tb.axis[p][d][pick];
            compose<u64>(out, ex, sm.st.im.img[p][ax - 1], sm.st.im.imx[p][ax - 1], sm.st.im.e[p][ax - 1]);
          }
          if (composed_sign<u64>(out, ex)) v = -v;     // sign flips are exact
        }
        sm.rkey[r] = out;
        sm.rlam[r] = v;
        sm.ridx[r] = (unsigned short)r;
      }
    }
    __syncthreads();
    // bitonic network on (key, raw position): equal keys stay in raw order, padding ends up last
    pg_sort_pairs(sm, m, raw, sm.ckey, key_bits);        // the sources are dead: ckey + clam are one 64 KB block
    // run sums (sequential, raw order), drop rule, ordered compaction into the generator's own
    // arrays: kept flags of all rows first (one table of per-warp counts, scanned once), then the
    // sums again for the kept heads -- duplicates are rare, two barriers instead of one per row
    const int rows = (raw + kPgThreads - 1) / kPgThreads;      // <= kRawCap / kPgThreads = 16
    auto run_sum = [&](int e, u64 key) {
      double sum = sm.rlam[sm.ridx[e]];
      for (int j = e + 1; j < raw && sm.rkey[j] == key; ++j) sum += sm.rlam[sm.ridx[j]];
      return sum;
    };
    u32 kept_rows = 0;
    for (int r = 0; r < rows; ++r) {
      const int e = r * kPgThreads + tid;
      bool kept = false;
      if (e < raw) {
        const u64 key = sm.rkey[e];
        if (e == 0 || sm.rkey[e - 1] != key) kept = fabs(run_sum(e, key)) >= eps;
      }
      const u32 votes = __ballot_sync(QX_FULL_MASK, kept);
      if (lane_id() == 0) sm.kept_tab[r * kPgWarps + (tid >> 5)] = __popc(votes);
      if (kept) kept_rows |= 1u << r;
    }
    __syncthreads();
    if (tid < 32) {
      constexpr int kEach = ((kRawCap + kPgThreads - 1) / kPgThreads * kPgWarps + 31) / 32;     // table entries per lane
      const int n_ent = rows * kPgWarps;
      u32 loc[kEach], sum = 0;
#pragma unroll
      for (int i = 0; i < kEach; ++i) {
        const int at = tid * kEach + i;
        loc[i] = at < n_ent ? sm.kept_tab[at] : 0u;
        sum += loc[i];
      }
      u32 incl = warp_inclusive_sum(sum);
      u32 runx = incl - sum;
#pragma unroll
      for (int i = 0; i < kEach; ++i) {
        const int at = tid * kEach + i;
        if (at < n_ent) sm.kept_tab[at] = runx;
        runx += loc[i];
      }
      if (tid == 31) sm.kept_total = incl;
    }
    __syncthreads();
    const int kept_before = (int)sm.kept_total;
    for (int r = 0; r < rows; ++r) {
      const bool kept = (kept_rows >> r) & 1u;
      const u32 votes = __ballot_sync(QX_FULL_MASK, kept);
      if (kept) {
        const int e = r * kPgThreads + tid;
        const int pos = (int)sm.kept_tab[r * kPgWarps + (tid >> 5)] + __popc(votes & lanemask_lt());
        if (pos < kSrcCap) {
          const u64 key = sm.rkey[e];
          sm.ckey[pos] = key;
          sm.clam[pos] = run_sum(e, key);
        }
      }
    }
    __syncthreads();
    if (tid == 0) host.ranks[(int64_t)st->rank_row * n_seg + g] = kept_before;
    if (kept_before > kSrcCap) {
      bad = true;
      bad_step = si;
      break;
    }
    len = kept_before;
    sorted = true;
    __syncthreads();
  }
  if (bad) len = 0;
  // compact output across the generators
  if ((tid >> 5) == 0) {
    const u64 excl = lookback_exclusive(status, g, (u64)len);
    if (lane_id() == 0) sm.base = excl;
  }
  __syncthreads();
  const int64_t base = (int64_t)sm.base;
  const bool to_host = host.keys != nullptr && base + len <= host.cap;
  for (int e = tid; e < len; e += kPgThreads) {
    const u64 k = sm.ckey[e];
    const double l = sm.clam[e];
    keys_out[base + e] = k;
    lam_out[base + e] = l;
    if (to_host) {
      host.keys[base + e] = k;
      host.lam[base + e] = l;
    }
  }
  if (tid == 0) {
    seg_out[g] = base;
    host.seg[g] = base;
    if (g == n_seg - 1) {
      seg_out[n_seg] = base + len;
      host.seg[n_seg] = base + len;
    }
    host.flags[g] = (bad ? 1 : 0) | (to_host ? 0 : 2) | ((int64_t)bad_step << 8);
    host.raw[g] = (int64_t)raw_sum;
    long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    host.clock[g] = t_start;
    host.clock[n_seg + g] = t_end;
  }
}
