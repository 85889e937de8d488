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

struct PgSmem {
  u64 rkey[kPgRawCap];
  double rlam[kPgRawCap];
  u64 ckey[kPgSrcCap];
  double clam[kPgSrcCap];
  unsigned short ridx[kPgRawCap];
  unsigned short soff[kPgSrcCap + 8];
  OperatorTable tb;
  ImageTable<u64> im;
  u64 scan[kPgWarps + 1];
  u64 base;
};

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
  int64_t* flags;              // [n_seg] bit 0: did not fit, bit 1: result did not fit the host buffers
  int64_t* raw;                // [n_seg] raw branches of the generator's branching steps
  int64_t* seg;                // [n_seg + 1] offsets of the result
  int64_t* ranks;              // [rows][n_seg]
  u64* keys;                   // result terms (may be NULL): same layout as the store's
  double* lam;
  int64_t cap;
};

__global__ void __launch_bounds__(kPgThreads, 1)
k_small_circuit(const u64* __restrict__ keys_in, const double* __restrict__ lam_in,
                const int64_t* __restrict__ seg_in, int n_seg, const PgStep* __restrict__ steps, int n_steps,
                u64* __restrict__ keys_out, double* __restrict__ lam_out, int64_t* __restrict__ seg_out,
                u64* status, double eps, const __grid_constant__ PgInit init, const __grid_constant__ PgHost host) {
  extern __shared__ __align__(16) unsigned char pg_raw[];
  PgSmem& sm = *reinterpret_cast<PgSmem*>(pg_raw);
  const int g = (int)blockIdx.x;             // in-order dispatch (look-back at the very end only)
  const int tid = threadIdx.x;
  int len;
  bool bad = false;
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
    bad = len > kPgSrcCap;
    if (bad) len = 0;
    for (int e = tid; e < len; e += kPgThreads) {
      sm.ckey[e] = keys_in[start + e];
      sm.clam[e] = lam_in[start + e];
    }
  }
  __syncthreads();

  for (int si = 0; si < n_steps && !bad && len > 0; ++si) {
    const PgStep* st = steps + si;
    const int kind = st->kind;
    if (kind == PG_SORT) {
      int m = 32;
      while (m < len) m <<= 1;
      for (int e = len + tid; e < m; e += kPgThreads) sm.ckey[e] = ~0ull;
      __syncthreads();
      for (int k = 2; k <= m; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int t = tid; t < (m >> 1); t += kPgThreads) {
            const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
            const int hi = lo | j;
            const u64 ka = sm.ckey[lo], kb = sm.ckey[hi];
            if ((ka > kb) == ((lo & k) == 0)) {
              sm.ckey[lo] = kb; sm.ckey[hi] = ka;
              const double la = sm.clam[lo]; sm.clam[lo] = sm.clam[hi]; sm.clam[hi] = la;
            }
          }
          __syncthreads();
        }
      }
      continue;
    }
    // tables of the step
    {
      const u32* isrc = reinterpret_cast<const u32*>(&st->im);
      u32* idst = reinterpret_cast<u32*>(&sm.im);
      for (int i = tid; i < (int)(sizeof(ImageTable<u64>) / 4); i += kPgThreads) idst[i] = isrc[i];
      if (kind == PG_OPRUN) {
        const u32* src = reinterpret_cast<const u32*>(&st->tb);
        u32* dst = reinterpret_cast<u32*>(&sm.tb);
        for (int i = tid; i < (int)(sizeof(OperatorTable) / 4); i += kPgThreads) dst[i] = src[i];
      }
    }
    __syncthreads();
    if (kind == PG_CLIFFORD) {
      for (int e = tid; e < len; e += kPgThreads) {
        u64 out;
        if (pg_image(sm.im, sm.ckey[e], out)) sm.clam[e] = -sm.clam[e];
        sm.ckey[e] = out;
      }
      __syncthreads();
      continue;
    }
    // ---- oprun
    if (st->order && len >= 3 && len <= kPgOrdCap) {
      // the reference's string order: pattern word (branch count minus one of every digit), then word
      int m = 32;
      while (m < len) m <<= 1;
      u64* pat = sm.rkey;
      for (int e = tid; e < m; e += kPgThreads) {
        u64 p = ~0ull;
        if (e < len) {
          const u64 key = sm.ckey[e];
          p = 0;
          for (u64 sup = support_mask(key); sup;) {
            const int b = __ffsll((long long)sup) - 1;
            sup &= sup - 1;
            p |= (u64)(sm.tb.cnt[b >> 1][((key >> b) & 3ull) - 1] - 1) << b;
          }
        } else {
          sm.ckey[e] = ~0ull;
        }
        pat[e] = p;
      }
      __syncthreads();
      for (int k = 2; k <= m; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int t = tid; t < (m >> 1); t += kPgThreads) {
            const int a = ((t & ~(j - 1)) << 1) | (t & (j - 1));
            const int b = a | j;
            const u64 pa = pat[a], pb = pat[b], ka = sm.ckey[a], kb = sm.ckey[b];
            const bool greater = pa > pb || (pa == pb && ka > kb);
            if (greater == ((a & k) == 0)) {
              pat[a] = pb; pat[b] = pa;
              sm.ckey[a] = kb; sm.ckey[b] = ka;
              const double la = sm.clam[a]; sm.clam[a] = sm.clam[b]; sm.clam[b] = la;
            }
          }
          __syncthreads();
        }
      }
    }
    // branch counts -> exclusive raw offsets (consecutive sources per thread)
    const int per = (len + kPgThreads - 1) / kPgThreads;
    const int e0 = tid * per, e1 = min(len, e0 + per);
    u64 mine = 0;
    for (int e = e0; e < e1; ++e) mine += branch_count(sm.ckey[e], sm.tb.cnt);
    u64 total;
    u64 run = pg_block_exclusive_sum<u64>(mine, sm.scan, total);
    if (total > (u64)kPgRawCap) {
      bad = true;
      break;
    }
    for (int e = e0; e < e1; ++e) {
      sm.soff[e] = (unsigned short)run;
      run += branch_count(sm.ckey[e], sm.tb.cnt);
    }
    if (tid == 0) sm.soff[len] = (unsigned short)total;
    raw_sum += total;
    __syncthreads();
    const int raw = (int)total;
    int m = 32;
    while (m < raw) m <<= 1;
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
        for (u64 mask = support_mask(key); mask;) {
          const int bit = __ffsll((long long)mask) - 1;
          mask &= mask - 1;
          const u32 c = sm.tb.cnt[bit >> 1][(u32)((key >> bit) & 3ull) - 1u];
          const u32 q = b / c;
          picks |= (u64)(b - q * c) << bit;
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
          v = __dmul_rn(v, sm.tb.w[p][d][pick]);
          const u32 ax = sm.tb.axis[p][d][pick];
          compose<u64>(out, ex, sm.im.img[p][ax - 1], sm.im.imx[p][ax - 1], sm.im.e[p][ax - 1]);
        }
        if (composed_sign<u64>(out, ex)) v = -v;     // sign flips are exact
      }
      sm.rkey[r] = out;
      sm.rlam[r] = v;
      sm.ridx[r] = (unsigned short)r;
    }
    __syncthreads();
    // bitonic network on (key, raw position): equal keys stay in raw order, padding ends up last
    for (int k = 2; k <= m; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = tid; t < (m >> 1); t += kPgThreads) {
          const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
          const int hi = lo | j;
          const u64 ka = sm.rkey[lo], kb = sm.rkey[hi];
          const unsigned short ia = sm.ridx[lo], ib = sm.ridx[hi];
          const bool greater = ka > kb || (ka == kb && ia > ib);
          if (greater == ((lo & k) == 0)) {
            sm.rkey[lo] = kb; sm.rkey[hi] = ka;
            sm.ridx[lo] = ib; sm.ridx[hi] = ia;
          }
        }
        __syncthreads();
      }
    }
    // run sums (sequential, raw order), drop rule, ordered compaction row by row into the
    // generator's own arrays
    const int rows = (raw + kPgThreads - 1) / kPgThreads;
    int kept_before = 0;
    for (int r = 0; r < rows; ++r) {
      const int e = r * kPgThreads + tid;
      bool kept = false;
      u64 key = 0;
      double sum = 0.0;
      if (e < raw) {
        key = sm.rkey[e];
        if (e == 0 || sm.rkey[e - 1] != key) {
          sum = sm.rlam[sm.ridx[e]];
          for (int j = e + 1; j < raw && sm.rkey[j] == key; ++j) sum += sm.rlam[sm.ridx[j]];
          kept = fabs(sum) >= eps;
        }
      }
      int row_total;
      const int excl = pg_block_exclusive_sum<int>(kept ? 1 : 0, sm.scan, row_total);
      const int pos = kept_before + excl;
      if (kept && pos < kPgSrcCap) {
        sm.ckey[pos] = key;
        sm.clam[pos] = sum;
      }
      kept_before += row_total;
    }
    if (tid == 0) host.ranks[(int64_t)st->rank_row * n_seg + g] = kept_before;
    if (kept_before > kPgSrcCap) {
      bad = true;
      break;
    }
    len = kept_before;
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
    host.flags[g] = (bad ? 1 : 0) | (to_host ? 0 : 2);
    host.raw[g] = (int64_t)raw_sum;
  }
}
