// a4 + a5 + a2 + a6 for operators with a large fan-out: grouped dense accumulation.
//
// The reference expands every term of a generator into its Cartesian product of branches
// (stabilizer.py:289-322 _flatten_ragged), then canonicalize sorts the raw list and sums
// duplicates (stabilizer.py:325-337).  Which raw terms can collide is known before anything is
// expanded: a single-qubit block maps input axis a to the set A(a) of output axes with non-zero
// weight; two input axes can meet on an output axis only if they are in the same connected
// component ("class") of that relation, and a class C writes into O(C) = union of A(a), a in C.
// Replace every non-identity digit of a term by its class id: terms of one generator with
// different class words never produce the same output word, terms with the same class word
// ("group") all write into the same dense box of prod_j |O(C_j)| output words ("slots").
//
// So instead of expand -> sort raw -> reduce, the large path is
//   1. class word per source term, stable segmented sort of the sources by class word;
//   2. one scan over the sorted sources: groups, their slot offsets, per-generator slot counts;
//   3. one thread per SLOT: sum over the sources of its group of lambda * prod_j w_j, factors taken
//      qubit 0 first like the reference (stabilizer.py:311-319), sources in input order; drop rule
//      |sum| >= eps (stabilizer.py:336); ordered compaction (ballot prefix + decoupled look-back);
//      the Clifford run that follows the operator is folded in as an image composition
//      (expand.cuh), so the kept terms leave the kernel conjugated, as 32-bit keys when 2n <= 32;
//   4. sort only (merge.cuh, do_reduce = false): slots are distinct words and the run is a
//      bijection, so nothing is left to sum or drop.
// The raw list is never written: HBM holds slots, not branches.  xyz_chain(10,3): 1.3e9 raw terms
// -> 3.3e6 slots; xyz_chain(16,2): every group has one source, slots = raw = 1.72e8, 27 % of
// them are dropped before the sort instead of after it, and the reduce pass disappears.
//
// A slot that no source reaches with a non-zero weight (a class whose relation is not complete)
// sums to exactly 0 and is dropped by eps > 0; with eps == 0 the caller takes the raw path.
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "bucket.cuh"
#include "expand.cuh"
#include "merge.cuh"

using namespace qxe;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPer = 8;
constexpr int kTileSlots = kThreads * kPer;      // 2048 slots (or sources) per tile
constexpr int kChunk = 8;                        // sources accumulated per round of the one-group path
constexpr int kPhiCap = 1024;                    // partial products held per round

// class id (1..3, the smallest input axis of the class) of input axis a+1 at digit position p
struct ClassIds {
  unsigned char cls[QX_MAX_QUBITS][3];
};

template <typename K>
__device__ __forceinline__ K class_word(K key, const unsigned char (*cls)[3]) {
  K m = KeyOps<K>::support(key), c = 0;
  while (m) {
    const int b = KeyOps<K>::lowest(m);
    m &= m - 1;
    c |= (K)cls[b >> 1][((u32)(key >> b) & 3u) - 1u] << b;
  }
  return c;
}

// ---- 1. class words ------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
k_class_words(const u64* __restrict__ keys, int64_t n, u64* __restrict__ cw, double* __restrict__ idx,
              const __grid_constant__ ClassIds ids) {
  __shared__ unsigned char s_cls[QX_MAX_QUBITS][3];
  for (int i = threadIdx.x; i < QX_MAX_QUBITS * 3; i += kThreads) s_cls[i / 3][i % 3] = ids.cls[i / 3][i % 3];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    cw[i] = class_word<u64>(keys[i], s_cls);
    idx[i] = __longlong_as_double(i);          // payload of the sort: moved, never computed with
  }
}

// ---- 2. groups -----------------------------------------------------------------------------
__device__ __forceinline__ u64 slots_of(u64 cw, const unsigned char (*cnt)[3]) {
  u64 m = support_mask(cw), c = 1;
  while (m) {
    const int b = __ffsll((long long)m) - 1;
    m &= m - 1;
    c *= cnt[b >> 1][((cw >> b) & 3ull) - 1];
  }
  return c;
}

// ---- 1 + 2 for few sources: one CTA does it all ------------------------------------------------
// Up to kPrepSmall sources: class words, bitonic sort on (generator, class word, input position)
// in shared memory, group heads, both scans, gathers -- one launch instead of the dozen of the
// general path (the probe of an operator costs as little as counting its raw branches).
constexpr int kPrepSmall = 1024;
constexpr int kPrepThreads = 256;

__global__ void __launch_bounds__(kPrepThreads)
k_group_prep_small(const u64* __restrict__ keys_in, const double* __restrict__ lam_in,
                   const int64_t* __restrict__ seg, int n_seg, int n, u64* __restrict__ cw_out,
                   u64* __restrict__ skey, double* __restrict__ slam, u64* __restrict__ gsrc,
                   u64* __restrict__ gslot, int64_t* __restrict__ seg_slot, u64* __restrict__ totals,
                   const __grid_constant__ ClassIds ids, const __grid_constant__ OperatorTable tb) {
  __shared__ u64 s_cw[kPrepSmall];
  __shared__ unsigned short s_seg[kPrepSmall], s_idx[kPrepSmall];
  __shared__ u64 s_slots[kPrepSmall];          // slots of a head (0 otherwise) -> exclusive prefix
  __shared__ unsigned short s_heads[kPrepSmall];   // head flag -> exclusive prefix
  __shared__ unsigned char s_cls[QX_MAX_QUBITS][3], s_cnt[QX_MAX_QUBITS][3];
  __shared__ u64 s_scan[kPrepThreads / 32 + 1];
  const int tid = threadIdx.x;
  for (int i = tid; i < QX_MAX_QUBITS * 3; i += kPrepThreads) {
    s_cls[i / 3][i % 3] = ids.cls[i / 3][i % 3];
    s_cnt[i / 3][i % 3] = tb.cnt[i / 3][i % 3];
  }
  __syncthreads();
  int m = 32;
  while (m < n) m <<= 1;
  for (int e = tid; e < m; e += kPrepThreads) {
    if (e < n) {
      s_cw[e] = class_word<u64>(keys_in[e], s_cls);
      s_seg[e] = (unsigned short)segment_of(seg, n_seg, e);
    } else {
      s_cw[e] = ~0ull;
      s_seg[e] = 0xffffu;                        // padding sorts last
    }
    s_idx[e] = (unsigned short)e;
  }
  __syncthreads();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < (m >> 1); t += kPrepThreads) {
        const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int hi = lo | j;
        const unsigned short sa = s_seg[lo], sb = s_seg[hi], ia = s_idx[lo], ib = s_idx[hi];
        const u64 ca = s_cw[lo], cb = s_cw[hi];
        const bool greater = sa != sb ? sa > sb : (ca != cb ? ca > cb : ia > ib);
        if (greater == ((lo & k) == 0)) {
          s_seg[lo] = sb; s_seg[hi] = sa;
          s_cw[lo] = cb; s_cw[hi] = ca;
          s_idx[lo] = ib; s_idx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  // heads and their slot counts; four consecutive sources per thread
  constexpr int kEach = kPrepSmall / kPrepThreads;
  u64 my_slots = 0;
  u32 my_heads = 0;
  for (int r = 0; r < kEach; ++r) {
    const int e = tid * kEach + r;
    u64 sl = 0;
    unsigned short hd = 0;
    if (e < n) {
      hd = (e == 0 || s_seg[e - 1] != s_seg[e] || s_cw[e - 1] != s_cw[e]) ? 1 : 0;
      if (hd) sl = slots_of(s_cw[e], s_cnt);
    }
    s_slots[e] = sl;
    s_heads[e] = hd;
    my_slots += sl;
    my_heads += hd;
  }
  u64 tot_s, tot_h;
  u64 ex_s = block_exclusive_sum<u64>(my_slots, s_scan, tot_s);
  u64 ex_h = block_exclusive_sum<u64>((u64)my_heads, s_scan, tot_h);
  for (int r = 0; r < kEach; ++r) {
    const int e = tid * kEach + r;
    const u64 sl = s_slots[e];
    const unsigned short hd = s_heads[e];
    s_slots[e] = ex_s;                            // first slot of the group this source opens / belongs after
    if (e < n) {
      const int j = s_idx[e];
      cw_out[e] = s_cw[e];
      skey[e] = keys_in[j];
      slam[e] = lam_in[j];
      if (hd) {
        gsrc[ex_h] = (u64)e;
        gslot[ex_h] = ex_s;
      }
    }
    ex_s += sl;
    ex_h += hd;
  }
  __syncthreads();
  // slot offset of every generator: the first slot of its first source (sources are in generator
  // order), or the next generator's / the total for an empty one
  for (int g = tid; g <= n_seg; g += kPrepThreads) {
    const int64_t first = seg[g];                 // index of its first source in INPUT order = sorted position
    seg_slot[g] = first < n ? (int64_t)s_slots[first] : (int64_t)tot_s;
  }
  if (tid == 0) {
    gsrc[tot_h] = (u64)n;
    gslot[tot_h] = tot_s;
    totals[0] = tot_h;
    totals[1] = tot_s;
  }
}

// One pass over the sources in (generator, class word) order.  A source is a group head if it
// opens a generator or its class word differs from its predecessor's.  Two exclusive scans
// (heads, slots of heads) give every group its index and its first slot.  Also gathers the
// source terms into sorted order so that the slot kernel reads them without indirection.
//   gsrc[g]  = first sorted source of group g        (gsrc[NG] = n)
//   gslot[g] = first slot of group g                 (gslot[NG] = total slots)
//   seg_slot = slot offsets of the generators        (n_seg + 1)
__global__ void __launch_bounds__(kThreads)
k_group_scan(const u64* __restrict__ cw, const double* __restrict__ idx, const u64* __restrict__ keys_in,
             const double* __restrict__ lam_in, const int64_t* __restrict__ seg, int n_seg, int64_t n,
             u64* __restrict__ skey, double* __restrict__ slam, u64* __restrict__ gsrc,
             u64* __restrict__ gslot, int64_t* __restrict__ seg_slot, u64* __restrict__ totals,
             u64* status_heads, u64* status_slots, u32* ticket, const __grid_constant__ OperatorTable tb) {
  __shared__ int s_tile;
  __shared__ u64 s_scan[kWarps + 1];
  __shared__ u64 s_base[2];
  __shared__ unsigned char s_cnt[QX_MAX_QUBITS][3];
  for (int i = threadIdx.x; i < QX_MAX_QUBITS * 3; i += kThreads) s_cnt[i / 3][i % 3] = tb.cnt[i / 3][i % 3];
  const int tile = take_ticket(ticket, &s_tile);
  const int64_t ntiles = n > 0 ? (n + kTileSlots - 1) / kTileSlots : 1;
  if (tile >= ntiles) return;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t wbase = (int64_t)tile * kTileSlots + (int64_t)warp * (32 * kPer);
  u64 pre_h[kPer], pre_s[kPer];
  u32 flags = 0;                 // bit k: head, bit 8+k: opens a generator
  u64 run_h = 0, run_s = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    u64 r = 0;
    bool head = false;
    if (i < n) {
      const u64 c = cw[i];
      const int g = segment_of(seg, n_seg, i);
      const bool opens = seg[g] == i;
      head = opens || cw[i - 1] != c;
      if (opens) flags |= 1u << (8 + k);
      if (head) {
        flags |= 1u << k;
        r = slots_of(c, s_cnt);
      }
      const int64_t j = __double_as_longlong(idx[i]);
      skey[i] = keys_in[j];
      slam[i] = lam_in[j];
    }
    const u32 votes = __ballot_sync(QX_FULL_MASK, head);
    pre_h[k] = run_h + __popc(votes & lanemask_lt());
    run_h += __popc(votes);
    const u64 inc = warp_inclusive_sum(r);
    pre_s[k] = run_s + inc - r;
    run_s += __shfl_sync(QX_FULL_MASK, inc, 31);
  }
  u64 tot_h, tot_s;
  u64 wex_h = block_exclusive_sum<u64>(lane == 0 ? run_h : 0ull, s_scan, tot_h);
  wex_h = __shfl_sync(QX_FULL_MASK, wex_h, 0);
  u64 wex_s = block_exclusive_sum<u64>(lane == 0 ? run_s : 0ull, s_scan, tot_s);
  wex_s = __shfl_sync(QX_FULL_MASK, wex_s, 0);
  if (warp == 0) {
    const u64 eh = lookback_exclusive(status_heads, tile, tot_h);
    const u64 es = lookback_exclusive(status_slots, tile, tot_s);
    if (lane == 0) {
      s_base[0] = eh;
      s_base[1] = es;
    }
  }
  __syncthreads();
  const u64 base_h = s_base[0] + wex_h, base_s = s_base[1] + wex_s;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    if (flags & (1u << k)) {
      gsrc[base_h + pre_h[k]] = (u64)i;
      gslot[base_h + pre_h[k]] = base_s + pre_s[k];
    }
    if (flags & (1u << (8 + k)))
      open_offsets(seg, seg_slot, segment_of(seg, n_seg, i), i, (int64_t)(base_s + pre_s[k]));
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) {
    const u64 ng = s_base[0] + tot_h, total = s_base[1] + tot_s;
    gsrc[ng] = (u64)n;
    gslot[ng] = total;
    totals[0] = ng;
    totals[1] = total;
    close_offsets(seg, seg_slot, n_seg, n, (int64_t)total);
  }
}
// group and generator of the first slot of every slot tile
__global__ void k_tile_groups(const u64* __restrict__ gslot, const u64* __restrict__ totals,
                              const int64_t* __restrict__ seg_slot, int n_seg,
                              int2* __restrict__ tile_info, int64_t ntiles) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntiles) {
    const u64 r0 = (u64)t * kTileSlots;
    tile_info[t] = make_int2((int)last_le(gslot, (int64_t)totals[0], r0), segment_of(seg_slot, n_seg, (int64_t)r0));
  }
}

// groups -> page-locked host memory for the planner of the bucketed step (bucket.cuh):
// [0] = groups, [1] = slots, then class word / first source / first slot of up to `cap` groups
__global__ void k_group_export(const u64* __restrict__ cw, const u64* __restrict__ gsrc, const u64* __restrict__ gslot,
                               const u64* __restrict__ totals, u64* __restrict__ host, int cap) {
  const u64 ng = totals[0];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    host[0] = ng;
    host[1] = totals[1];
  }
  if (ng > (u64)cap || (u64)i > ng) return;
  u64* h_cw = host + 2;
  u64* h_src = h_cw + (cap + 1);
  u64* h_slot = h_src + (cap + 1);
  h_src[i] = gsrc[i];
  h_slot[i] = gslot[i];
  h_cw[i] = (u64)i < ng ? cw[gsrc[i]] : 0ull;
}

// kept counts -> compact offsets (n_seg is small: one thread)
__global__ void k_counts_to_offsets(const u64* __restrict__ seg_count, int n_seg, int64_t* __restrict__ seg_out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t run = 0;
    for (int g = 0; g < n_seg; ++g) {
      seg_out[g] = run;
      run += (int64_t)seg_count[g];
    }
    seg_out[n_seg] = run;
  }
}

// ---- 3. one thread per slot ----------------------------------------------------------------
constexpr int kMaxBlocks = 512;      // blocks of one tile in the one-group path (needs L >= 4 ...)
constexpr int kFastMin = 128;        // a group part with fewer slots in a tile is worked off by the per-slot path
constexpr int kBlockedMin = 64;      // groups with at least this many sources take the factored sum
constexpr int kSrcRound = 512;       //   sources staged per round (two per thread)
constexpr int kBlockRound = 24;      //   source blocks folded per round
constexpr int kRows = 9;             // one-group path: rows of A = L * (256 / L) slots, ceil(2048 / 243) = 9
#ifndef QX_EMIT_MINB
#define QX_EMIT_MINB 5
#endif
constexpr int kHistPasses = 8;       // digit histograms kept per CTA (8 bits each, 64-bit keys)

template <typename K> struct __align__(16) HiEntry {   // per block of the tile
  double p;        // lambda * high weights of the group's first source
  K word;          // output word of the high digits
  u32 e;           // its phase exponent
};
template <typename K> struct __align__(16) LowEntry {  // per low branch of the group
  K word;
  K imx;
  u32 e;
  u32 pick;
};

template <typename K>
struct GroupSmem {
  OperatorTable tb;                  // class-expanded: cnt/axis describe the class, w may hold zeros
  ImageTable<K> im;
  HiEntry<K> hi[kMaxBlocks];
  K choice[kMaxBlocks];              // picks of the high digits, two bits per digit position
  double p_hi[kPhiCap];              // [source of the round][block]: lambda * high weights
  double low_w[kChunk + 1][27][4];   // [first source | source of the round][low branch][low digit], 32-byte rows
  LowEntry<K> low[27];
  u32 hist[sizeof(K) == 4 ? 4 : kHistPasses][QX_RADIX];   // digit counts of the kept terms (all passes of the sort)
  u64 scan[kWarps + 1];
  u64 base;
  K blk_key[kBlockRound];            // factored sum: a representative key per source block
  unsigned short blk_first[kBlockRound + 1];
  int consumed;
};

// digit = byte `which` of the key
__device__ __forceinline__ u32 digit_of(u32 key, int which) { return (key >> (8 * which)) & 255u; }
__device__ __forceinline__ u32 digit_of(u64 key, int which) { return (u32)(key >> (8 * which)) & 255u; }

// K = working word type (u32 for n <= 16), KO = type of the keys written, FUSED = compose the
// images of the Clifford run that follows (im) instead of placing the output digits.
// Persistent CTAs stride over the slot tiles.  Kept terms of generator g go to
// [seg_slot[g], seg_slot[g] + kept_g) of the output: space is handed out with one atomic per tile
// (order inside a generator is irrelevant, the sort follows; a tile-ordered compaction would
// chain every tile to its predecessor's FINISHED sums -- 34 % of the stall samples of the first
// version of this kernel, profiles/r01h).  The digit histograms of the sort that follows are
// counted here, on the keys while they are in registers (hist[g][pass][digit]).
template <typename K, typename KO, bool FUSED>
__global__ void __launch_bounds__(kThreads, sizeof(K) == 8 ? 2 : QX_EMIT_MINB)
k_group_emit(const u64* __restrict__ cw, const u64* __restrict__ skey, const double* __restrict__ slam,
             const u64* __restrict__ gsrc, const u64* __restrict__ gslot, const u64* __restrict__ totals,
             const int2* __restrict__ tile_info, const int64_t* __restrict__ seg_slot, int n_seg,
             KO* __restrict__ keys_out, double* __restrict__ lam_out, u64* __restrict__ seg_count,
             u32* __restrict__ hist, int passes, double eps, int part, int parts,
             const int64_t* __restrict__ pre_off, const double* __restrict__ pre,
             const __grid_constant__ OperatorTable tb, const __grid_constant__ ImageTable<K> im) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GroupSmem<K>& sm = *reinterpret_cast<GroupSmem<K>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
  {
    const u32* src = reinterpret_cast<const u32*>(&tb);
    u32* dst = reinterpret_cast<u32*>(&sm.tb);
    for (int i = tid; i < (int)(sizeof(OperatorTable) / 4); i += kThreads) dst[i] = src[i];
    if (FUSED) {
      const u32* isrc = reinterpret_cast<const u32*>(&im);
      u32* idst = reinterpret_cast<u32*>(&sm.im);
      for (int i = tid; i < (int)(sizeof(ImageTable<K>) / 4); i += kThreads) idst[i] = isrc[i];
    }
    for (int i = tid; i < (int)(sizeof(sm.hist) / 4); i += kThreads) (&sm.hist[0][0])[i] = 0u;
  }
  const int64_t ngroups = (int64_t)totals[0];
  const u64 total = totals[1];
  const int64_t ntiles = (int64_t)((total + kTileSlots - 1) / kTileSlots);
  // multi-GPU: this device works off the part-th of `parts` contiguous tile ranges (slots are
  // independent, so the ranges need no communication)
  const int64_t tile_lo = ntiles * part / parts, tile_hi = ntiles * (part + 1) / parts;
  int cached_group = -1;              // group whose low table is in shared memory
  int hist_seg = -1;                  // generator the shared histogram belongs to
  LowGroup<K> lg = {};
  K cwg = 0;
  u32 magic = 0;

  for (int64_t tile = tile_lo + blockIdx.x; tile < tile_hi; tile += gridDim.x) {
   const u64 t0_slot = (u64)tile * kTileSlots;
   const u64 t1_slot = min(t0_slot + (u64)kTileSlots, total);
   const int2 ti = tile_info[tile];
   int g_next = ti.x, seg_next = ti.y;
   // A tile is worked off in PIECES: the part of one group that lies in it (one-group path, as
   // long as it has kFastMin slots or is all that is left), or a run of smaller group parts
   // (per-slot path).  Most tiles of a heavy operator are one piece.
   for (u64 r0 = t0_slot; r0 < t1_slot;) {
    while (gslot[g_next + 1] <= r0) ++g_next;
    while ((u64)seg_slot[seg_next + 1] <= r0) ++seg_next;
    const int g0 = g_next, seg0 = seg_next;
    const u64 gs0 = gslot[g0];
    u64 r1 = min(gslot[g0 + 1], t1_slot);
    bool piece_single = true;
    if (r1 - r0 < (u64)kFastMin && r1 < t1_slot) {
      piece_single = false;
      int gg = g0 + 1;
      while (r1 < t1_slot && min(gslot[gg + 1], t1_slot) - r1 < (u64)kFastMin) {
        r1 = min(gslot[gg + 1], t1_slot);
        ++gg;
      }
    }
    const u32 n_out = (u32)(r1 - r0);
    const bool one_seg = (u64)seg_slot[seg0 + 1] >= r1;

    // my slots of the tile: slot_of(k), k < kRows.  One-group path: row k, column tid of rows of
    // A = L * (256 / L) slots, so that a thread keeps ONE low branch for the whole tile (its word,
    // phase and weights stay in registers); per-slot path: warp-contiguous, eight per thread.
    double acc[kRows];
    K word[kRows];
    u32 neg = 0;                                  // bit k: the composed word carries a minus sign
    u32 live = 0;                                 // bit k: slot k of mine exists
    u32 row_stride = 32, slot0 = (u32)(warp * (32 * kPer) + lane);
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      acc[k] = 0.0;
      word[k] = 0;
    }
    __syncthreads();                              // previous tile fully consumed (and tables copied)
    if (one_seg && hist_seg != seg0) {            // the shared histogram changes generator: flush
      if (hist_seg >= 0) {
        for (int i = tid; i < passes * QX_RADIX; i += kThreads) {
          const u32 c = (&sm.hist[0][0])[i];
          if (c) atomicAdd(hist + (size_t)hist_seg * passes * QX_RADIX + i, c);
          (&sm.hist[0][0])[i] = 0u;
        }
      }
      hist_seg = seg0;
    }

    bool single = piece_single;
    int n_blocks = 0;
    u64 h0 = 0;
    u32 bl0 = 0;
    const bool fresh = cached_group != g0;
    if (single) {
      if (fresh) {
        cwg = (K)cw[gsrc[g0]];
        lg = low_group<K>(cwg, sm.tb);
        magic = 65536u / lg.L + 1u;               // t / L == (t * magic) >> 16 for t < 2^16 / L
      }
      // a group of a <= 16-qubit system has at most 3^16 < 2^32 slots: divide in the word's width
      // (a 64-bit divide is ~100 instructions and every thread of the tile would run it)
      const K b0 = (K)(r0 - gs0);
      h0 = (u64)(b0 / (K)lg.L);
      bl0 = (u32)(b0 - (K)h0 * (K)lg.L);
      n_blocks = (int)(((bl0 + n_out - 1u) * magic >> 16) + 1u);
      if (n_blocks > kMaxBlocks) {                // tiny low group: take the per-slot path
        single = false;
        cached_group = -1;
      }
    }
    if (single) {
      // ---- the whole tile lies in one group: two-level decode shared by all its sources.  The
      // digits split into a LOW group (three least significant, L <= 27 branches) and the HIGH
      // rest; a "block" is the L consecutive slots that share the high picks.
      const int64_t s0 = (int64_t)gsrc[g0];
      const int n_src = (int)((int64_t)gsrc[g0 + 1] - s0);
      const K key0 = (K)skey[s0];
      if (fresh && tid < (int)lg.L) {
        u32 b = tid, picks = 0;
        K w = 0;
        u32 ex = 0;
        u32 pick[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          pick[j] = b % lg.rad[j];
          b /= lg.rad[j];
          picks |= pick[j] << (2 * j);
        }
#pragma unroll
        for (int j = 2; j >= 0; --j) {
          double wt = 1.0;
          if (lg.bit[j] >= 0) {
            const int p = lg.bit[j] >> 1;
            const u32 ax = sm.tb.axis[p][lg.dig[j]][pick[j]];
            if (FUSED) compose<K>(w, ex, sm.im.img[p][ax - 1], sm.im.imx[p][ax - 1], sm.im.e[p][ax - 1]);
            else w |= (K)ax << lg.bit[j];
            wt = sm.tb.w[p][(u32)((key0 >> lg.bit[j]) & 3u) - 1u][pick[j]];
          }
          sm.low_w[0][tid][j] = wt;               // weights of the first source: all of them if n_src == 1
        }
        LowEntry<K> le;
        le.word = w;
        le.imx = (w ^ (w >> 1)) & Plane<K>::lo;
        le.e = ex & 3u;
        le.pick = picks;
        sm.low[tid] = le;
      }
      cached_group = g0;
      // high digits of every block: picks, output word, partial product of the first source
      const double lam0 = slam[s0];
      for (int e = tid; e < n_blocks; e += kThreads) {
        K h = (K)(h0 + (u64)e);
        K ch = 0;
        for (K m = lg.hi_mask; m;) {
          const int bit = KeyOps<K>::lowest(m);
          m &= m - 1;
          u32 pick;
          divmod_small<K>(h, sm.tb.cnt[bit >> 1][(u32)((cwg >> bit) & 3u) - 1u], h, pick);
          ch |= (K)pick << bit;
        }
        K out = 0;
        u32 ex = 0;
        double v = lam0;
        for (K m = lg.hi_mask; m;) {               // qubit 0 first (stabilizer.py:311-319)
          const int bit = KeyOps<K>::highest(m);
          m ^= (K)1 << bit;
          const u32 pick = (u32)(ch >> bit) & 3u;
          const u32 ax = sm.tb.axis[bit >> 1][(u32)((cwg >> bit) & 3u) - 1u][pick];
          v *= sm.tb.w[bit >> 1][(u32)((key0 >> bit) & 3u) - 1u][pick];
          if (FUSED) compose<K>(out, ex, sm.im.img[bit >> 1][ax - 1], sm.im.imx[bit >> 1][ax - 1], sm.im.e[bit >> 1][ax - 1]);
          else out |= (K)ax << bit;
        }
        HiEntry<K> he;
        he.p = v;
        he.word = out;
        he.e = ex & 3u;
        sm.hi[e] = he;
        sm.choice[e] = ch;
      }
      __syncthreads();
      // my column: low branch bl and first block e0; row k adds bpr blocks
      const u32 bpr = (u32)kThreads / lg.L;       // blocks per row
      const u32 A = bpr * lg.L;                   // slots per row (243 for L = 27)
      const u32 t0 = bl0 + (u32)tid;
      const u32 e0 = (t0 * magic) >> 16;
      const u32 bl = t0 - e0 * lg.L;
      row_stride = A;
      slot0 = (u32)tid;
      if ((u32)tid < A) {
#pragma unroll
        for (int k = 0; k < kRows; ++k)
          if ((u32)k * A + (u32)tid < n_out) live |= 1u << k;
      }
      // first source: low branch in registers, one packed load per slot
      {
        const LowEntry<K> le = sm.low[bl];
        const double2 w01 = *reinterpret_cast<const double2*>(&sm.low_w[0][bl][0]);
        const double w2 = sm.low_w[0][bl][2];
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
          if (live & (1u << k)) {
            const HiEntry<K> he = sm.hi[e0 + (u32)k * bpr];
            double v = __dmul_rn(he.p, w2);        // ((p_hi * w2) * w1) * w0, absent = 1.0
            v = __dmul_rn(v, w01.y);
            acc[k] = __dmul_rn(v, w01.x);
            K out = he.word;
            if (FUSED) {
              u32 ex = he.e;
              compose<K>(out, ex, le.word, le.imx, le.e);
              neg |= composed_sign<K>(out, ex) << k;
            } else {
              out |= le.word;
            }
            word[k] = out;
          }
        }
      }
      // remaining sources of the group
      const int64_t po = pre_off ? pre_off[g0] : -1;
      if (po >= 0) {
        // the group's sums were evaluated mode by mode beforehand (k_group_kron): take them
        const double* pv = pre + po + (int64_t)(r0 - gs0) + tid;
#pragma unroll
        for (int k = 0; k < kRows; ++k)
          if (live & (1u << k)) acc[k] = pv[(u32)k * A];
      } else if (n_src >= kBlockedMin) {
        // ---- many sources: factor the sum.  Sources of the group that agree on all HIGH digits (a
        // "source block": adjacent when the input is in canonical order, at most L of them) share
        // the high product, so  sum_s lambda_s * hi_s(h) * lo_s(l)  =  sum_blocks hi_blk(h) * q_blk(l)
        // with q_blk(l) = sum_{s in blk} lambda_s * lo_s(l): up to L times fewer (source, slot)
        // pairs.  Any split into blocks is valid (an unsorted input only gives shorter blocks).
        // The association of the products differs from the reference's left-to-right order, so
        // coefficients agree with it to rounding (~1e-16 relative), not bitwise; groups with fewer
        // sources take the exact loop below.
        const K hm2 = lg.hi_mask | (lg.hi_mask << 1);
        const int nb_max = max(1, min(kBlockRound, kPhiCap / n_blocks));
        K* src_key = reinterpret_cast<K*>(sm.p_hi);                       // staged sources alias p_hi:
        double* src_lam = sm.p_hi + kSrcRound / (8 / sizeof(K)) ;         // consumed before p_hi is written
        double* q = &sm.low_w[1][0][0];                                     // [block][low branch]
        for (int c0 = 1; c0 < n_src;) {
          const int avail = min(kSrcRound, n_src - c0);
          __syncthreads();                          // previous round (or the first source) consumed
          for (int i = tid; i < avail; i += kThreads) {
            src_key[i] = (K)skey[s0 + c0 + i];
            src_lam[i] = slam[s0 + c0 + i];
          }
          if (tid == 0) sm.consumed = avail;
          __syncthreads();
          // block heads among the staged sources, two per thread
          const int i0 = 2 * tid, i1 = 2 * tid + 1;
          const bool hd0 = i0 < avail && (i0 == 0 || (src_key[i0] & hm2) != (src_key[i0 - 1] & hm2));
          const bool hd1 = i1 < avail && (src_key[i1] & hm2) != (src_key[i0] & hm2);
          u32 nheads;
          const u32 before = block_exclusive_sum<u32>((u32)hd0 + (u32)hd1, reinterpret_cast<u32*>(sm.scan), nheads);
          if (hd0) {
            const u32 id = before;
            if (id < (u32)nb_max) { sm.blk_first[id] = (unsigned short)i0; sm.blk_key[id] = src_key[i0]; }
            else if (id == (u32)nb_max) sm.consumed = i0;
          }
          if (hd1) {
            const u32 id = before + (u32)hd0;
            if (id < (u32)nb_max) { sm.blk_first[id] = (unsigned short)i1; sm.blk_key[id] = src_key[i1]; }
            else if (id == (u32)nb_max) sm.consumed = i1;
          }
          __syncthreads();
          const int nblk = min((int)nheads, nb_max);
          const int used = sm.consumed;
          // q[blk][l]: the block's sources summed in input order
          for (int w = tid; w < nblk * (int)lg.L; w += kThreads) {
            const int b = w / (int)lg.L, l = w - b * (int)lg.L;
            const u32 picks = sm.low[l].pick;
            const int first = sm.blk_first[b], last = (b + 1 < nblk) ? (int)sm.blk_first[b + 1] : used;
            double sum = 0.0;
            for (int i = first; i < last; ++i) {
              const K key = src_key[i];
              double v = src_lam[i];
#pragma unroll
              for (int j = 2; j >= 0; --j)
                if (lg.bit[j] >= 0)
                  v *= sm.tb.w[lg.bit[j] >> 1][(u32)((key >> lg.bit[j]) & 3u) - 1u][(picks >> (2 * j)) & 3u];
              sum += v;
            }
            q[b * 27 + l] = sum;
          }
          __syncthreads();                          // staged sources consumed: p_hi may be overwritten
          for (int w = tid; w < nblk * n_blocks; w += kThreads) {
            const int b = w / n_blocks, e = w - b * n_blocks;
            const K key = sm.blk_key[b];
            const K ch = sm.choice[e];
            double v = 1.0;
            for (K m = lg.hi_mask; m;) {             // qubit 0 first
              const int bit = KeyOps<K>::highest(m);
              m ^= (K)1 << bit;
              v *= sm.tb.w[bit >> 1][(u32)((key >> bit) & 3u) - 1u][(u32)(ch >> bit) & 3u];
            }
            sm.p_hi[b * n_blocks + e] = v;
          }
          __syncthreads();
          for (int b = 0; b < nblk; ++b) {
            const double qb = q[b * 27 + (int)bl];
            const double* ph = sm.p_hi + b * n_blocks + e0;
#pragma unroll
            for (int k = 0; k < kRows; ++k)
              if (live & (1u << k)) acc[k] += ph[(u32)k * bpr] * qb;
          }
          c0 += used;
        }
      } else if (n_src > 1) {
        // few sources: exact pairwise loop, kChunk (or fewer) per round
        const int per_round = max(1, min(kChunk, kPhiCap / n_blocks));
        for (int c0 = 1; c0 < n_src; c0 += per_round) {
          const int nc = min(per_round, n_src - c0);
          __syncthreads();                          // previous round (or the first source) consumed
          for (int w = tid; w < nc * n_blocks; w += kThreads) {
            const int c = w / n_blocks, e = w - c * n_blocks;
            const K key = (K)skey[s0 + c0 + c];
            const K ch = sm.choice[e];
            double v = slam[s0 + c0 + c];
            for (K m = lg.hi_mask; m;) {             // qubit 0 first
              const int bit = KeyOps<K>::highest(m);
              m ^= (K)1 << bit;
              v *= sm.tb.w[bit >> 1][(u32)((key >> bit) & 3u) - 1u][(u32)(ch >> bit) & 3u];
            }
            sm.p_hi[c * n_blocks + e] = v;
          }
          for (int w = tid; w < nc * (int)lg.L; w += kThreads) {
            const int c = w / (int)lg.L, l = w - c * (int)lg.L;
            const K key = (K)skey[s0 + c0 + c];
            const u32 picks = sm.low[l].pick;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              double wt = 1.0;
              if (lg.bit[j] >= 0)
                wt = sm.tb.w[lg.bit[j] >> 1][(u32)((key >> lg.bit[j]) & 3u) - 1u][(picks >> (2 * j)) & 3u];
              sm.low_w[1 + c][l][j] = wt;            // row 0 stays the first source's (cached per group)
            }
          }
          __syncthreads();
          for (int c = 0; c < nc; ++c) {
            const double2 w01 = *reinterpret_cast<const double2*>(&sm.low_w[1 + c][bl][0]);
            const double w2 = sm.low_w[1 + c][bl][2];
            const double* ph = sm.p_hi + c * n_blocks + e0;
#pragma unroll
            for (int k = 0; k < kRows; ++k) {
              if (live & (1u << k)) {
                // explicit roundings: a fused multiply-add of the last product into the sum would
                // round differently from the reference
                double v = __dmul_rn(ph[(u32)k * bpr], w2);
                v = __dmul_rn(v, w01.y);
                v = __dmul_rn(v, w01.x);
                acc[k] = __dadd_rn(acc[k], v);
              }
            }
          }
        }
      }
    } else {
      // ---- several (small) groups in the tile: every slot finds its group and walks its sources
#pragma unroll 1
      for (int k = 0; k < kPer; ++k) {
        const u32 idx = (u32)(warp * (32 * kPer) + k * 32 + lane);
        if (idx >= n_out) continue;
        live |= 1u << k;
        const u64 r = r0 + idx;
        int64_t lo = g0, hi = min(ngroups, (int64_t)g0 + (int64_t)n_out + 1);   // gslot[lo] <= r < gslot[hi]
        while (hi - lo > 1) {
          const int64_t mid = (lo + hi) >> 1;
          if (gslot[mid] <= r) lo = mid; else hi = mid;
        }
        const int64_t s0 = (int64_t)gsrc[lo], s1 = (int64_t)gsrc[lo + 1];
        const K cg = (K)cw[s0];
        K b = (K)(r - gslot[lo]);
        K ch = 0;
        for (K m = KeyOps<K>::support(cg); m;) {
          const int bit = KeyOps<K>::lowest(m);
          m &= m - 1;
          u32 pick;
          divmod_small<K>(b, sm.tb.cnt[bit >> 1][(u32)((cg >> bit) & 3u) - 1u], b, pick);
          ch |= (K)pick << bit;
        }
        K out = 0;
        u32 ex = 0;
        for (K m = KeyOps<K>::support(cg); m;) {
          const int bit = KeyOps<K>::highest(m);
          m ^= (K)1 << bit;
          const u32 ax = sm.tb.axis[bit >> 1][(u32)((cg >> bit) & 3u) - 1u][(u32)(ch >> bit) & 3u];
          if (FUSED) compose<K>(out, ex, sm.im.img[bit >> 1][ax - 1], sm.im.imx[bit >> 1][ax - 1], sm.im.e[bit >> 1][ax - 1]);
          else out |= (K)ax << bit;
        }
        double sum = 0.0;
        const int64_t po = pre_off ? pre_off[lo] : -1;
        if (po >= 0) {
          sum = pre[po + (int64_t)(r - gslot[lo])];
        } else {
          for (int64_t s = s0; s < s1; ++s) {
            const K key = (K)skey[s];
            double v = slam[s];
            for (K m = KeyOps<K>::support(cg); m;) {
              const int bit = KeyOps<K>::highest(m);
              m ^= (K)1 << bit;
              v = __dmul_rn(v, sm.tb.w[bit >> 1][(u32)((key >> bit) & 3u) - 1u][(u32)(ch >> bit) & 3u]);
            }
            sum = (s == s0) ? v : __dadd_rn(sum, v);
          }
        }
        acc[k] = sum;
        word[k] = out;
        if (FUSED) neg |= composed_sign<K>(out, ex) << k;
      }
    }

    // ---- drop rule and write-out
    u32 pre[kRows];
    u32 kept_bits = 0, running = 0;
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      if (neg & (1u << k)) acc[k] = -acc[k];     // sign flips are exact
      const bool kept = (live & (1u << k)) && fabs(acc[k]) >= eps;
      if (kept) kept_bits |= 1u << k;
      const u32 votes = __ballot_sync(QX_FULL_MASK, kept);
      pre[k] = running + __popc(votes & lanemask_lt());
      running += __popc(votes);
    }
    if (one_seg) {
      u64 tile_total;
      u64 warp_excl = block_exclusive_sum<u64>(lane == 0 ? (u64)running : 0ull, sm.scan, tile_total);
      warp_excl = __shfl_sync(QX_FULL_MASK, warp_excl, 0);
      if (tid == 0) sm.base = (u64)seg_slot[seg0] + atomicAdd(seg_count + seg0, tile_total);
      // digit counts: the two low bytes one shared atomic each; everything above them changes
      // slowly along the slots (high digits of the word), so a thread counts runs of equal
      // upper parts in a register and flushes a run with one atomic per pass
      {
        KO run_key = 0;
        u32 run_cnt = 0;
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
          if (kept_bits & (1u << k)) {
            const KO key = (KO)word[k];
            atomicAdd(&sm.hist[0][digit_of(key, 0)], 1u);
            if (passes > 1) atomicAdd(&sm.hist[1][digit_of(key, 1)], 1u);
            if (passes > 2) {
              if (run_cnt && (key >> 16) == (run_key >> 16)) {
                ++run_cnt;
              } else {
                if (run_cnt)
                  for (int p = 2; p < passes; ++p) atomicAdd(&sm.hist[p][digit_of(run_key, p)], run_cnt);
                run_key = key;
                run_cnt = 1;
              }
            }
          }
        }
        if (run_cnt)
          for (int p = 2; p < passes; ++p) atomicAdd(&sm.hist[p][digit_of(run_key, p)], run_cnt);
      }
      __syncthreads();
      const int64_t base = (int64_t)(sm.base + warp_excl);
#pragma unroll
      for (int k = 0; k < kRows; ++k) {
        if (kept_bits & (1u << k)) {
          const int64_t pos = base + pre[k];
          st_stream(keys_out + pos, (KO)word[k]);
          st_stream(lam_out + pos, acc[k]);
        }
      }
    } else {
      // the tile crosses a generator boundary (only tiny generators): one atomic per kept term
#pragma unroll 1
      for (int k = 0; k < kRows; ++k) {
        if (kept_bits & (1u << k)) {
          const int64_t r = (int64_t)(r0 + slot0 + (u32)k * row_stride);
          const int g = segment_of(seg_slot, n_seg, r);
          const int64_t pos = seg_slot[g] + (int64_t)atomicAdd(seg_count + g, 1ull);
          const KO key = (KO)word[k];
          st_stream(keys_out + pos, key);
          st_stream(lam_out + pos, acc[k]);
          for (int p = 0; p < passes; ++p)
            atomicAdd(hist + ((size_t)g * passes + p) * QX_RADIX + digit_of(key, p), 1u);
        }
      }
    }
    r0 = r1;
   }
  }
  __syncthreads();
  if (hist_seg >= 0) {
    for (int i = tid; i < passes * QX_RADIX; i += kThreads) {
      const u32 c = (&sm.hist[0][0])[i];
      if (c) atomicAdd(hist + (size_t)hist_seg * passes * QX_RADIX + i, c);
    }
  }
}

// ---- groups with many sources: the sums mode by mode ------------------------------------------------
// A group's slot values are  out[pick_1..pick_w] = sum over its sources of lambda * prod_j W_j[d_j][pick_j]:
// with the sources scattered into a dense 3^w tensor over their digits this is a Kronecker product
// applied to a vector, and contracting one digit at a time costs w * 3 * 3^w multiply-adds instead
// of (sources x slots) -- 1.6e5 instead of 4.3e7 for a full group of xyz_chain(8,4) (the factored
// sum of k_group_emit shares only the high product over the <= 27 sources of a block).  One CTA
// per group of at most 8 digits, two 3^8 tensors in shared memory, digits contracted qubit 0
// first; the result is written in slot order (lowest digit fastest, radices of the classes) and
// k_group_emit takes it instead of walking the sources.  The products are associated differently
// from the reference's left-to-right order (stabilizer.py:311-319), so these coefficients agree
// with it to rounding, like the factored sum they replace.
constexpr int kKronDigits = 8;
constexpr int kKronSize = 6561;                // 3^8

template <typename K>
__global__ void __launch_bounds__(256)
k_group_kron(const u64* __restrict__ cw, const u64* __restrict__ skey, const double* __restrict__ slam,
             const u64* __restrict__ gsrc, const int* __restrict__ flagged, const int64_t* __restrict__ pre_off,
             double* __restrict__ pre, const __grid_constant__ OperatorTable tb) {
  extern __shared__ __align__(16) unsigned char kron_raw[];
  double* A = reinterpret_cast<double*>(kron_raw);
  double* B = A + kKronSize;
  const int tid = threadIdx.x;
  const int g = flagged[blockIdx.x];
  const int64_t s0 = (int64_t)gsrc[g], s1 = (int64_t)gsrc[g + 1];
  const K cwg = (K)cw[s0];
  int pos[kKronDigits], rad[kKronDigits];
  int w = 0, size = 1;
  for (K m = KeyOps<K>::support(cwg); m; m &= m - 1) {
    const int bit = KeyOps<K>::lowest(m);
    pos[w] = bit;
    rad[w] = tb.cnt[bit >> 1][(u32)((cwg >> bit) & 3u) - 1u];
    ++w;
    size *= 3;
  }
  for (int i = tid; i < size; i += 256) A[i] = 0.0;
  __syncthreads();
  for (int64_t sidx = s0 + tid; sidx < s1; sidx += 256) {       // the sources' words are distinct
    const K key = (K)skey[sidx];
    int idx = 0, mul = 1;
    for (int j = 0; j < w; ++j) {
      idx += ((int)((key >> pos[j]) & 3u) - 1) * mul;
      mul *= 3;
    }
    A[idx] = slam[sidx];
  }
  __syncthreads();
  int stride = size / 3;
  for (int j = w - 1; j >= 0; --j, stride /= 3) {              // qubit 0 (the highest digit) first
    const int p = pos[j] >> 1;
    const double w00 = tb.w[p][0][0], w01 = tb.w[p][0][1], w02 = tb.w[p][0][2];
    const double w10 = tb.w[p][1][0], w11 = tb.w[p][1][1], w12 = tb.w[p][1][2];
    const double w20 = tb.w[p][2][0], w21 = tb.w[p][2][1], w22 = tb.w[p][2][2];
    const int radix = rad[j];
    for (int i = tid; i < size; i += 256) {
      const int t = (i / stride) % 3;
      const int base = i - t * stride;
      double v = 0.0;
      if (t < radix) {
        const double a0 = A[base], a1 = A[base + stride], a2 = A[base + 2 * stride];
        const double c0 = t == 0 ? w00 : t == 1 ? w01 : w02;
        const double c1 = t == 0 ? w10 : t == 1 ? w11 : w12;
        const double c2 = t == 0 ? w20 : t == 1 ? w21 : w22;
        v = __dadd_rn(__dadd_rn(__dmul_rn(a0, c0), __dmul_rn(a1, c1)), __dmul_rn(a2, c2));
      }
      B[i] = v;
    }
    __syncthreads();
    double* t2 = A;
    A = B;
    B = t2;
  }
  // picks (stride 3 per digit) -> slot inside the group's box (radices of the classes)
  double* out = pre + pre_off[g];
  for (int i = tid; i < size; i += 256) {
    int rest = i, slot = 0, mul = 1;
    bool ok = true;
    for (int j = 0; j < w; ++j) {
      const int t = rest % 3;
      rest /= 3;
      ok = ok && t < rad[j];
      slot += t * mul;
      mul *= rad[j];
    }
    if (ok) out[slot] = A[i];
  }
}

// ---- the same contraction for groups on 9..12 digits: the tensor (3^w doubles, <= 4.3 MB) lives
// in global memory (L2 resident), one launch per mode over all such groups (blockIdx.y = group).
constexpr int kKronWideDigits = 12;

template <typename K>
__global__ void __launch_bounds__(256)
k_kron_scatter(const u64* __restrict__ cw, const u64* __restrict__ skey, const double* __restrict__ slam,
               const u64* __restrict__ gsrc, const int* __restrict__ flagged, const int64_t* __restrict__ toff,
               double* __restrict__ tensor) {
  const int g = flagged[blockIdx.y];
  const int64_t s0 = (int64_t)gsrc[g], s1 = (int64_t)gsrc[g + 1];
  const K cwg = (K)cw[s0];
  int pos[kKronWideDigits];
  int w = 0;
  for (K m = KeyOps<K>::support(cwg); m; m &= m - 1) pos[w++] = KeyOps<K>::lowest(m);
  double* t = tensor + toff[blockIdx.y];
  for (int64_t sidx = s0 + (int64_t)blockIdx.x * 256 + threadIdx.x; sidx < s1; sidx += (int64_t)gridDim.x * 256) {
    const K key = (K)skey[sidx];
    int idx = 0, mul = 1;
    for (int j = 0; j < w; ++j) {
      idx += ((int)((key >> pos[j]) & 3u) - 1) * mul;
      mul *= 3;
    }
    t[idx] = slam[sidx];
  }
}

// mode `m` counted from the highest digit (qubit 0 side) of each group; groups with fewer digits copy
template <typename K>
__global__ void __launch_bounds__(256)
k_kron_mode(const u64* __restrict__ cw, const u64* __restrict__ gsrc, const int* __restrict__ flagged,
            const int64_t* __restrict__ toff, const double* __restrict__ src, double* __restrict__ dst, int m,
            const __grid_constant__ OperatorTable tb) {
  const int g = flagged[blockIdx.y];
  const K cwg = (K)cw[gsrc[g]];
  const K sup = KeyOps<K>::support(cwg);
  const int w = (int)Plane<K>::popc(sup);
  int size = 1;
  for (int j = 0; j < w; ++j) size *= 3;
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= size) return;
  const double* a = src + toff[blockIdx.y];
  double* b = dst + toff[blockIdx.y];
  if (m >= w) {
    b[i] = a[i];
    return;
  }
  const int j = w - 1 - m;
  K rest = sup;
  int stride = 1;
  for (int q = 0; q < j; ++q) {
    rest &= rest - 1;
    stride *= 3;
  }
  const int bit = KeyOps<K>::lowest(rest);
  const int p = bit >> 1;
  const int radix = tb.cnt[p][(u32)((cwg >> bit) & 3u) - 1u];
  const int t = (i / stride) % 3;
  const int base = i - t * stride;
  double v = 0.0;
  if (t < radix)
    v = __dadd_rn(__dadd_rn(__dmul_rn(a[base], tb.w[p][0][t]), __dmul_rn(a[base + stride], tb.w[p][1][t])),
                  __dmul_rn(a[base + 2 * stride], tb.w[p][2][t]));
  b[i] = v;
}

template <typename K>
__global__ void __launch_bounds__(256)
k_kron_pick(const u64* __restrict__ cw, const u64* __restrict__ gsrc, const int* __restrict__ flagged,
            const int64_t* __restrict__ toff, const double* __restrict__ tensor, const int64_t* __restrict__ pre_off,
            double* __restrict__ pre, const __grid_constant__ OperatorTable tb) {
  const int g = flagged[blockIdx.y];
  const K cwg = (K)cw[gsrc[g]];
  int rest = blockIdx.x * 256 + threadIdx.x, slot = 0, mul = 1;
  const int i = rest;
  bool ok = true;
  for (K m = KeyOps<K>::support(cwg); m; m &= m - 1) {
    const int bit = KeyOps<K>::lowest(m);
    const int radix = tb.cnt[bit >> 1][(u32)((cwg >> bit) & 3u) - 1u];
    const int t = rest % 3;
    rest /= 3;
    ok = ok && t < radix;
    slot += t * mul;
    mul *= radix;
  }
  if (ok && rest == 0) pre[pre_off[g] + slot] = tensor[toff[blockIdx.y] + i];
}

template <typename K>
int launch_kron_wide(qx_store* s, const u64* cw, const u64* skey, const double* slam, const u64* gsrc,
                     const int* d_flag, const int64_t* d_toff, int n_big, int w_max, int64_t max_src, double* ta,
                     double* tb2, int64_t tensor_total, const int64_t* pre_off, double* pre, const OperatorTable& ct) {
  int size = 1;
  for (int j = 0; j < w_max; ++j) size *= 3;
  const dim3 grid((unsigned)((size + 255) / 256), (unsigned)n_big);
  QX_CUDA(cudaMemsetAsync(ta, 0, sizeof(double) * (size_t)tensor_total, s->stream));
  const dim3 sgrid((unsigned)std::max<int64_t>(1, std::min<int64_t>((max_src + 255) / 256, 1024)), (unsigned)n_big);
  k_kron_scatter<K><<<sgrid, 256, 0, s->stream>>>(cw, skey, slam, gsrc, d_flag, d_toff, ta);
  for (int m = 0; m < w_max; ++m) {
    k_kron_mode<K><<<grid, 256, 0, s->stream>>>(cw, gsrc, d_flag, d_toff, ta, tb2, m, ct);
    std::swap(ta, tb2);
  }
  k_kron_pick<K><<<grid, 256, 0, s->stream>>>(cw, gsrc, d_flag, d_toff, ta, pre_off, pre, ct);
  qx_count_launches(w_max + 2);
  QX_CUDA(cudaGetLastError());
  return QX_OK;
}

template <typename K, typename KO, bool FUSED>
int launch_group_emit(qx_store* s, int64_t tiles, const u64* cw, const u64* skey, const double* slam,
                      const u64* gsrc, const u64* gslot, const u64* totals, const int2* tile_info,
                      const int64_t* seg_slot, int out, u64* seg_count, u32* hist, int passes, double eps,
                      int part, int parts, const int64_t* pre_off, const double* pre, const OperatorTable& tb,
                      const ImageTable<K>& im) {
  static int per_sm = 0;
  if (per_sm == 0) {
    QX_CUDA(cudaFuncSetAttribute(k_group_emit<K, KO, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(GroupSmem<K>)));
    QX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_group_emit<K, KO, FUSED>, kThreads,
                                                          sizeof(GroupSmem<K>)));
    per_sm = std::max(per_sm, 1);
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles / parts + 1, (int64_t)s->sm_count * per_sm));
  k_group_emit<K, KO, FUSED><<<grid, kThreads, sizeof(GroupSmem<K>), s->stream>>>(
      cw, skey, slam, gsrc, gslot, totals, tile_info, seg_slot, s->n_seg,
      reinterpret_cast<KO*>(s->keys[out]), s->lam[out], seg_count, hist, passes, eps, part, parts, pre_off, pre, tb, im);
  QX_CUDA(cudaGetLastError());
  return QX_OK;
}

// Connected components of "input axes that share an output axis", per digit position; the table
// handed to the kernels describes the class of each input axis (radix, output axes) and keeps the
// per-axis weights, zero where the axis does not reach that output.
void build_class_table(const OperatorTable& nz, int n_qubits, OperatorTable* ct, ClassIds* ids) {
  *ct = nz;
  memset(ids, 0, sizeof(*ids));
  for (int p = 0; p < QX_MAX_QUBITS; ++p) {
    unsigned reach[3];                            // bit (ax-1) set: input axis a reaches output ax
    for (int a = 0; a < 3; ++a) {
      reach[a] = 0;
      for (int b = 0; b < nz.cnt[p][a]; ++b) reach[a] |= 1u << (nz.axis[p][a][b] - 1);
    }
    int parent[3] = {0, 1, 2};
    for (int a = 0; a < 3; ++a)
      for (int b = a + 1; b < 3; ++b)
        if (reach[a] & reach[b]) {
          int ra = a, rb = b;
          while (parent[ra] != ra) ra = parent[ra];
          while (parent[rb] != rb) rb = parent[rb];
          if (ra != rb) parent[std::max(ra, rb)] = std::min(ra, rb);
        }
    // a second sweep closes chains (X~Y, Y~Z found in either order)
    for (int a = 0; a < 3; ++a) {
      int r = a;
      while (parent[r] != r) r = parent[r];
      parent[a] = r;
    }
    for (int a = 0; a < 3; ++a) {
      unsigned out = 0;
      for (int b = 0; b < 3; ++b)
        if (parent[b] == parent[a]) out |= reach[b];
      ids->cls[p][a] = (unsigned char)(parent[a] + 1);
      int c = 0;
      for (int ax = 1; ax <= 3; ++ax) {
        if (!(out & (1u << (ax - 1)))) continue;
        double w = 0.0;
        for (int b = 0; b < nz.cnt[p][a]; ++b)
          if (nz.axis[p][a][b] == ax) w = nz.w[p][a][b];
        ct->axis[p][a][c] = (unsigned char)ax;
        ct->w[p][a][c] = w;
        ++c;
      }
      ct->cnt[p][a] = (unsigned char)c;
      for (; c < 3; ++c) {
        ct->axis[p][a][c] = (unsigned char)(a + 1);
        ct->w[p][a][c] = 0.0;
      }
    }
  }
  (void)n_qubits;
}

template <typename T>
T* carve(char*& cursor, int64_t count) {
  T* p = reinterpret_cast<T*>(cursor);
  cursor += (sizeof(T) * (size_t)count + 255) / 256 * 256;
  return p;
}
inline int64_t padded(int64_t bytes) { return (bytes + 255) / 256 * 256; }

}  // namespace

namespace qxe {
void fill_images_u32(int n_qubits, const uint32_t* program, int n_ops, u32 cx_c, u32 cx_t, u32 cx_s,
                     ImageTable<u32>* im);
void fill_images_u64(int n_qubits, const uint32_t* program, int n_ops, u32 cx_c, u32 cx_t, u32 cx_s,
                     ImageTable<u64>* im);
}  // namespace qxe

// Host-only: the class decomposition the grouped path uses, for callers and tests (no GPU needed).
extern "C" int qx_operator_classes(int32_t n_qubits, const int32_t* counts, const int32_t* axes,
                                   const double* weights, int32_t* class_id, int32_t* class_radix,
                                   int32_t* class_axes, double* class_weights) {
  QX_REQUIRE(counts && axes && weights && class_id && class_radix, "NULL argument");
  QX_REQUIRE(n_qubits >= 1 && n_qubits <= QX_MAX_QUBITS, "n_qubits=%d out of range", n_qubits);
  OperatorTable nz;
  for (int p = 0; p < QX_MAX_QUBITS; ++p)
    for (int a = 0; a < 3; ++a) {
      nz.cnt[p][a] = 1;
      for (int b = 0; b < 3; ++b) {
        nz.axis[p][a][b] = (unsigned char)(a + 1);
        nz.w[p][a][b] = (b == 0) ? 1.0 : 0.0;
      }
    }
  for (int j = 0; j < n_qubits; ++j) {
    const int p = n_qubits - 1 - j;
    for (int a = 0; a < 3; ++a) {
      const int c = counts[j * 3 + a];
      QX_REQUIRE(c >= 1 && c <= 3, "qubit %d axis %d: %d nonzero weights (need 1..3)", j, a + 1, c);
      nz.cnt[p][a] = (unsigned char)c;
      for (int b = 0; b < c; ++b) {
        const int ax = axes[(j * 3 + a) * 3 + b];
        QX_REQUIRE(ax >= 1 && ax <= 3, "qubit %d axis %d: output axis %d out of range", j, a + 1, ax);
        nz.axis[p][a][b] = (unsigned char)ax;
        nz.w[p][a][b] = weights[(j * 3 + a) * 3 + b];
      }
    }
  }
  OperatorTable ct;
  ClassIds ids;
  build_class_table(nz, n_qubits, &ct, &ids);
  for (int j = 0; j < n_qubits; ++j) {
    const int p = n_qubits - 1 - j;
    for (int a = 0; a < 3; ++a) {
      class_id[j * 3 + a] = ids.cls[p][a];
      class_radix[j * 3 + a] = ct.cnt[p][a];
      for (int b = 0; b < 3; ++b) {
        if (class_axes) class_axes[(j * 3 + a) * 3 + b] = b < ct.cnt[p][a] ? ct.axis[p][a][b] : 0;
        if (class_weights) class_weights[(j * 3 + a) * 3 + b] = b < ct.cnt[p][a] ? ct.w[p][a][b] : 0.0;
      }
    }
  }
  return QX_OK;
}

namespace {
int g_bucket_on = -1;          // -1: not decided yet (QX_NO_BUCKET in the environment switches it off)
bool bucket_enabled() {
  if (g_bucket_on < 0) g_bucket_on = getenv("QX_NO_BUCKET") ? 0 : 1;
  return g_bucket_on != 0;
}
}  // namespace

int64_t g_dense_last[4] = {0, 0, 0, 0};   // qx_dense_last

extern "C" int qx_dense_last(int64_t out[4]) {
  QX_REQUIRE(out != nullptr, "NULL argument");
  for (int i = 0; i < 4; ++i) out[i] = g_dense_last[i];
  return QX_OK;
}

extern "C" int qx_bucket_enable(int32_t on) {
  const int before = bucket_enabled() ? 1 : 0;
  g_bucket_on = on ? 1 : 0;
  return before;
}

extern "C" int qx_bucket_last(int64_t out[8]) {
  QX_REQUIRE(out != nullptr, "NULL argument");
  const qxb::BucketStats& st = qxb::bucket_stats();
  out[0] = st.groups;
  out[1] = st.tiles;
  out[2] = st.units;
  out[3] = st.max_unit;
  out[4] = st.slots;
  out[5] = st.ell;
  out[6] = st.cap;
  out[7] = st.ctas_per_sm;
  return QX_OK;
}

// ---- packed form behind the bucketed step (a store that is only downloaded next) ---------------
// The bucketed step leaves canonical 64-bit keys.  What crosses PCIe for n <= 16 is the packed form
// of the sort's last pass (merge.cuh): 16-bit low halves + per generator the first position of
// every value of the high 16 bits.  One pass makes it from the sorted keys: 8 B read, 2 B written
// per term; a term whose predecessor has another high half opens its bucket (positions are unique:
// plain stores); the empty buckets are filled by the suffix-minimum kernel of the sort.  The halves
// and the table go into the store's DEAD key buffer, which then becomes the live one.
namespace {
__global__ void __launch_bounds__(256)
k_pack_keys(const u64* __restrict__ keys, const int64_t* __restrict__ seg, unsigned short* __restrict__ lows,
            u32* __restrict__ bnd) {
  const int g = blockIdx.y;
  const int64_t lo = seg[g], hi = seg[g + 1];
  u32* row = bnd + (size_t)g * (QX_PACK_BUCKETS + 1);
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    const u64 k = keys[i];
    lows[i] = (unsigned short)k;
    const u32 h = (u32)(k >> 16);
    if (i == lo || (u32)(keys[i - 1] >> 16) != h) row[h] = (u32)(i - lo);
  }
}

// *packed = false: the form does not apply (small result, a generator of 2^32 terms, no room)
int pack_for_download(qx_store* s, int64_t total, int64_t ub_seg, bool* packed) {
  *packed = false;
  const int n_seg = s->n_seg;
  const int64_t bnd_bytes = 4ll * n_seg * (QX_PACK_BUCKETS + 1);
  const int64_t lo_bytes = (2 * total + 255) / 256 * 256;
  if (s->n_qubits > 16 || total < 8ll * n_seg * QX_PACK_BUCKETS || ub_seg >= (1ll << 32) - 1 ||
      lo_bytes + bnd_bytes > 8 * s->cap)
    return QX_OK;
  const int live = s->cur, dead = s->cur ^ 1;
  unsigned short* lows = reinterpret_cast<unsigned short*>(s->keys[dead]);
  u32* bnd = reinterpret_cast<u32*>(reinterpret_cast<char*>(s->keys[dead]) + lo_bytes);
  QX_CUDA(cudaMemsetAsync(bnd, 0xff, (size_t)bnd_bytes, s->stream));
  {
    QxProfileScope prof(QX_K_DENSE_PREP, s->stream, 10.0 * (double)total, 2);
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((ub_seg + 255) / 256, (int64_t)s->sm_count * 4));
    k_pack_keys<<<dim3(gx, (unsigned)n_seg), 256, 0, s->stream>>>(s->keys[live], s->seg[live], lows, bnd);
    QX_CUDA(cudaGetLastError());
    qxm::k_pack_bounds<<<n_seg, 1024, 0, s->stream>>>(bnd, s->seg[live]);
    QX_CUDA(cudaGetLastError());
  }
  // the key buffers trade places: keys[cur] is the packed block now, next to the coefficients it belongs to
  std::swap(s->keys[live], s->keys[dead]);
  s->narrow_keys = true;
  s->pack_bnd = bnd;
  *packed = true;
  return QX_OK;
}
}  // namespace

// The large operator step.  On entry the store holds the merged input terms (exact offsets on
// the host); on exit it holds the canonical result and exact offsets.  `nz` is the operator's
// non-zero branch table (fill_table in branch.cu).
// probe_fanout > 0: the caller has not counted the raw branches; group the sources first and go
// on only if the operator is worth it (some generator above the small-merge limit and at least
// probe_fanout slots per source), otherwise leave the store untouched and report *done = false.
int qx_dense_operator_step(qx_store* s, const OperatorTable& nz, const uint32_t* program, int n_ops,
                           u32 cx_c, u32 cx_t, u32 cx_s, double eps, int64_t* slots_total,
                           int64_t probe_fanout, bool* done, int part, int parts) {
  if (done) *done = false;
  QX_CUDA(cudaSetDevice(s->device));
  const int n_seg = s->n_seg;
  const int64_t n = s->h_seg[n_seg];
  OperatorTable ct;
  ClassIds ids;
  build_class_table(nz, s->n_qubits, &ct, &ids);

  // ---- temporaries of the source side (caching allocator: microseconds after the first run)
  const int64_t src_tiles = std::max<int64_t>(1, (n + kTileSlots - 1) / kTileSlots);
  const int64_t bytes1 = 2 * padded(8 * n) + 2 * padded(8 * n) + padded(8 * n) + padded(8 * n) +
                         2 * padded(8 * (n + 1)) + padded(8 * ((int64_t)n_seg + 1)) + 256 +
                         2 * padded(8 * (src_tiles + 1)) + 256;
  void* block1 = nullptr;
  QX_TRY(qx_dev_alloc(&block1, bytes1, s->stream, s->device));
  struct Release {
    void* p;
    cudaStream_t st;
    ~Release() { qx_dev_free(p, st); }
  } rel1{block1, s->stream};
  char* cur = reinterpret_cast<char*>(block1);
  u64* cwb[2] = {carve<u64>(cur, n), carve<u64>(cur, n)};
  double* idb[2] = {carve<double>(cur, n), carve<double>(cur, n)};
  u64* skey = carve<u64>(cur, n);
  double* slam = carve<double>(cur, n);
  u64* gsrc = carve<u64>(cur, n + 1);
  u64* gslot = carve<u64>(cur, n + 1);
  int64_t* seg_slot = carve<int64_t>(cur, (int64_t)n_seg + 1);
  u64* totals = carve<u64>(cur, 2);
  u64* st_heads = carve<u64>(cur, src_tiles + 1);
  u64* st_slots = carve<u64>(cur, src_tiles + 1);
  u32* ticket1 = carve<u32>(cur, 2);
  QX_CUDA(cudaMemsetAsync(totals, 0, (size_t)(reinterpret_cast<char*>(ticket1) + 256 - reinterpret_cast<char*>(totals)),
                          s->stream));

  const int in = s->cur;
  int sorted;
  if (n <= kPrepSmall && n_seg < 65535) {
    QxProfileScope prof(QX_K_DENSE_PREP, s->stream, 72.0 * (double)n);
    k_group_prep_small<<<1, kPrepThreads, 0, s->stream>>>(s->keys[in], s->lam[in], s->seg[in], n_seg, (int)n,
                                                         cwb[in], skey, slam, gsrc, gslot, seg_slot, totals, ids, ct);
    QX_CUDA(cudaGetLastError());
    sorted = in;
  } else {
    {
      QxProfileScope prof(QX_K_DENSE_PREP, s->stream, 8.0 * (double)n + 16.0 * (double)n);
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, (int64_t)s->sm_count * 8));
      k_class_words<<<grid, kThreads, 0, s->stream>>>(s->keys[in], n, cwb[in], idb[in], ids);
      QX_CUDA(cudaGetLastError());
    }
    {
      // stable segmented sort of (class word, source index) by class word
      qxm::MergeBuffers<double> mb;
      mb.keys[in] = cwb[in];
      mb.keys[in ^ 1] = cwb[in ^ 1];
      mb.vals[in] = idb[in];
      mb.vals[in ^ 1] = idb[in ^ 1];
      mb.seg[0] = s->seg[0];
      mb.seg[1] = s->seg[1];
      mb.cur = in;
      mb.n_seg = n_seg;
      mb.ub_total = n;
      mb.ub_seg = 0;
      for (int g = 0; g < n_seg; ++g) mb.ub_seg = std::max(mb.ub_seg, s->h_seg[g + 1] - s->h_seg[g]);
      QX_TRY((qxm::merge_large<double, u64>(s, mb, 0.0, QX_K_REDUCE, false, QX_K_DENSE_PREP, QX_K_DENSE_PREP)));
      sorted = mb.cur;
    }
    {
      QxProfileScope prof(QX_K_DENSE_PREP, s->stream, 48.0 * (double)n);
      k_group_scan<<<(unsigned)src_tiles, kThreads, 0, s->stream>>>(
          cwb[sorted], idb[sorted], s->keys[in], s->lam[in], s->seg[in], n_seg, n, skey, slam, gsrc, gslot,
          seg_slot, totals, st_heads, st_slots, ticket1, ct);
      QX_CUDA(cudaGetLastError());
    }
  }
  // slot offsets of the generators + totals -> host (sizes the output); the groups go along for
  // planner of the bucketed step and for the mode-by-mode sums of groups with many sources
  const bool bucket_ok = bucket_enabled() && eps > 0.0;
  qxb::bucket_stats().cap = 0;
  u64* h_groups = nullptr;
  struct ReleasePinned {
    void* p;
    ~ReleasePinned() { if (p) qx_pinned_free(p); }
  } relg{nullptr};
  static const bool no_kron = getenv("QX_NO_KRON") != nullptr;
  if (bucket_ok || !no_kron) {
    QX_TRY(qx_pinned_alloc(reinterpret_cast<void**>(&h_groups), 8ll * (2 + 3 * (qxb::kNgCap + 1))));
    relg.p = h_groups;
    k_group_export<<<(qxb::kNgCap + 1 + 255) / 256, 256, 0, s->stream>>>(cwb[sorted], gsrc, gslot, totals, h_groups,
                                                                       qxb::kNgCap);
    qx_count_launches(1);
    QX_CUDA(cudaGetLastError());
  }
  QX_TRY(qx_readback(s->stream, s->h_pinned, seg_slot, (int64_t)n_seg + 1));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  g_dense_last[0] = h_groups ? (int64_t)h_groups[0] : -1;
  g_dense_last[1] = g_dense_last[2] = g_dense_last[3] = 0;
  const int64_t total = s->h_pinned[n_seg];
  int64_t ub_seg = 0;
  for (int g = 0; g < n_seg; ++g) ub_seg = std::max(ub_seg, s->h_pinned[g + 1] - s->h_pinned[g]);
  if (slots_total) *slots_total = total;
  if (probe_fanout > 0 && !(ub_seg > QX_SMALL_MAX && total >= probe_fanout * n)) return QX_OK;
  if (done) *done = true;
  // the sources live in skey/slam now: both store buffers are free for the output
  QX_TRY(qx_store_reserve(s, total, false));
  const int out = s->cur ^ 1;

  // ---- bucketed step: slots leave the kernel in canonical order, no sort (bucket.cuh)
  if (bucket_ok && h_groups[0] >= 1 && h_groups[0] <= (u64)qxb::kNgCap && ub_seg > QX_SMALL_MAX) {
    const int ng = (int)h_groups[0];
    const u64* h_cw = h_groups + 2;
    const u64* h_src = h_cw + (qxb::kNgCap + 1);
    const u64* h_slot = h_src + (qxb::kNgCap + 1);
    std::vector<int64_t> h_seg_slot(s->h_pinned, s->h_pinned + n_seg + 1);   // the step reuses h_pinned
    // a store that is only downloaded next: 32-bit keys (want_narrow 1), or -- large results, form
    // 2 -- 64-bit keys that are packed to 16-bit halves + bucket tables right behind the step
    const int64_t bnd_room = 4ll * n_seg * (QX_PACK_BUCKETS + 1) + (2 * total + 255) / 256 * 256;
    const bool will_pack = s->n_qubits <= 16 && s->want_narrow == 2 && total >= 8ll * n_seg * QX_PACK_BUCKETS &&
                           ub_seg < (1ll << 32) - 1 && bnd_room <= 8 * s->cap;
    const bool narrow_out = s->n_qubits <= 16 && s->want_narrow != 0 && !will_pack;
    bool handled = false;
    if (s->n_qubits <= 16) {
      ImageTable<u32> im;
      fill_images_u32(s->n_qubits, program, n_ops, cx_c, cx_t, cx_s, &im);
      QX_TRY((qxb::bucket_step<u32>(s, ct, im, ng, h_cw, h_src, h_slot, h_seg_slot.data(), total, skey, slam, n, out,
                                    narrow_out, eps, part, parts, &handled)));
    } else {
      ImageTable<u64> im;
      fill_images_u64(s->n_qubits, program, n_ops, cx_c, cx_t, cx_s, &im);
      QX_TRY((qxb::bucket_step<u64>(s, ct, im, ng, h_cw, h_src, h_slot, h_seg_slot.data(), total, skey, slam, n, out,
                                    false, eps, part, parts, &handled)));
    }
    if (handled) {
      s->cur = out;
      s->exact = false;
      s->ub_total = total;
      s->ub_seg = ub_seg;
      s->narrow_keys = narrow_out;
      s->pack_bnd = nullptr;
      QX_TRY(qx_store_refresh(s));                  // kept counts: exact offsets for the caller
      if (will_pack) {
        bool packed = false;
        int64_t kept_max = 0;
        for (int g = 0; g < n_seg; ++g) kept_max = std::max(kept_max, s->h_seg[g + 1] - s->h_seg[g]);
        QX_TRY(pack_for_download(s, s->h_seg[n_seg], kept_max, &packed));
      }
      return QX_OK;
    }
  }

  const int64_t tiles = std::max<int64_t>(1, (total + kTileSlots - 1) / kTileSlots);
  const int passes = std::min(qxm::kMaxPasses, (2 * s->n_qubits + QX_RADIX_BITS - 1) / QX_RADIX_BITS);
  const int64_t hist_words = (int64_t)n_seg * passes * QX_RADIX;
  const int64_t bytes2 = padded(8 * tiles) + padded(8 * (int64_t)n_seg) + padded(4 * hist_words);
  void* block2 = nullptr;
  QX_TRY(qx_dev_alloc(&block2, bytes2, s->stream, s->device));
  Release rel2{block2, s->stream};
  cur = reinterpret_cast<char*>(block2);
  int2* tile_info = carve<int2>(cur, tiles);
  u64* seg_count = carve<u64>(cur, n_seg);
  u32* hist = carve<u32>(cur, hist_words);
  QX_CUDA(cudaMemsetAsync(seg_count, 0, (size_t)(padded(8 * (int64_t)n_seg) + 4 * hist_words), s->stream));
  k_tile_groups<<<(unsigned)((tiles + 255) / 256), 256, 0, s->stream>>>(gslot, totals, seg_slot, n_seg, tile_info, tiles);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());

  const bool small_keys = s->n_qubits <= 16;
  static const bool no_narrow = getenv("QX_NO_NARROW") != nullptr;
  const bool narrow = small_keys && !no_narrow && ub_seg > QX_SMALL_MAX;

  // ---- groups with many sources on few digits: their sums mode by mode, ahead of the slot kernel
  const int64_t* d_pre_off = nullptr;
  const double* d_pre = nullptr;
  void* block3 = nullptr;
  Release rel3{nullptr, s->stream};
  if (!no_kron && h_groups && h_groups[0] >= 1 && h_groups[0] <= (u64)qxb::kNgCap) {
    const int ng = (int)h_groups[0];
    const u64* h_cw = h_groups + 2;
    const u64* h_src = h_cw + (qxb::kNgCap + 1);
    const u64* h_slot = h_src + (qxb::kNgCap + 1);
    std::vector<int64_t> off((size_t)ng, -1), toff;
    std::vector<int> flagged, big;               // tensor in shared memory (<= 8 digits) / in global memory
    int64_t pre_total = 0, tensor_total = 0, max_src = 0;
    int w_max = 0;
    constexpr int64_t kTensorCap = 1ll << 26;    // doubles per ping-pong buffer (512 MB)
    for (int g = 0; g < ng; ++g) {
      const double n_src = (double)(h_src[g + 1] - h_src[g]), slots = (double)(h_slot[g + 1] - h_slot[g]);
      const u64 sup = (h_cw[g] | (h_cw[g] >> 1)) & 0x5555555555555555ull;
      const int w = __builtin_popcountll(sup);
      if (n_src < kBlockedMin || w < 1 || w > kKronWideDigits || slots < 1) continue;
      int64_t tensor = 1;
      for (int j = 0; j < w; ++j) tensor *= 3;
      // worth it when the factored sum's (source block, slot) pairs outnumber the contraction's terms
      static const double factor = getenv("QX_KRON_FACTOR") ? atof(getenv("QX_KRON_FACTOR")) : 0.25;
      if (n_src * slots / 16.0 < factor * (3.0 * w * (double)tensor + n_src)) continue;
      if (w > kKronDigits) {
        if (tensor_total + tensor > kTensorCap) continue;
        toff.push_back(tensor_total);
        tensor_total += tensor;
        big.push_back(g);
        w_max = std::max(w_max, w);
        max_src = std::max<int64_t>(max_src, (int64_t)n_src);
      } else {
        flagged.push_back(g);
      }
      off[(size_t)g] = pre_total;
      pre_total += (int64_t)slots;
    }
    if (!flagged.empty() || !big.empty()) {
      const int64_t n_small = (int64_t)flagged.size(), n_big = (int64_t)big.size();
      const int64_t bytes3 = padded(8ll * ng) + padded(4 * (n_small + 1)) + padded(4 * (n_big + 1)) +
                             padded(8 * (n_big + 1)) + padded(8 * pre_total) + 2 * padded(8 * tensor_total);
      QX_TRY(qx_dev_alloc(&block3, bytes3, s->stream, s->device));
      rel3.p = block3;
      char* c3 = reinterpret_cast<char*>(block3);
      int64_t* d_off = carve<int64_t>(c3, ng);
      int* d_flag = carve<int>(c3, n_small + 1);
      int* d_big = carve<int>(c3, n_big + 1);
      int64_t* d_toff = carve<int64_t>(c3, n_big + 1);
      double* pre = carve<double>(c3, pre_total);
      double* ta = carve<double>(c3, tensor_total);
      double* tb2 = carve<double>(c3, tensor_total);
      QX_CUDA(cudaMemcpyAsync(d_off, off.data(), 8 * (size_t)ng, cudaMemcpyHostToDevice, s->stream));
      QxProfileScope prof(QX_K_DENSE_PREP, s->stream, 16.0 * (double)n + 8.0 * (double)pre_total);
      if (n_small > 0) {
        QX_CUDA(cudaMemcpyAsync(d_flag, flagged.data(), 4 * (size_t)n_small, cudaMemcpyHostToDevice, s->stream));
        const size_t kron_smem = 2 * (size_t)kKronSize * sizeof(double);
        if (small_keys) {
          static bool attr32 = false;
          if (!attr32) {
            QX_CUDA(cudaFuncSetAttribute(k_group_kron<u32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kron_smem));
            attr32 = true;
          }
          k_group_kron<u32><<<(unsigned)n_small, 256, kron_smem, s->stream>>>(cwb[sorted], skey, slam, gsrc, d_flag,
                                                                            d_off, pre, ct);
        } else {
          static bool attr64 = false;
          if (!attr64) {
            QX_CUDA(cudaFuncSetAttribute(k_group_kron<u64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kron_smem));
            attr64 = true;
          }
          k_group_kron<u64><<<(unsigned)n_small, 256, kron_smem, s->stream>>>(cwb[sorted], skey, slam, gsrc, d_flag,
                                                                            d_off, pre, ct);
        }
        qx_count_launches(1);
        QX_CUDA(cudaGetLastError());
      }
      if (n_big > 0) {
        QX_CUDA(cudaMemcpyAsync(d_big, big.data(), 4 * (size_t)n_big, cudaMemcpyHostToDevice, s->stream));
        QX_CUDA(cudaMemcpyAsync(d_toff, toff.data(), 8 * (size_t)n_big, cudaMemcpyHostToDevice, s->stream));
        if (small_keys)
          QX_TRY(launch_kron_wide<u32>(s, cwb[sorted], skey, slam, gsrc, d_big, d_toff, (int)n_big, w_max, max_src, ta,
                                       tb2, tensor_total, d_off, pre, ct));
        else
          QX_TRY(launch_kron_wide<u64>(s, cwb[sorted], skey, slam, gsrc, d_big, d_toff, (int)n_big, w_max, max_src, ta,
                                       tb2, tensor_total, d_off, pre, ct));
        flagged.insert(flagged.end(), big.begin(), big.end());
      }
      d_pre_off = d_off;
      d_pre = pre;
      g_dense_last[1] = (int64_t)flagged.size();
      g_dense_last[2] = pre_total;
      for (int g : flagged) g_dense_last[3] += (int64_t)(h_src[g + 1] - h_src[g]);
    }
  }
  {
    QxProfileScope prof(QX_K_DENSE_EMIT, s->stream, 16.0 * (double)n + (narrow ? 12.0 : 16.0) * (double)total);
    if (small_keys) {
      ImageTable<u32> im;
      memset(&im, 0, sizeof(im));
      if (n_ops > 0) fill_images_u32(s->n_qubits, program, n_ops, cx_c, cx_t, cx_s, &im);
#define QX_GE(KO, F) launch_group_emit<u32, KO, F>(s, tiles, cwb[sorted], skey, slam, gsrc, gslot, totals, \
                                                   tile_info, seg_slot, out, seg_count, hist, passes, eps, part, parts, d_pre_off, d_pre, ct, im)
      if (n_ops > 0 && narrow) QX_TRY((QX_GE(u32, true)));
      else if (n_ops > 0) QX_TRY((QX_GE(u64, true)));
      else if (narrow) QX_TRY((QX_GE(u32, false)));
      else QX_TRY((QX_GE(u64, false)));
#undef QX_GE
    } else {
      ImageTable<u64> im;
      memset(&im, 0, sizeof(im));
      if (n_ops > 0) {
        fill_images_u64(s->n_qubits, program, n_ops, cx_c, cx_t, cx_s, &im);
        QX_TRY((launch_group_emit<u64, u64, true>(s, tiles, cwb[sorted], skey, slam, gsrc, gslot, totals,
                                                  tile_info, seg_slot, out, seg_count, hist, passes, eps, part, parts, d_pre_off, d_pre, ct, im)));
      } else {
        QX_TRY((launch_group_emit<u64, u64, false>(s, tiles, cwb[sorted], skey, slam, gsrc, gslot, totals,
                                                   tile_info, seg_slot, out, seg_count, hist, passes, eps, part, parts, d_pre_off, d_pre, ct, im)));
      }
    }
  }
  k_counts_to_offsets<<<1, 32, 0, s->stream>>>(seg_count, n_seg, s->seg[out]);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  s->cur = out;
  s->exact = false;
  s->ub_total = total;
  s->ub_seg = ub_seg;
  // The sort only needs upper bounds from the host (it reads the offsets on the device), so it is
  // queued behind the slot kernel without waiting for the kept counts; instrumented runs wait,
  // so that the passes are booked with the bytes they really move.
  if (qx_profile_on()) QX_TRY(qx_store_refresh(s));
  // ---- canonical order: distinct words, nothing left to sum or drop
  qxm::MergeBuffers<double> mb;
  for (int b = 0; b < 2; ++b) {
    mb.keys[b] = s->keys[b];
    mb.vals[b] = s->lam[b];
    mb.seg[b] = s->seg[b];
  }
  mb.cur = s->cur;
  mb.n_seg = n_seg;
  mb.ub_total = s->ub_total;
  mb.ub_seg = s->ub_seg;
  // the kept terms of generator g sit at its slot offset; the first pass reads them from there
  // a store that is only downloaded next keeps its 32-bit keys: 12 bytes per term cross PCIe
  // instead of 16 and the host widens them while the copy runs (qx_store_download_narrow_async)
  const bool keep_narrow = narrow && s->want_narrow != 0;
  // ... or, for results large enough that the bucket tables do not matter (10 bytes per term on
  // the wire): 16-bit low halves + per generator the first position of every high half.  The
  // table sits in the output key block behind the halves (8 bytes of room per term, 2 used).
  u32* pack_bnd = nullptr;
  const int64_t bnd_bytes = 4ll * n_seg * (QX_PACK_BUCKETS + 1);
  {
    const int passes_now = std::min(qxm::kMaxPasses, (2 * s->n_qubits + QX_RADIX_BITS - 1) / QX_RADIX_BITS);
    const int out_buf = mb.cur ^ (passes_now & 1);            // the buffer the last pass writes
    const int64_t lo_bytes = (2 * total + 255) / 256 * 256;
    // positions inside a generator are 32-bit in the bucket table: a generator of 2^32 terms
    // (n = 16, every word present) keeps 32-bit keys instead
    if (keep_narrow && s->want_narrow == 2 && total >= 8ll * n_seg * QX_PACK_BUCKETS && ub_seg < (1ll << 32) - 1 &&
        lo_bytes + bnd_bytes <= 8 * s->cap)
      pack_bnd = reinterpret_cast<u32*>(reinterpret_cast<char*>(s->keys[out_buf]) + lo_bytes);
  }
  if (narrow) QX_TRY((qxm::merge_large<double, u32>(s, mb, eps, QX_K_REDUCE, false, QX_K_SORT_PASS, QX_K_SORT_HIST, seg_slot, hist, !keep_narrow, pack_bnd)));
  else QX_TRY((qxm::merge_large<double, u64>(s, mb, eps, QX_K_REDUCE, false, QX_K_SORT_PASS, QX_K_SORT_HIST, seg_slot, hist)));
  s->cur = mb.cur;
  s->narrow_keys = keep_narrow;
  s->pack_bnd = pack_bnd;
  if (!s->exact) QX_TRY(qx_store_refresh(s));      // kept counts: exact offsets for the caller
  return QX_OK;
}
