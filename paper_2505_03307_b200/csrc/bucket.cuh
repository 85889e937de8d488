// a4 + a5 + a2 + a6 in ONE pass for operators whose groups are large boxes with few sources and
// whose Clifford run leaves the high key bits independent of a block of low qubits: the
// BUCKETED operator step.  The grouped step of dense.cu writes every kept slot once and then
// sorts the result (four onesweep passes for 2n = 32: 96 bytes moved per term to place 12).
// Here the slots leave the kernel already in canonical order, so the sort disappears.
//
// Reference semantics kept (bitwise): coefficient of a slot = sum over the group's sources, in
// input order, of lambda * prod_j w_j with the factors taken qubit 0 first
// (stabilizer.py:311-319); drop rule |sum| >= eps (stabilizer.py:336); ascending unique keys
// (stabilizer.py:337).  The CX run behind the operator (stabilizer.py:340-363) is composed in
// as images of the single-digit factors (expand.cuh).
//
// How.  A group (dense.cu) is a box: every non-identity digit of its class word picks one of the
// class's output axes.  Split a group's digits into the tile-local ones L (a run of the LOWEST
// digits, prod radix <= 729) and the high rest H.  A TILE is one choice of the H digits: <= 729
// slots.  The output word of a slot is  image(H picks) ^ image(L picks)  (conjugation is linear
// on the x/z bits), so if the images of the L digits only touch the low ELL bits of the word,
// the TOP bits of every slot of a tile are known from its H picks alone.  Tiles that share
// (generator, top bits) form a BUCKET; buckets in (generator, top) order are key ranges in
// canonical order.  One CTA per bucket:
//   1. for every tile of the bucket: mid table (the L digits above the lowest three, folded onto
//      the tile's precomputed high word / high products), then one thread per slot: three
//      multiplies per source, image composition, sign, drop rule; a kept slot sets bit
//      (word & (2^ELL - 1)) of a bitmap in shared memory and parks (low bits, sum) in slot order;
//   2. the keys of a generator's slots are DISTINCT (different groups never share an output
//      word, slots of a group are different words, the run is a bijection), so the rank of a
//      kept slot inside the bucket is the number of set bits below its own: one popcount scan
//      of the bitmap, then rank = prefix[word] + popc(bits below) -- no comparison sort;
//   3. the bucket's first output position comes from a decoupled look-back over the buckets in
//      order (one 64-bit status word per bucket), so the output is written compact, coalesced,
//      in final order, in the store's own format.
// What does not qualify (a group with >= 64 sources -> factored sums of dense.cu; images of the
// low digits that reach the top bits, e.g. a CX ladder running the other way; a bucket above
// the shared-memory cap) takes the grouped step + sort of dense.cu; results are identical.
#pragma once

#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "expand.cuh"
#include "merge.cuh"

namespace qxb {

using namespace qxe;

constexpr int kBThreads = 256;
constexpr int kBWarps = kBThreads / 32;
constexpr int kBRows = 3;                    // slots per thread per tile: tile <= kBRows * A
constexpr int kNgCap = 4096;                 // groups the host plans
constexpr int kMaxMid = 128;                 // mid entries per tile
#ifndef QX_BUCKET_ELL
#define QX_BUCKET_ELL 14
#endif
#ifndef QX_FLUSH_UNROLL
#define QX_FLUSH_UNROLL 1
#endif
constexpr int kFlushUnroll = QX_FLUSH_UNROLL;
constexpr int kEll = QX_BUCKET_ELL;          // low key bits ranked inside a bucket (7 digits)
static_assert(kEll >= 13 && kEll <= 16, "bitmap words per thread and 16-bit staged keys");
constexpr int kSrcChunk = 4;                 // sources folded per round
constexpr int kPerThread = 12;               // parked slots per thread
constexpr int kCapMax = kBThreads * kPerThread;   // slots per bucket (3072)
constexpr int kSrcMax = 63;                  // sources per group (above: factored sums of dense.cu)
constexpr int kTileIdBits = 40;

template <typename K>
struct __align__(16) BGroup {                // one per group, planned on the host
  K cw;                // class word
  K l_mask;            // support bits (even positions) of the tile-local digits
  K h_mask;            // support bits of the high digits
  u32 src0, n_src;     // its sorted sources
  u32 seg;
  u32 T;               // slots per tile
  u32 Lw, n_mid;       // low branches (<= 27), mid entries
  u32 pad;
  u64 tile0;           // id of its first tile
  u64 phi0;            // its first high product
};

template <typename K>
struct __align__(16) TileDesc {
  K word;              // image of the high picks
  u32 e;               // its phase exponent
  u32 group;
};

template <typename K> struct __align__(16) BMid {
  K word;
  u32 e;
  u32 picks;           // two bits per mid digit
};
template <typename K> struct __align__(16) BLow {
  K word;
  K imx;
  u32 e;
  u32 picks;
};

// ---- tiles: high picks -> image word, bucket key, high products ------------------------------
template <typename K>
__global__ void __launch_bounds__(256)
k_tile_desc(const BGroup<K>* __restrict__ groups, int ng, u64 n_tiles, const u64* __restrict__ skey,
            const double* __restrict__ slam, TileDesc<K>* __restrict__ desc, double* __restrict__ phi,
            u64* __restrict__ sort_key, double* __restrict__ sort_val, int ell, int top_bits,
            const __grid_constant__ OperatorTable tb, const __grid_constant__ ImageTable<K> im) {
  const u64 t = (u64)blockIdx.x * 256 + threadIdx.x;
  if (t >= n_tiles) return;
  int lo = 0, hi = ng;                          // groups[lo].tile0 <= t < groups[hi].tile0
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (groups[mid].tile0 <= t) lo = mid; else hi = mid;
  }
  const BGroup<K> g = groups[lo];
  u64 h = t - g.tile0;
  const u64 h_index = h;
  K picks = 0;                                  // two bits per high digit
  for (K m = g.h_mask; m;) {
    const int bit = KeyOps<K>::lowest(m);
    m &= m - 1;
    const u32 c = tb.cnt[bit >> 1][(u32)((g.cw >> bit) & 3u) - 1u];
    const u32 pick = (u32)(h % c);
    h /= c;
    picks |= (K)pick << bit;
  }
  K word = 0;
  u32 e = 0;
  for (K m = g.h_mask; m;) {                    // qubit 0 first (stabilizer.py:311-319)
    const int bit = KeyOps<K>::highest(m);
    m ^= (K)1 << bit;
    const u32 ax = tb.axis[bit >> 1][(u32)((g.cw >> bit) & 3u) - 1u][(u32)(picks >> bit) & 3u];
    compose<K>(word, e, im.img[bit >> 1][ax - 1], im.imx[bit >> 1][ax - 1], im.e[bit >> 1][ax - 1]);
  }
  TileDesc<K> d;
  d.word = word;
  d.e = e & 3u;
  d.group = (u32)lo;
  desc[t] = d;
  for (u32 s = 0; s < g.n_src; ++s) {
    const K key = (K)skey[g.src0 + s];
    double v = slam[g.src0 + s];
    for (K m = g.h_mask; m;) {
      const int bit = KeyOps<K>::highest(m);
      m ^= (K)1 << bit;
      v = __dmul_rn(v, tb.w[bit >> 1][(u32)((key >> bit) & 3u) - 1u][(u32)(picks >> bit) & 3u]);
    }
    phi[g.phi0 + h_index * g.n_src + s] = v;
  }
  sort_key[t] = ((u64)g.seg << top_bits) | (u64)(word >> ell);
  sort_val[t] = __longlong_as_double((long long)(t | ((u64)g.T << kTileIdBits)));
}

// ---- tile records of the bucket kernel -------------------------------------------------------------
// Everything a CTA needs to start a tile, in sorted (bucket) order: one coalesced load per bucket
// instead of the chain tile id -> descriptor -> group -> sources.  The first 16 bytes are what
// every thread reads; the rest is for the threads that build the tile's tables.
template <typename K>
struct __align__(16) TileFat {
  u32 shape, group, n_src, T;   // Lw | n_mid << 8 | (tables reusable across the group's tiles) << 16; group; sources; slots
  K word;              // image of the high picks
  K cw;                // class word of the group
  K l_mask;            // its tile-local digits
  u32 e;               // phase exponent of `word`
  K key01[2];          // keys of the group's first two sources
  u32 src0, pad;
  u64 phi_at;          // index of the tile's first high product
  double phi01[2];     // high products of the first two sources
  u64 pad2;
};

struct __align__(16) UnitHdr {
  u32 tile0, n_tiles;  // its tiles in sorted order
  u64 top;             // (generator, top bits): the sort key of its tiles
};

// sorted tile i -> its self-contained record (done inside k_unit_scan: one launch less)
template <typename K>
__device__ __forceinline__ void make_tile_fat(const BGroup<K>* __restrict__ groups, const TileDesc<K>* __restrict__ desc,
                                              const double* __restrict__ phi, const double* __restrict__ sort_val,
                                              const u64* __restrict__ skey, u64 i, TileFat<K>* __restrict__ fat) {
  const u64 tile = (u64)__double_as_longlong(sort_val[i]) & (((u64)1 << kTileIdBits) - 1);
  const TileDesc<K> d = desc[tile];
  const BGroup<K> g = groups[d.group];
  TileFat<K> f;
  f.word = d.word;
  f.cw = g.cw;
  f.l_mask = g.l_mask;
  f.e = d.e;
  f.src0 = g.src0;
  f.pad = 0;
  f.pad2 = 0;
  f.n_src = g.n_src;
  f.T = g.T;
  {
    K mid_mask = g.l_mask;                       // tile-local digits above the three lowest
    mid_mask &= mid_mask - 1;
    mid_mask &= mid_mask - 1;
    mid_mask &= mid_mask - 1;
    const u32 reusable = g.n_src <= 2 && Plane<K>::popc(mid_mask) <= 3 ? 1u : 0u;
    f.shape = g.Lw | (g.n_mid << 8) | (reusable << 16);
  }
  f.group = d.group;
  f.phi_at = g.phi0 + (tile - g.tile0) * g.n_src;
  f.key01[0] = (K)skey[g.src0];
  f.phi01[0] = phi[f.phi_at];
  f.key01[1] = g.n_src > 1 ? (K)skey[g.src0 + 1] : (K)0;
  f.phi01[1] = g.n_src > 1 ? phi[f.phi_at + 1] : 0.0;
  fat[i] = f;
}

// ---- buckets: heads of runs of equal (generator, top) among the sorted tiles ---------------------
//   unit_tile0[u] = first sorted tile of bucket u        (unit_tile0[NU] = n_tiles)
//   seg_first[g]  = first bucket of generator g          (untouched for a generator without slots)
//   info[0] = NU, info[1] = largest bucket (slots)
template <typename K>
__global__ void __launch_bounds__(256)
k_unit_scan(const u64* __restrict__ sort_key, const double* __restrict__ sort_val, u64 n_tiles, int top_bits,
            u32* __restrict__ unit_tile0, u32* __restrict__ seg_first, u64* __restrict__ status,
            u64* __restrict__ info, u32* __restrict__ ticket, const BGroup<K>* __restrict__ groups,
            const TileDesc<K>* __restrict__ desc, const double* __restrict__ phi, const u64* __restrict__ skey,
            TileFat<K>* __restrict__ fat) {
  __shared__ u64 s_scan[kBWarps + 1];
  __shared__ u64 s_base;
  const int tile = qx_tile_id(ticket);
  constexpr int kPer = 8;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const u64 wbase = (u64)tile * (256 * kPer) + (u64)warp * (32 * kPer);
  u32 pre[kPer];
  u32 flags = 0, run = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const u64 i = wbase + k * 32 + lane;
    bool head = false;
    if (i < n_tiles) {
      const u64 key = sort_key[i];
      head = i == 0 || sort_key[i - 1] != key;
      if (head) flags |= 1u << k;
      if (i == 0 || (sort_key[i - 1] >> top_bits) != (key >> top_bits)) flags |= 1u << (8 + k);
    }
    const u32 votes = __ballot_sync(QX_FULL_MASK, head);
    pre[k] = run + __popc(votes & lanemask_lt());
    run += __popc(votes);
    if (i < n_tiles) make_tile_fat<K>(groups, desc, phi, sort_val, skey, i, fat);
  }
  u64 tot;
  u64 wex = block_exclusive_sum<u64>(lane == 0 ? (u64)run : 0ull, s_scan, tot);
  wex = __shfl_sync(QX_FULL_MASK, wex, 0);
  if (warp == 0) {
    const u64 ex = lookback_exclusive(status, tile, tot);
    if (lane == 0) s_base = ex;
  }
  __syncthreads();
  const u64 base = s_base + wex;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const u64 i = wbase + k * 32 + lane;
    if (flags & (1u << k)) unit_tile0[base + pre[k]] = (u32)i;
    if (flags & (1u << (8 + k))) seg_first[(u32)(sort_key[i] >> top_bits)] = (u32)(base + pre[k]);
  }
  if ((u64)(tile + 1) * (256 * kPer) >= n_tiles && threadIdx.x == 0) {
    const u64 nu = s_base + tot;
    unit_tile0[nu] = (u32)n_tiles;
    info[0] = nu;
  }
}

struct UnitHdr;
// A bucket's record: UnitHdr followed by a copy of its first tile's TileFat (fat16 = the tile
// records as 16-byte words, fat_words of them per tile), so that one round trip behind the bucket
// id brings everything the first tile needs.
__global__ void k_unit_sizes(const u32* __restrict__ unit_tile0, const u64* __restrict__ sort_key,
                             const double* __restrict__ sort_val, uint4* __restrict__ hdr, u64* __restrict__ info,
                             const uint4* __restrict__ fat16, int fat_words) {
  const u64 nu = info[0];
  u32 worst = 0;
  for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += (u64)gridDim.x * blockDim.x) {
    u32 slots = 0;
    for (u32 i = unit_tile0[u]; i < unit_tile0[u + 1]; ++i)
      slots += (u32)((u64)__double_as_longlong(sort_val[i]) >> kTileIdBits);
    worst = max(worst, slots);
    const u32 first = unit_tile0[u];
    const u64 key = sort_key[first];
    uint4* rec = hdr + u * (u64)(1 + fat_words);
    rec[0] = make_uint4(first, unit_tile0[u + 1] - first, (u32)key, (u32)(key >> 32));   // UnitHdr
    for (int i = 0; i < fat_words; ++i) rec[1 + i] = fat16[(u64)first * fat_words + i];
  }
  worst = __reduce_max_sync(QX_FULL_MASK, worst);
  if (lane_id() == 0 && worst) atomicMax(reinterpret_cast<unsigned long long*>(info + 1), (unsigned long long)worst);
}

// generator offsets of the compact output from the inclusive prefixes the buckets left behind.
// One warp: a generator without slots takes the first bucket of the next one that has some (a fill
// from the right, 32 generators per round), then one status word per generator, all loads in
// flight at once (one thread walking the 2 x n_seg dependent loads took 9 us of the step).
__global__ void k_bucket_offsets(const u64* __restrict__ status, u32* __restrict__ seg_first, int n_seg,
                                 u32 u_lo, u32 u_hi, u32 n_units, int64_t* __restrict__ seg_out) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int lane = (int)threadIdx.x;
  u32 carry = n_units;
  for (int hi = n_seg; hi > 0; hi -= 32) {          // lane l <-> generator hi - 1 - l
    const int g = hi - 1 - lane;
    u32 v = g >= 0 ? seg_first[g] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 o = __shfl_up_sync(QX_FULL_MASK, v, d);
      if (v == 0xffffffffu && lane >= d) v = o;
    }
    if (v == 0xffffffffu) v = carry;
    if (g >= 0) seg_first[g] = v;
    carry = __shfl_sync(QX_FULL_MASK, v, min(31, hi - 1));
  }
  __syncwarp();
  for (int g = lane; g <= n_seg; g += 32) {
    u32 u = g < n_seg ? seg_first[g] : n_units;
    u = min(max(u, u_lo), u_hi);
    seg_out[g] = u == u_lo ? 0 : (int64_t)(status[u - 1 - u_lo] & QX_LB_VAL);
  }
}

#ifndef QX_BUCKET_TRIP
#define QX_BUCKET_TRIP 3
#endif
constexpr int kTrip = QX_BUCKET_TRIP;        // tiles whose slots a thread keeps in registers
constexpr int kHeld = kTrip * kBRows;        // 9

template <typename K>
struct BSmem {
  OperatorTable tb;                  // class-expanded (dense.cu build_class_table)
  ImageTable<K> im;
  BLow<K> low[2][27];                // low-digit tables, double-buffered: rebuilt when the group changes
  BLow<K> gmid[2][27];               // mid digits of the group alone (image word, picks), same buffering
  double gmid_w[2][2][27][4];        // [buffer][source][mid entry][mid digit]: weights, 1.0 where absent
  BMid<K> mid[2][kMaxMid];
  double low_w[2][2][27][4];         // [buffer][source of the round][low branch][low digit]
  double p_mid[2][2][kMaxMid];       // [parity][source of the round][mid entry]: lambda * high * mid weights
  __align__(16) u32 warp_tot[kBWarps + 4];
  u64 base;
  u32 unit;
};

inline size_t bucket_smem_bytes(size_t fixed, int ell, int cap) {
  const size_t words = (size_t)1 << (ell - 5);
  return fixed + 4 * words + 2 * words + 8 * (size_t)cap + 2 * (size_t)cap + 64;
}

// status words of the buckets: bits 63-62 = 0 not counted yet, 1 kept count, 2 inclusive prefix
__device__ __forceinline__ void bucket_publish(u64* status, u32 idx, u64 kept) {
  st_volatile_u64(status + idx, (idx == 0 ? QX_LB_INC : QX_LB_AGG) | kept);
}
// all 32 lanes of one warp: exclusive prefix of bucket idx (its own count is published already)
__device__ __noinline__ u64 bucket_resolve(u64* status, u32 idx, u64 kept) {
  if (idx == 0) return 0;
#ifndef QX_BUCKET_LB_R
#define QX_BUCKET_LB_R 1         // status words per lane and round trip (windows of 32: 1.082 ms; 64: 1.091; 96: 1.105)
#endif
  constexpr int R = QX_BUCKET_LB_R;
  u64 excl = 0;
  int base = (int)idx - 1;
  bool done = false;
  while (!done) {
    u64 w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int t = base - r * 32 - (int)lane_id();
      w[r] = t >= 0 ? ld_volatile_u64(status + t) : QX_LB_INC;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!done) {
        const int t = base - r * 32 - (int)lane_id();
        while ((w[r] >> 62) == 0) w[r] = ld_volatile_u64(status + t);
        const u32 inc = __ballot_sync(QX_FULL_MASK, (w[r] >> 62) == 2);
        u64 v = w[r] & QX_LB_VAL;
        if (inc) {
          const int first = __ffs(inc) - 1;
          if ((int)lane_id() > first) v = 0;
          done = true;
        }
        excl += warp_sum(v);
      }
    }
    base -= 32 * R;
  }
  if (lane_id() == 0) st_volatile_u64(status + idx, QX_LB_INC | (excl + kept));
  return excl;
}

// One CTA per bucket, buckets handed out in order by a ticket.  A bucket's kept count is known
// only after all its sums, and its first output position needs the counts of every bucket
// before it: the CTA does not wait -- it publishes the count, keeps the ranked terms in shared
// memory, goes on with its NEXT bucket (whose sums stay in registers meanwhile) and writes the
// previous one out after that, when its predecessors have long published theirs.
#ifndef QX_BUCKET_MINB
#define QX_BUCKET_MINB 4
#endif
template <typename K, typename KO>
__global__ void __launch_bounds__(kBThreads, QX_BUCKET_MINB)
k_bucket_emit(const TileFat<K>* __restrict__ fat, const double* __restrict__ phi,
              const uint4* __restrict__ units, u32 u_lo, u32 u_hi, const u64* __restrict__ skey,
              KO* __restrict__ keys_out, double* __restrict__ lam_out, u64* __restrict__ status,
              u32* __restrict__ ticket, int ell, int top_bits, int cap, double eps,
              const __grid_constant__ OperatorTable tb, const __grid_constant__ ImageTable<K> im) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BSmem<K>& sm = *reinterpret_cast<BSmem<K>*>(smem_raw);
  // the low key bits ranked inside a bucket are fixed at compile time (kEll): bitmap, prefix and
  // the coefficients of the staging area sit at constant offsets, the scan has one shape
  (void)ell;
  constexpr int ell_c = kEll;
  constexpr int words = 1 << (kEll - 5);
  u32* bitmap = reinterpret_cast<u32*>(smem_raw + ((sizeof(BSmem<K>) + 15) & ~(size_t)15));
  unsigned short* prefix = reinterpret_cast<unsigned short*>(bitmap + words);
  double* st_lam = reinterpret_cast<double*>(prefix + words);
  unsigned short* st_key = reinterpret_cast<unsigned short*>(st_lam + cap);
  const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
  {
    const u32* src = reinterpret_cast<const u32*>(&tb);
    u32* dst = reinterpret_cast<u32*>(&sm.tb);
    for (int i = tid; i < (int)(sizeof(OperatorTable) / 4); i += kBThreads) dst[i] = src[i];
    const u32* isrc = reinterpret_cast<const u32*>(&im);
    u32* idst = reinterpret_cast<u32*>(&sm.im);
    for (int i = tid; i < (int)(sizeof(ImageTable<K>) / 4); i += kBThreads) idst[i] = isrc[i];
  }
  constexpr K low_bits = (K)(((u64)1 << ell_c) - 1);
  const u64 top_mask = ((u64)1 << top_bits) - 1;
  int par = 0;
  bool pending = false;                          // a ranked bucket sits in st_key / st_lam
  u32 pend_idx = 0, pend_kept = 0;
  u64 pend_top = 0;
  // my column of a tile: low branch my_bl, first mid entry my_m0; row k adds bpr mid entries.
  // Depends on the tile's Lw only, which rarely changes from one tile to the next.
  u32 geo_Lw = 0, bpr = 0, A = 0, my_m0 = 0, my_bl = 0, geo_live = 0;   // geo_Lw: Lw | n_mid << 8
  // tables of the low digits (and, where the group allows, of its mid digits) stay in shared memory
  // from tile to tile of one group; lpar = the buffer in use
  u32 cur_group = 0xffffffffu;
  int lpar = 0;

  // the previous bucket: first output position, then out (coalesced, final order, store format)
  auto flush_pending = [&]() {
    // (a look-back by the whole CTA -- 2048 status words per round trip instead of 256 by one warp --
    // was slower: the status loads of all threads sit in registers next to the held sums, which
    // spills, and the extra L2 reads cost more than the dependent round trips they save)
    if (warp == 0) {
      const u64 ex = bucket_resolve(status, pend_idx, (u64)pend_kept);
      if (lane == 0) sm.base = ex;
    }
    __syncthreads();
    KO* kp = keys_out + (int64_t)sm.base + tid;
    double* lp = lam_out + (int64_t)sm.base + tid;
#pragma unroll kFlushUnroll
    for (u32 r = (u32)tid; r < pend_kept; r += kBThreads, kp += kBThreads, lp += kBThreads) {
      st_stream(kp, (KO)(pend_top | (u64)st_key[r]));
      st_stream(lp, st_lam[r]);
    }
    __syncthreads();
    pending = false;
  };

  // A bucket id is taken when the previous bucket has been written out, right before the ranks of
  // the current one are applied: the atomic's round trip hides behind that step.  Not earlier: a
  // CTA that holds an id while it WAITS for its predecessors (flush_pending) leaves that bucket
  // uncounted for as long, and the look-back of every bucket behind it stalls on it.
  if (tid == 0) sm.unit = u_lo + atomicAdd(ticket, 1u);
  for (;;) {
    __syncthreads();                              // ranks of the previous bucket taken; tables copied; id visible
    const u32 unit = sm.unit;
    if (unit >= u_hi) break;
    constexpr u32 kRecWords = 1u + (u32)(sizeof(TileFat<K>) / 16);
    const uint4* rec = units + (size_t)unit * kRecWords;        // UnitHdr + its first tile (k_unit_sizes)
    const uint4 hdr = rec[0];
    const TileFat<K>* first_tile = reinterpret_cast<const TileFat<K>*>(rec + 1);
    const u32 t_begin = hdr.x, t_end = hdr.x + hdr.y;
    const u32 n_tiles_unit = hdr.y;
    const u64 unit_top = (u64)hdr.z | ((u64)hdr.w << 32);
    const bool slow = n_tiles_unit > (u32)kTrip;  // more tiles than the registers hold: park them
    for (int i = tid; i < words; i += kBThreads) bitmap[i] = 0u;
    if (n_tiles_unit > 1) {                       // descriptors of the later tiles: on their way to L1
      const u32 bytes = (min(n_tiles_unit, (u32)kTrip) - 1u) * (u32)sizeof(TileFat<K>);
      if ((u32)tid * 32u < bytes)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(fat + t_begin + 1) + tid * 32));
    }
    if (slow && pending) flush_pending();         // parking needs the staging area
    u32 parked = 0;
    double held[kHeld];
    // low key bits of the held slots, two per register (ELL <= 16)
    u32 held_y[(kHeld + 1) / 2];
    auto put_y = [&](int i, u32 y) {               // i is a compile-time constant where this is called
      if (i & 1) held_y[i >> 1] = (held_y[i >> 1] & 0xffffu) | (y << 16);
      else held_y[i >> 1] = (held_y[i >> 1] & 0xffff0000u) | y;
    };
    auto get_y = [&](int i) -> u32 { return (i & 1) ? held_y[i >> 1] >> 16 : held_y[i >> 1] & 0xffffu; };

    for (u32 t0 = t_begin; t0 < t_end; t0 += kTrip) {
#pragma unroll
      for (int k = 0; k < kHeld; ++k) held[k] = 0.0;
#pragma unroll
      for (int t = 0; t < kTrip; ++t) {
        if (t0 + t >= t_end) continue;            // uniform
        const TileFat<K>* tfp = (t == 0 && t0 == t_begin) ? first_tile : fat + (t0 + t);
        const uint4 geo = *reinterpret_cast<const uint4*>(tfp);
        const u32 Lw = geo.x & 0xffu, n_mid = (geo.x >> 8) & 0xffu, n_src = geo.z;
        const bool reusable = (geo.x >> 16) != 0u;
        const bool fresh = !reusable || geo.y != cur_group;   // uniform: the tables have to be built
        if (fresh) {
          lpar ^= 1;
          cur_group = reusable ? geo.y : 0xffffffffu;
        }
        const u32 ns2 = min(n_src, 2u);
        if ((geo.x & 0xffffu) != geo_Lw) {        // uniform
          geo_Lw = geo.x & 0xffffu;
          const u32 magic = 65536u / Lw + 1u;     // t / Lw == (t * magic) >> 16 for t < 2^16 / Lw
          bpr = ((u32)kBThreads * magic) >> 16;   // mid entries per row
          A = bpr * Lw;                           // slots per row
          my_m0 = ((u32)tid * magic) >> 16;
          my_bl = (u32)tid - my_m0 * Lw;
          geo_live = 0;
          if ((u32)tid < A) {
#pragma unroll
            for (int k = 0; k < kBRows; ++k)
              if (my_m0 + (u32)k * bpr < n_mid) geo_live |= 1u << k;
          }
        }
        // ---- tables of the tile: mid entries by the first threads, low branches by warp 4
        if ((u32)tid < n_mid && reusable) {
          // the group's mid digits on their own (once per group), then per tile: image of the high
          // picks x that word, high product x the three weights (qubit 0 first; 1.0 is exact)
          if (fresh) {
            const K cwg = tfp->cw;
            const K key0 = tfp->key01[0], key1 = tfp->key01[1];
            K mm = tfp->l_mask;
            mm &= mm - 1;
            mm &= mm - 1;
            mm &= mm - 1;
            u32 b = (u32)tid, picks = 0;
            K w = 0;
            u32 ex = 0;
            int mbit[3];
            u32 pick[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              mbit[j] = -1;
              pick[j] = 0;
              if (mm) {
                mbit[j] = KeyOps<K>::lowest(mm);
                mm &= mm - 1;
                u32 q;
                divmod_small<u32>(b, sm.tb.cnt[mbit[j] >> 1][(u32)((cwg >> mbit[j]) & 3u) - 1u], q, pick[j]);
                b = q;
                picks |= pick[j] << (2 * j);
              }
            }
#pragma unroll
            for (int j = 2; j >= 0; --j) {
              double w0 = 1.0, w1 = 1.0;
              if (mbit[j] >= 0) {
                const int p = mbit[j] >> 1;
                const u32 ax = sm.tb.axis[p][(u32)((cwg >> mbit[j]) & 3u) - 1u][pick[j]];
                compose<K>(w, ex, sm.im.img[p][ax - 1], sm.im.imx[p][ax - 1], sm.im.e[p][ax - 1]);
                w0 = sm.tb.w[p][(u32)((key0 >> mbit[j]) & 3u) - 1u][pick[j]];
                if (ns2 > 1) w1 = sm.tb.w[p][(u32)((key1 >> mbit[j]) & 3u) - 1u][pick[j]];
              }
              sm.gmid_w[lpar][0][tid][j] = w0;
              sm.gmid_w[lpar][1][tid][j] = w1;
            }
            BLow<K> ge;
            ge.word = w;
            ge.imx = (w ^ (w >> 1)) & Plane<K>::lo;
            ge.e = ex & 3u;
            ge.picks = picks;
            sm.gmid[lpar][tid] = ge;                // read back by this thread only
          }
          const BLow<K> ge = sm.gmid[lpar][tid];
          K w = tfp->word;
          u32 ex = tfp->e;
          compose<K>(w, ex, ge.word, ge.imx, ge.e);
          const double2 a01 = *reinterpret_cast<const double2*>(&sm.gmid_w[lpar][0][tid][0]);
          double v0 = __dmul_rn(tfp->phi01[0], sm.gmid_w[lpar][0][tid][2]);
          v0 = __dmul_rn(v0, a01.y);
          v0 = __dmul_rn(v0, a01.x);
          double v1 = 0.0;
          if (ns2 > 1) {
            const double2 b01 = *reinterpret_cast<const double2*>(&sm.gmid_w[lpar][1][tid][0]);
            v1 = __dmul_rn(tfp->phi01[1], sm.gmid_w[lpar][1][tid][2]);
            v1 = __dmul_rn(v1, b01.y);
            v1 = __dmul_rn(v1, b01.x);
          }
          BMid<K> me;
          me.word = w;
          me.e = ex & 3u;
          me.picks = ge.picks;
          sm.mid[par][tid] = me;
          sm.p_mid[par][0][tid] = v0;
          sm.p_mid[par][1][tid] = v1;
        } else if ((u32)tid < n_mid) {
          const K cwg = tfp->cw;
          K mid_mask = tfp->l_mask;
          mid_mask &= mid_mask - 1;               // without the three lowest digits
          mid_mask &= mid_mask - 1;
          mid_mask &= mid_mask - 1;
          const K key0 = tfp->key01[0], key1 = tfp->key01[1];
          u32 b = (u32)tid, picks = 0;
          int idx = 0;
          for (K m = mid_mask; m; ++idx) {
            const int bit = KeyOps<K>::lowest(m);
            m &= m - 1;
            u32 q, r;
            divmod_small<u32>(b, sm.tb.cnt[bit >> 1][(u32)((cwg >> bit) & 3u) - 1u], q, r);
            picks |= r << (2 * idx);
            b = q;
          }
          K w = tfp->word;
          u32 ex = tfp->e;
          double v0 = tfp->phi01[0], v1 = tfp->phi01[1];
          --idx;
          for (K m = mid_mask; m; --idx) {          // qubit 0 first (stabilizer.py:311-319)
            const int bit = KeyOps<K>::highest(m);
            m ^= (K)1 << bit;
            const int p = bit >> 1;
            const u32 pick = (picks >> (2 * idx)) & 3u;
            const u32 ax = sm.tb.axis[p][(u32)((cwg >> bit) & 3u) - 1u][pick];
            compose<K>(w, ex, sm.im.img[p][ax - 1], sm.im.imx[p][ax - 1], sm.im.e[p][ax - 1]);
            v0 = __dmul_rn(v0, sm.tb.w[p][(u32)((key0 >> bit) & 3u) - 1u][pick]);
            if (ns2 > 1) v1 = __dmul_rn(v1, sm.tb.w[p][(u32)((key1 >> bit) & 3u) - 1u][pick]);
          }
          BMid<K> me;
          me.word = w;
          me.e = ex & 3u;
          me.picks = picks;
          sm.mid[par][tid] = me;
          sm.p_mid[par][0][tid] = v0;
          sm.p_mid[par][1][tid] = v1;
        } else if (fresh && tid >= 128 && (u32)(tid - 128) < Lw) {
          const int l = tid - 128;
          const K cwg = tfp->cw;
          const K key0 = tfp->key01[0], key1 = tfp->key01[1];
          K mm = tfp->l_mask;
          u32 b = (u32)l, picks = 0;
          K w = 0;
          u32 ex = 0;
          int lbit[3];
          u32 pick[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            lbit[j] = -1;
            pick[j] = 0;
            if (mm) {
              lbit[j] = KeyOps<K>::lowest(mm);
              mm &= mm - 1;
              u32 q;
              divmod_small<u32>(b, sm.tb.cnt[lbit[j] >> 1][(u32)((cwg >> lbit[j]) & 3u) - 1u], q, pick[j]);
              b = q;
              picks |= pick[j] << (2 * j);
            }
          }
#pragma unroll
          for (int j = 2; j >= 0; --j) {
            double w0 = 1.0, w1 = 1.0;
            if (lbit[j] >= 0) {
              const int p = lbit[j] >> 1;
              const u32 ax = sm.tb.axis[p][(u32)((cwg >> lbit[j]) & 3u) - 1u][pick[j]];
              compose<K>(w, ex, sm.im.img[p][ax - 1], sm.im.imx[p][ax - 1], sm.im.e[p][ax - 1]);
              w0 = sm.tb.w[p][(u32)((key0 >> lbit[j]) & 3u) - 1u][pick[j]];
              if (ns2 > 1) w1 = sm.tb.w[p][(u32)((key1 >> lbit[j]) & 3u) - 1u][pick[j]];
            }
            sm.low_w[lpar][0][l][j] = w0;
            sm.low_w[lpar][1][l][j] = w1;
          }
          BLow<K> le;
          le.word = w;
          le.imx = (w ^ (w >> 1)) & Plane<K>::lo;
          le.e = ex & 3u;
          le.picks = picks;
          sm.low[lpar][l] = le;
        }
        __syncthreads();
        const u32 live = geo_live;
        double acc[kBRows];
#pragma unroll
        for (int k = 0; k < kBRows; ++k) acc[k] = 0.0;
        if (live) {
          // ((p * w2) * w1) * w0 with explicit roundings: no fused multiply-add into the sum
          {
            const double2 w01 = *reinterpret_cast<const double2*>(&sm.low_w[lpar][0][my_bl][0]);
            const double w2 = sm.low_w[lpar][0][my_bl][2];
            const double* pm = &sm.p_mid[par][0][my_m0];
#pragma unroll
            for (int k = 0; k < kBRows; ++k) {
              if (live & (1u << k)) {
                double v = __dmul_rn(pm[(u32)k * bpr], w2);
                v = __dmul_rn(v, w01.y);
                acc[k] = __dmul_rn(v, w01.x);
              }
            }
          }
          if (ns2 > 1) {
            const double2 w01 = *reinterpret_cast<const double2*>(&sm.low_w[lpar][1][my_bl][0]);
            const double w2 = sm.low_w[lpar][1][my_bl][2];
            const double* pm = &sm.p_mid[par][1][my_m0];
#pragma unroll
            for (int k = 0; k < kBRows; ++k) {
              if (live & (1u << k)) {
                double v = __dmul_rn(pm[(u32)k * bpr], w2);
                v = __dmul_rn(v, w01.y);
                v = __dmul_rn(v, w01.x);
                acc[k] = __dadd_rn(acc[k], v);
              }
            }
          }
        }
        // further sources of the group, two per round, in input order (rare: the tables of the
        // round replace those of the first two behind a barrier)
        if (n_src > 2) {
          const K cwg = tfp->cw;
          K mid_mask = tfp->l_mask;
          int lbit[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            lbit[j] = -1;
            if (mid_mask) {
              lbit[j] = KeyOps<K>::lowest(mid_mask);
              mid_mask &= mid_mask - 1;
            }
          }
          const int n_mid_digits = (int)Plane<K>::popc(mid_mask);
          const u32 src0 = tfp->src0;
          const u64 phi_at = tfp->phi_at;
          (void)cwg;
#pragma unroll 1
          for (u32 c0 = 2; c0 < n_src; c0 += 2) {
            const u32 nc = min(2u, n_src - c0);
            __syncthreads();
            for (u32 w = (u32)tid; w < nc * n_mid; w += kBThreads) {
              const u32 c = w >= n_mid ? 1u : 0u, m = w - c * n_mid;
              const K key = (K)skey[src0 + c0 + c];
              const u32 picks = sm.mid[par][m].picks;
              double v = phi[phi_at + c0 + c];
              int idx = n_mid_digits - 1;
              for (K m2 = mid_mask; m2; --idx) {
                const int bit = KeyOps<K>::highest(m2);
                m2 ^= (K)1 << bit;
                v = __dmul_rn(v, sm.tb.w[bit >> 1][(u32)((key >> bit) & 3u) - 1u][(picks >> (2 * idx)) & 3u]);
              }
              sm.p_mid[par][c][m] = v;
            }
            for (u32 w = (u32)tid; w < nc * Lw; w += kBThreads) {
              const u32 c = w >= Lw ? 1u : 0u, l = w - c * Lw;
              const K key = (K)skey[src0 + c0 + c];
              const u32 picks = sm.low[lpar][l].picks;
#pragma unroll
              for (int j = 0; j < 3; ++j) {
                double wt = 1.0;
                if (lbit[j] >= 0)
                  wt = sm.tb.w[lbit[j] >> 1][(u32)((key >> lbit[j]) & 3u) - 1u][(picks >> (2 * j)) & 3u];
                sm.low_w[lpar][c][l][j] = wt;
              }
            }
            __syncthreads();
            if (live) {
              for (u32 c = 0; c < nc; ++c) {
                const double2 w01 = *reinterpret_cast<const double2*>(&sm.low_w[lpar][c][my_bl][0]);
                const double w2 = sm.low_w[lpar][c][my_bl][2];
                const double* pm = &sm.p_mid[par][c][my_m0];
#pragma unroll
                for (int k = 0; k < kBRows; ++k) {
                  if (live & (1u << k)) {
                    double v = __dmul_rn(pm[(u32)k * bpr], w2);
                    v = __dmul_rn(v, w01.y);
                    v = __dmul_rn(v, w01.x);
                    acc[k] = __dadd_rn(acc[k], v);
                  }
                }
              }
            }
          }
          __syncthreads();                          // the round tables are not double-buffered
        }
        // words, signs, drop rule; a kept slot marks the bitmap and stays in registers
        if (live) {
          const BLow<K> le = sm.low[lpar][my_bl];
#pragma unroll
          for (int k = 0; k < kBRows; ++k) {
            if (live & (1u << k)) {
              const BMid<K> me = sm.mid[par][my_m0 + (u32)k * bpr];
              K out = me.word;
              u32 ex = me.e;
              compose<K>(out, ex, le.word, le.imx, le.e);
              double v = acc[k];
              if (composed_sign<K>(out, ex)) v = -v;            // sign flips are exact
              const u32 y = (u32)(out & low_bits);
              if (fabs(v) >= eps) {                              // eps > 0: a kept sum is never 0
                atomicOr(&bitmap[y >> 5], 1u << (y & 31u));
                held[t * kBRows + k] = v;
                put_y(t * kBRows + k, y);
              }
            }
          }
        }
        par ^= 1;
      }
      if (slow) {
        // park this triple in slot order (any order would do: ranks come from the bitmap); dropped
        // slots are parked as 0.0 so that nothing stale is taken for a kept sum later
        // (the tiles' geometry is read again here, not carried through the sums in registers: the
        // fast path -- buckets of at most kTrip tiles -- never needs it)
#pragma unroll
        for (int t = 0; t < kTrip; ++t) {
          if (t0 + t >= t_end) continue;          // uniform
          const uint4 geo = *reinterpret_cast<const uint4*>(fat + (t0 + t));
          const u32 Lw = geo.x & 0xffu, n_mid = (geo.x >> 8) & 0xffu;
          const u32 magic = 65536u / Lw + 1u;
          const u32 pb = ((u32)kBThreads * magic) >> 16;
          const u32 pm0 = ((u32)tid * magic) >> 16;
          const u32 pbl = (u32)tid - pm0 * Lw;
          if ((u32)tid < pb * Lw) {
#pragma unroll
            for (int k = 0; k < kBRows; ++k) {
              if (pm0 + (u32)k * pb < n_mid) {
                const u32 at = parked + (pm0 + (u32)k * pb) * Lw + pbl;
                st_key[at] = (unsigned short)get_y(t * kBRows + k);
                st_lam[at] = held[t * kBRows + k];
              }
            }
          }
          parked += geo.w;
        }
      }
    }
    __syncthreads();
    // ranks: popcount scan of the bitmap
    u32 kept_total;
    {
      u32 cnt, c0 = 0;
      constexpr int per = words / kBThreads;      // words is a power of two
      const int w0 = tid * per;
      if (per == 2) {
        const uint2 b = *reinterpret_cast<const uint2*>(bitmap + w0);
        c0 = __popc(b.x);
        cnt = c0 + __popc(b.y);
      } else {
        cnt = 0;
        if (per == 0) {
          if (tid < words) cnt = __popc(bitmap[tid]);
        } else {
          for (int i = 0; i < per; ++i) cnt += __popc(bitmap[w0 + i]);
        }
      }
      u32 incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 o = __shfl_up_sync(QX_FULL_MASK, incl, d);
        if (lane >= d) incl += o;
      }
      if (lane == 31) sm.warp_tot[warp] = incl;
      __syncthreads();
      const uint4 ta = *reinterpret_cast<const uint4*>(&sm.warp_tot[0]);
      const uint4 tb4 = *reinterpret_cast<const uint4*>(&sm.warp_tot[4]);
      const u32 wt[kBWarps] = {ta.x, ta.y, ta.z, ta.w, tb4.x, tb4.y, tb4.z, tb4.w};
      u32 before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kBWarps; ++w) {
        if (w < warp) before += wt[w];
        total += wt[w];
      }
      kept_total = total;
      u32 run = before + incl - cnt;
      if (per == 2) {
        *reinterpret_cast<u32*>(prefix + w0) = run | ((run + c0) << 16);
      } else if (per == 0) {
        if (tid < words) prefix[tid] = (unsigned short)run;
      } else {
        for (int i = 0; i < per; ++i) {
          prefix[w0 + i] = (unsigned short)run;
          run += __popc(bitmap[w0 + i]);
        }
      }
    }
    if (tid == 0) bucket_publish(status, unit - u_lo, (u64)kept_total);
    if (!slow) {
      if (pending) flush_pending();               // barriers inside: prefix[] is visible after them
      else __syncthreads();
      if (tid == 0) sm.unit = u_lo + atomicAdd(ticket, 1u);   // every thread has read this bucket's id long ago
      // kept sums -> rank order in the staging area
#pragma unroll
      for (int t = 0; t < kTrip; ++t) {
        if ((u32)t < n_tiles_unit) {              // uniform
#pragma unroll
          for (int k = 0; k < kBRows; ++k) {
            const double v = held[t * kBRows + k];
            if (v != 0.0) {
              const u32 y = get_y(t * kBRows + k);
              const u32 r = (u32)prefix[y >> 5] + __popc(bitmap[y >> 5] & ((1u << (y & 31u)) - 1u));
              st_key[r] = (unsigned short)y;
              st_lam[r] = v;
            }
          }
        }
      }
    } else {
      // parked slots -> rank order, in place through registers
      __syncthreads();
      if (tid == 0) sm.unit = u_lo + atomicAdd(ticket, 1u);
      unsigned short rk[kPerThread];
      double rl[kPerThread];
#pragma unroll
      for (int j = 0; j < kPerThread; ++j) {
        const u32 i = (u32)tid + (u32)j * kBThreads;
        rl[j] = 0.0;
        rk[j] = 0;
        if (i < parked) {
          rl[j] = st_lam[i];
          rk[j] = st_key[i];
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kPerThread; ++j) {
        if (rl[j] != 0.0) {
          const u32 y = rk[j];
          const u32 r = (u32)prefix[y >> 5] + __popc(bitmap[y >> 5] & ((1u << (y & 31u)) - 1u));
          st_key[r] = rk[j];
          st_lam[r] = rl[j];
        }
      }
    }
    pending = true;
    pend_idx = unit - u_lo;
    pend_kept = kept_total;
    pend_top = (unit_top & top_mask) << ell_c;
  }
  if (pending) {
    __syncthreads();
    flush_pending();
  }
}

// ---- host side -------------------------------------------------------------------------------------
template <typename T>
inline T* bcarve(char*& cursor, int64_t count) {
  T* p = reinterpret_cast<T*>(cursor);
  cursor += (sizeof(T) * (size_t)count + 255) / 256 * 256;
  return p;
}
inline int64_t bpadded(int64_t bytes) { return (bytes + 255) / 256 * 256; }

struct BucketStats {           // what the last bucketed step did (qx_bucket_last, tools and tests)
  int64_t groups, tiles, units, max_unit, slots;
  int ell, cap, ctas_per_sm;
};
inline BucketStats& bucket_stats() {
  static BucketStats st = {};
  return st;
}

// Plan the groups for `ell` low bits.  Returns false if the operator does not qualify.
template <typename K>
bool plan_groups(int n_qubits, int n_seg, int ell, const OperatorTable& ct, const ImageTable<K>& im, int ng,
                 const u64* h_cw, const u64* h_gsrc, const u64* h_gslot, const int64_t* h_seg_slot,
                 std::vector<BGroup<K>>& out, u64* n_tiles, u64* n_phi) {
  out.resize((size_t)ng + 1);
  u64 tiles = 0, phis = 0;
  int seg = 0;
  for (int g = 0; g < ng; ++g) {
    BGroup<K> d;
    memset(&d, 0, sizeof(d));
    const K cw = (K)h_cw[g];
    const u64 n_src = h_gsrc[g + 1] - h_gsrc[g];
    const u64 slots = h_gslot[g + 1] - h_gslot[g];
    if (n_src == 0 || n_src > (u64)kSrcMax || slots == 0) return false;
    while (seg + 1 < n_seg && (u64)h_seg_slot[seg + 1] <= h_gslot[g]) ++seg;
    u32 T = 1, Lw = 1, n_mid = 1;
    int nl = 0;
    K l_mask = 0, h_mask = 0;
    bool open = true;
    for (int p = 0; p < n_qubits; ++p) {
      const u32 cls = (u32)((cw >> (2 * p)) & 3u);
      if (!cls) continue;
      const u32 radix = ct.cnt[p][cls - 1];
      if (open) {
        K infl = 0;
        for (u32 c = 0; c < radix; ++c) infl |= im.img[p][ct.axis[p][cls - 1][c] - 1];
        bool fits = ell >= (int)(8 * sizeof(K)) || (infl >> ell) == 0;
        if (fits) {
          if (nl < 3) {
            Lw *= radix;
          } else {
            const u32 nm = n_mid * radix;
            if (nm > (u32)kMaxMid || nm > (u32)kBRows * ((u32)kBThreads / Lw)) fits = false;
            else n_mid = nm;
          }
        }
        if (fits) {
          T *= radix;
          ++nl;
          l_mask |= (K)1 << (2 * p);
          continue;
        }
        open = false;
      }
      h_mask |= (K)1 << (2 * p);
    }
    d.cw = cw;
    d.l_mask = l_mask;
    d.h_mask = h_mask;
    d.src0 = (u32)h_gsrc[g];
    d.n_src = (u32)n_src;
    d.seg = (u32)seg;
    d.T = T;
    d.Lw = Lw;
    d.n_mid = n_mid;
    d.tile0 = tiles;
    d.phi0 = phis;
    out[g] = d;
    tiles += slots / T;
    phis += (slots / T) * n_src;
  }
  BGroup<K> end;
  memset(&end, 0, sizeof(end));
  end.tile0 = tiles;
  end.phi0 = phis;
  out[ng] = end;
  *n_tiles = tiles;
  *n_phi = phis;
  return true;
}

// The bucketed step.  On entry: sorted sources in skey/slam, groups on the host (class word, first
// source, first slot; ng + 1 entries of gsrc/gslot), slot offsets of the generators on the host,
// the output buffer `out` of the store can hold `total` terms.  *handled = false: nothing was
// written, take the grouped step + sort.  On success the store's buffer `out` holds the
// canonical result of this part and s->seg[out] its offsets.
template <typename K>
int bucket_step(qx_store* s, const OperatorTable& ct, const ImageTable<K>& im, int ng, const u64* h_cw,
                const u64* h_gsrc, const u64* h_gslot, const int64_t* h_seg_slot, int64_t total,
                const u64* skey, const double* slam, int64_t n_sources, int out, bool narrow_out, double eps,
                int part, int parts, bool* handled) {
  *handled = false;
  const int n_seg = s->n_seg;
  const int ell = kEll;
  const int top_bits = 2 * s->n_qubits - ell;
  if (top_bits <= 0 || ng <= 0 || ng > kNgCap || total <= 0) return QX_OK;
  int seg_bits = 1;
  while ((1ll << seg_bits) < n_seg) ++seg_bits;
  if (top_bits + seg_bits > 62) return QX_OK;
  std::vector<BGroup<K>> groups;
  u64 n_tiles = 0, n_phi = 0;
  if (!plan_groups<K>(s->n_qubits, n_seg, ell, ct, im, ng, h_cw, h_gsrc, h_gslot, h_seg_slot, groups, &n_tiles, &n_phi))
    return QX_OK;
  // tiles must be worth a CTA's while, and their ids must fit the payload of the tile sort
  if (n_tiles == 0 || n_tiles >= (1ull << 31) || (u64)total < 128 * n_tiles || n_phi > (1ull << 28)) return QX_OK;

  const int64_t scan_tiles = (int64_t)((n_tiles + 2047) / 2048);
  const int64_t bytes = bpadded((int64_t)sizeof(BGroup<K>) * (ng + 1)) + bpadded((int64_t)sizeof(TileDesc<K>) * (int64_t)n_tiles) +
                        bpadded(8 * (int64_t)n_phi) + 4 * bpadded(8 * (int64_t)n_tiles) + 2 * 256 +
                        bpadded(4 * ((int64_t)n_tiles + 1)) + bpadded(4 * (int64_t)n_seg) +
                        bpadded(8 * (scan_tiles + 1)) + 256 + bpadded(8 * ((int64_t)n_tiles + 1)) + 256 +
                        bpadded((int64_t)sizeof(TileFat<K>) * (int64_t)n_tiles) +
                        bpadded((16 + (int64_t)sizeof(TileFat<K>)) * ((int64_t)n_tiles + 1));
  void* block = nullptr;
  QX_TRY(qx_dev_alloc(&block, bytes, s->stream, s->device));
  struct Release {
    void* p;
    cudaStream_t st;
    ~Release() { qx_dev_free(p, st); }
  } rel{block, s->stream};
  char* cur = reinterpret_cast<char*>(block);
  BGroup<K>* d_groups = bcarve<BGroup<K>>(cur, ng + 1);
  TileDesc<K>* d_desc = bcarve<TileDesc<K>>(cur, (int64_t)n_tiles);
  double* d_phi = bcarve<double>(cur, (int64_t)n_phi);
  u64* skeys[2] = {bcarve<u64>(cur, (int64_t)n_tiles), bcarve<u64>(cur, (int64_t)n_tiles)};
  double* svals[2] = {bcarve<double>(cur, (int64_t)n_tiles), bcarve<double>(cur, (int64_t)n_tiles)};
  int64_t* sseg[2] = {bcarve<int64_t>(cur, 2), bcarve<int64_t>(cur, 2)};
  u32* unit_tile0 = bcarve<u32>(cur, (int64_t)n_tiles + 1);
  u32* seg_first = bcarve<u32>(cur, n_seg);
  u64* scan_status = bcarve<u64>(cur, scan_tiles + 1);
  u64* info = bcarve<u64>(cur, 2);
  u64* unit_status = bcarve<u64>(cur, (int64_t)n_tiles + 1);
  u32* ticket = bcarve<u32>(cur, 2);
  TileFat<K>* d_fat = bcarve<TileFat<K>>(cur, (int64_t)n_tiles);
  static_assert(sizeof(TileFat<K>) % 16 == 0, "tile records are copied as 16-byte words");
  constexpr int kFatWords = (int)(sizeof(TileFat<K>) / 16);
  uint4* d_units = bcarve<uint4>(cur, (1 + kFatWords) * ((int64_t)n_tiles + 1));

  // groups and the offsets of the one-segment tile sort: host -> device through pinned staging
  const int64_t stage_bytes = (int64_t)sizeof(BGroup<K>) * (ng + 1) + 16;
  void* h_stage = nullptr;
  QX_TRY(qx_pinned_alloc(&h_stage, stage_bytes));
  struct ReleasePinned {
    void* p;
    ~ReleasePinned() { qx_pinned_free(p); }
  } relp{h_stage};
  memcpy(h_stage, groups.data(), sizeof(BGroup<K>) * (size_t)(ng + 1));
  int64_t* h_off = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(h_stage) + sizeof(BGroup<K>) * (size_t)(ng + 1));
  h_off[0] = 0;
  h_off[1] = (int64_t)n_tiles;
  QX_CUDA(cudaMemcpyAsync(d_groups, h_stage, sizeof(BGroup<K>) * (size_t)(ng + 1), cudaMemcpyHostToDevice, s->stream));
  QX_CUDA(cudaMemcpyAsync(sseg[0], h_off, 16, cudaMemcpyHostToDevice, s->stream));
  QX_CUDA(cudaMemsetAsync(seg_first, 0xff, 4 * (size_t)n_seg, s->stream));
  QX_CUDA(cudaMemsetAsync(scan_status, 0, (size_t)(reinterpret_cast<char*>(ticket) + 256 - reinterpret_cast<char*>(scan_status)),
                          s->stream));
  int sorted = 0;
  {
    QxProfileScope prof(QX_K_DENSE_PREP, s->stream, 48.0 * (double)n_tiles + 16.0 * (double)n_sources);
    k_tile_desc<K><<<(unsigned)((n_tiles + 255) / 256), 256, 0, s->stream>>>(
        d_groups, ng, n_tiles, skey, slam, d_desc, d_phi, skeys[0], svals[0], ell, top_bits, ct, im);
    QX_CUDA(cudaGetLastError());
  }
  {
    // tiles into (generator, top bits) order: the merge's own onesweep, sort only, one segment
    qxm::MergeBuffers<double> mb;
    for (int b = 0; b < 2; ++b) {
      mb.keys[b] = skeys[b];
      mb.vals[b] = svals[b];
      mb.seg[b] = sseg[b];
    }
    mb.cur = 0;
    mb.n_seg = 1;
    mb.ub_total = (int64_t)n_tiles;
    mb.ub_seg = (int64_t)n_tiles;
    QX_TRY((qxm::merge_large<double, u64>(s, mb, 0.0, QX_K_REDUCE, false, QX_K_DENSE_PREP, QX_K_DENSE_PREP, nullptr,
                                          nullptr, true, nullptr, top_bits + seg_bits)));
    sorted = mb.cur;
  }
  {
    QxProfileScope prof(QX_K_DENSE_PREP, s->stream, 20.0 * (double)n_tiles + (double)sizeof(TileFat<K>) * (double)n_tiles, 2);
    k_unit_scan<K><<<(unsigned)scan_tiles, 256, 0, s->stream>>>(skeys[sorted], svals[sorted], n_tiles, top_bits,
                                                               unit_tile0, seg_first, scan_status, info, ticket + 1,
                                                               d_groups, d_desc, d_phi, skey, d_fat);
    QX_CUDA(cudaGetLastError());
    k_unit_sizes<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(((int64_t)n_tiles + 255) / 256, 1024)), 256, 0, s->stream>>>(
        unit_tile0, skeys[sorted], svals[sorted], d_units, info, reinterpret_cast<const uint4*>(d_fat), kFatWords);
    QX_CUDA(cudaGetLastError());
  }
  QX_TRY(qx_readback(s->stream, s->h_pinned, reinterpret_cast<const int64_t*>(info), 2));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  const int64_t n_units = s->h_pinned[0], max_unit = s->h_pinned[1];
  BucketStats& st = bucket_stats();
  st.groups = ng;
  st.tiles = (int64_t)n_tiles;
  st.units = n_units;
  st.max_unit = max_unit;
  st.slots = total;
  st.ell = ell;
  st.cap = 0;
  st.ctas_per_sm = 0;
  if (n_units <= 0 || max_unit > kCapMax) return QX_OK;
  const int cap = (int)std::max<int64_t>(256, (max_unit + 255) / 256 * 256);
  const size_t fixed = (sizeof(BSmem<K>) + 15) & ~(size_t)15;
  const size_t smem = bucket_smem_bytes(fixed, ell, cap);
  const u32 u_lo = (u32)(n_units * part / parts), u_hi = (u32)(n_units * (part + 1) / parts);
  int per_sm = 0;
  auto launch = [&](auto kernel, auto* keys_out) -> int {
    // attribute + occupancy of (kernel, shared-memory size): asked once, the answers do not change
    // (two driver calls on the critical path of every step otherwise: the GPU is idle behind the
    // read-back of the bucket sizes)
    static thread_local const void* cached_kernel = nullptr;
    static thread_local size_t cached_smem = 0;
    static thread_local int cached_per_sm = 0;
    static thread_local int cached_device = -1;
    if (cached_kernel != reinterpret_cast<const void*>(kernel) || cached_smem != smem || cached_device != s->device) {
      QX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      QX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached_per_sm, kernel, kBThreads, smem));
      cached_kernel = reinterpret_cast<const void*>(kernel);
      cached_smem = smem;
      cached_device = s->device;
    }
    per_sm = std::max(cached_per_sm, 1);
    static const int cap_per_sm = getenv("QX_BUCKET_CTAS") ? atoi(getenv("QX_BUCKET_CTAS")) : 0;   // experiments
    if (cap_per_sm > 0) per_sm = std::min(per_sm, cap_per_sm);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)u_hi - u_lo, (int64_t)s->sm_count * per_sm));
    kernel<<<grid, kBThreads, smem, s->stream>>>(d_fat, d_phi, d_units, u_lo, u_hi, skey, keys_out, s->lam[out],
                                                  unit_status, ticket, ell, top_bits, cap, eps, ct, im);
    QX_CUDA(cudaGetLastError());
    return QX_OK;
  };
  {
    QxProfileScope prof(QX_K_BUCKET_EMIT, s->stream, 16.0 * (double)n_sources + (narrow_out ? 12.0 : 16.0) * (double)total);
    if (narrow_out) {
      if constexpr (sizeof(K) == 4) QX_TRY(launch(k_bucket_emit<K, u32>, reinterpret_cast<u32*>(s->keys[out])));
      else return qx_fail(QX_ERR_CONSISTENCY, "narrow output needs 32-bit working keys (internal error)");
    } else {
      QX_TRY(launch(k_bucket_emit<K, u64>, reinterpret_cast<u64*>(s->keys[out])));
    }
  }
  k_bucket_offsets<<<1, 32, 0, s->stream>>>(unit_status, seg_first, n_seg, u_lo, u_hi, (u32)n_units, s->seg[out]);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  st.cap = cap;
  st.ctas_per_sm = per_sm;
  *handled = true;
  return QX_OK;
}

}  // namespace qxb
