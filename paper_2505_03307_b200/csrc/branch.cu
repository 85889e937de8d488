// Non-Clifford gate-apply: the kernels that make terms branch.
//
//   qx_apply_split    -- v1, one rotation on one qubit: each term keeps its first
//                        branch and, where the gate mixes axes, emits a second one
//                        (reference engine.py:183-218).  Single pass: warp ballot
//                        prefix sums + one decoupled look-back per tile give every
//                        term its compacted output slot.
//   qx_apply_operator -- v2/v3, a whole U_k: substitute the per-qubit 3x3 blocks and
//                        flatten the Cartesian product (reference stabilizer.py:189-206
//                        sub, :289-322 _flatten_ragged).  The (S, n, 4) weight tensor
//                        is never materialised: a count pass gives each term its raw
//                        offset, then one thread per OUTPUT term decodes its branch
//                        id as a mixed-radix number over the term's non-identity
//                        digits (qubit 0 slowest) and multiplies the weights left to
//                        right in qubit order, like the reference does.
//
// Both leave the store unmerged (raw); qx_merge follows.  Output order inside a
// segment is "term-major, branches ascending", which keeps duplicates of one key in
// the same relative order as the reference's raw lists, so the merge sums them in
// the same order.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "expand.cuh"

using namespace qxe;

namespace {

constexpr int kThreads = QX_SCAN_THREADS;
constexpr int kItems = QX_SCAN_ITEMS;
constexpr int kTile = QX_SCAN_TILE;
constexpr int kWarps = kThreads / 32;
constexpr int kSegSmem = 1024;          // offsets cached in shared memory up to this many segments

// ---------------------------------------------------------------------------------
// v1 split
// ---------------------------------------------------------------------------------
struct SplitTable {
  double w1[4], w2[4];
  u32 a1[4], a2[4];
  u32 shift;
};

__global__ void __launch_bounds__(kThreads)
k_split(const u64* __restrict__ keys_in, const double* __restrict__ lam_in,
        const int64_t* __restrict__ seg_in, int n_seg, u64* __restrict__ keys_out,
        double* __restrict__ lam_out, int64_t* __restrict__ seg_out, u64* status, u32* ticket,
        const SplitTable tb) {
  __shared__ int s_tile;
  __shared__ u64 s_scan[kWarps + 1];
  __shared__ u64 s_base;
  const int tile = take_ticket(ticket, &s_tile);
  const int64_t total = seg_in[n_seg];
  const int64_t ntiles = total > 0 ? (total + kTile - 1) / kTile : 1;
  if (tile >= ntiles) return;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t wbase = (int64_t)tile * kTile + (int64_t)warp * (32 * kItems);
  {   // the tile a CTA kPrefetchAhead positions later will read: have it in L2 by then
    const int64_t far = ((int64_t)tile + kPrefetchAhead) * kTile;
    if (far < total) {
      const int cnt = (int)min((int64_t)kTile, total - far);
      prefetch_l2(keys_in + far, cnt);
      prefetch_l2(lam_in + far, cnt);
    }
  }

  u64 key[kItems];
  double lam[kItems];
  u32 dig[kItems];
  u32 pre[kItems];                         // second-branch count before this item, inside the warp
  u32 running = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    const bool live = i < total;
    key[k] = live ? ld_stream(keys_in + i) : 0ull;
    lam[k] = live ? ld_stream(lam_in + i) : 0.0;
    dig[k] = (u32)(key[k] >> tb.shift) & 3u;
    const bool second = live && tb.w2[dig[k]] != 0.0;
    const u32 votes = __ballot_sync(QX_FULL_MASK, second);
    pre[k] = running + __popc(votes & lanemask_lt());
    running += __popc(votes);
  }
  // exclusive prefix of the warp totals, then of the tile
  u64 tile_total;
  const u64 mine = (lane == 0) ? (u64)running : 0ull;
  u64 warp_excl = block_exclusive_sum<u64>(mine, s_scan, tile_total);
  warp_excl = __shfl_sync(QX_FULL_MASK, warp_excl, 0);
  if (warp == 0) {
    const u64 excl = lookback_exclusive(status, tile, tile_total);
    if (lane == 0) s_base = excl;
  }
  __syncthreads();
  const u64 base = s_base + warp_excl;
  // Does a segment start inside this warp's 32 * kItems terms?  One search per warp (the same
  // addresses for every lane) instead of one per term: with 29 000 tiles and 16 generators almost
  // no warp sees a boundary.
  const int g_warp = segment_of(seg_in, n_seg, min(wbase, total - 1));
  const bool no_opens = seg_in[g_warp] < wbase && seg_in[g_warp + 1] >= wbase + 32 * kItems;

#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    if (i >= total) continue;
    const int64_t pos = i + (int64_t)(base + pre[k]);
    const u32 d = dig[k];
    const u64 cleared = key[k] & ~(3ull << tb.shift);
    st_stream(keys_out + pos, cleared | ((u64)tb.a1[d] << tb.shift));
    st_stream(lam_out + pos, lam[k] * tb.w1[d]);
    if (tb.w2[d] != 0.0) {
      st_stream(keys_out + pos + 1, cleared | ((u64)tb.a2[d] << tb.shift));
      st_stream(lam_out + pos + 1, lam[k] * tb.w2[d]);
    }
    if (!no_opens) {
      const int g = segment_of(seg_in, n_seg, i);
      if (seg_in[g] == i) open_offsets(seg_in, seg_out, g, i, pos);
    }
  }
  if (tile == ntiles - 1 && threadIdx.x == 0)
    close_offsets(seg_in, seg_out, n_seg, total, total + (int64_t)(s_base + tile_total));
}

// ---------------------------------------------------------------------------------
// v2/v3 operator
// ---------------------------------------------------------------------------------
// OperatorTable, ImageTable, LowGroup and the decode helpers live in expand.cuh (shared with dense.cu)

// roff[i] = raw terms produced by input terms before i (roff[total] = raw total).
__global__ void __launch_bounds__(kThreads)
k_expand_count(const u64* __restrict__ keys_in, const int64_t* __restrict__ seg_in, int n_seg,
               u64* __restrict__ roff, u64* status, u32* ticket,
               const __grid_constant__ OperatorTable tb) {
  __shared__ int s_tile;
  __shared__ u64 s_scan[kWarps + 1];
  __shared__ u64 s_base;
  __shared__ unsigned char s_cnt[QX_MAX_QUBITS][3];
  for (int i = threadIdx.x; i < QX_MAX_QUBITS * 3; i += kThreads) s_cnt[i / 3][i % 3] = tb.cnt[i / 3][i % 3];
  const int tile = take_ticket(ticket, &s_tile);     // has the __syncthreads that publishes s_cnt
  const int64_t total = seg_in[n_seg];
  const int64_t ntiles = total > 0 ? (total + kTile - 1) / kTile : 1;
  if (tile >= ntiles) return;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t wbase = (int64_t)tile * kTile + (int64_t)warp * (32 * kItems);
  u64 pre[kItems];
  u64 running = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    const u64 c = (i < total) ? branch_count(ld_stream(keys_in + i), s_cnt) : 0ull;
    const u64 inc = warp_inclusive_sum(c);
    pre[k] = running + inc - c;
    running += __shfl_sync(QX_FULL_MASK, inc, 31);
  }
  u64 tile_total;
  const u64 mine = (lane == 0) ? running : 0ull;
  u64 warp_excl = block_exclusive_sum<u64>(mine, s_scan, tile_total);
  warp_excl = __shfl_sync(QX_FULL_MASK, warp_excl, 0);
  if (warp == 0) {
    const u64 excl = lookback_exclusive(status, tile, tile_total);
    if (lane == 0) s_base = excl;
  }
  __syncthreads();
  const u64 base = s_base + warp_excl;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    if (i < total) roff[i] = base + pre[k];
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) roff[total] = s_base + tile_total;
}

__global__ void k_gather_offsets(const int64_t* __restrict__ seg_in, int n_seg,
                                 const u64* __restrict__ roff, int64_t* __restrict__ seg_out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g <= n_seg) seg_out[g] = (int64_t)roff[seg_in[g]];
}



constexpr int kEmitPer = 8;                          // outputs per thread, striped
constexpr int kEmitTile = kThreads * kEmitPer;       // 2048 raw terms per tile

template <typename K>
struct EmitSmem {
  OperatorTable tb;
  ImageTable<K> im;
  unsigned char e_hi[kEmitTile + 1];
  u64 win[kEmitTile + 2];      // raw offsets of the sources feeding the tile (+ end sentinel)
  u32 blk[kEmitTile + 2];      // exclusive prefix of blocks per source
  double p_hi[kEmitTile + 1];
  K k_hi[kEmitTile + 1];
  u32 scan[kThreads / 32 + 1];
  int64_t lohi[2];
  u64 hfirst0;                 // first block id of the first source (it may start mid-way)
  // one-source tiles: everything the 27 (or fewer) low-group branches of the source contribute
  double low_w[27][3];         // weights of the three low digits (1.0 where absent)
  K low_word[27];              // FUSED: composed image of the low digits; else the digits themselves
  K low_imx[27];
  u32 low_e[27];
};

// K = working key type, KO = type of the keys written (u32 = narrow raw terms for the sort),
// FUSED = compose Clifford images (im) instead of placing digits.
template <typename K, typename KO, bool FUSED>
__global__ void __launch_bounds__(kThreads)
k_expand_emit(const u64* __restrict__ keys_in, const double* __restrict__ lam_in,
              const u64* __restrict__ roff, int64_t total_in, KO* __restrict__ keys_out,
              double* __restrict__ lam_out, const __grid_constant__ OperatorTable tb,
              const __grid_constant__ ImageTable<K> im) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EmitSmem<K>& sm = *reinterpret_cast<EmitSmem<K>*>(smem_raw);
  {
    const u32* src = reinterpret_cast<const u32*>(&tb);
    u32* dst = reinterpret_cast<u32*>(&sm.tb);
    for (int i = threadIdx.x; i < (int)(sizeof(OperatorTable) / 4); i += kThreads) dst[i] = src[i];
    if (FUSED) {
      const u32* isrc = reinterpret_cast<const u32*>(&im);
      u32* idst = reinterpret_cast<u32*>(&sm.im);
      for (int i = threadIdx.x; i < (int)(sizeof(ImageTable<K>) / 4); i += kThreads) idst[i] = isrc[i];
    }
  }
  const u64 raw_total = roff[total_in];
  const int64_t ntiles = (int64_t)((raw_total + kEmitTile - 1) / kEmitTile);
  // Each CTA owns a contiguous run of tiles, so the source feeding a tile is found by stepping
  // from the previous tile's instead of a binary search in global memory, and a source with a
  // large fan-out (the heavy case: 3^k branches, k up to n) keeps its tables across tiles.
  const int64_t per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t tile_begin = (int64_t)blockIdx.x * per_cta;
  const int64_t tile_end = min(ntiles, tile_begin + per_cta);
  int64_t src = -1, cached = -1;          // source of the tile's first raw term; source whose low table is in smem
  u64 off_src = 0, off_next = 0;          // roff[src], roff[src + 1]
  K key0 = 0;
  LowGroup<K> g0 = {};
  double lam0 = 0.0;
  u32 magic = 0;                          // ceil(2^16 / L): t / L == (t * magic) >> 16 for t < 2^16 / L
  for (int64_t tile = tile_begin; tile < tile_end; ++tile) {
    const u64 r0 = (u64)tile * kEmitTile;
    const u64 r1 = min(r0 + (u64)kEmitTile, raw_total);          // exclusive
    if (src < 0) {
      src = last_le(roff, total_in, r0);
      off_src = roff[src];
      off_next = roff[src + 1];
    } else {
      while (off_next <= r0) {
        ++src;
        off_src = off_next;
        off_next = roff[src + 1];
      }
    }
    if (off_next >= r1) {
      // ---- one source feeds the whole tile: no searches, two barriers, ~40 instructions per output
      if (cached != src) {
        __syncthreads();                                         // previous tile done with the low table
        key0 = (K)keys_in[src];
        lam0 = lam_in[src];
        g0 = low_group<K>(key0, sm.tb);
        magic = 65536u / g0.L + 1u;
        if (threadIdx.x < g0.L) {
          u32 b = threadIdx.x, pick[3];
          K word = 0;
          u32 ex = 0;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            pick[j] = b % g0.rad[j];
            b /= g0.rad[j];
          }
#pragma unroll
          for (int j = 2; j >= 0; --j) {
            double w = 1.0;
            if (g0.bit[j] >= 0) {
              const int p = g0.bit[j] >> 1;
              w = sm.tb.w[p][g0.dig[j]][pick[j]];
              const u32 ax = sm.tb.axis[p][g0.dig[j]][pick[j]];
              if (FUSED) compose<K>(word, ex, sm.im.img[p][ax - 1], sm.im.imx[p][ax - 1], sm.im.e[p][ax - 1]);
              else word |= (K)ax << g0.bit[j];
            }
            sm.low_w[threadIdx.x][j] = w;
          }
          sm.low_word[threadIdx.x] = word;
          sm.low_imx[threadIdx.x] = (word ^ (word >> 1)) & Plane<K>::lo;
          sm.low_e[threadIdx.x] = ex & 3u;
        }
        cached = src;
      }
      const u64 b0 = r0 - off_src;                               // first branch of the tile
      const u64 h0 = b0 / g0.L;                                  // its block
      const u32 bl0 = (u32)(b0 - h0 * g0.L);
      const u32 n_out = (u32)(r1 - r0);
      const u32 n_blocks = (bl0 + n_out - 1u) / g0.L + 1u;
      __syncthreads();                                           // low table visible, p_hi/k_hi free
      for (u32 e = threadIdx.x; e < n_blocks; e += kThreads) {
        K h = (K)(h0 + e);
        K choice = 0;
        for (K m = g0.hi_mask; m;) {
          const int bit = KeyOps<K>::lowest(m);
          m &= m - 1;
          u32 pick;
          divmod_small<K>(h, sm.tb.cnt[bit >> 1][(u32)((key0 >> bit) & 3u) - 1u], h, pick);
          choice |= (K)pick << bit;
        }
        double v = lam0;
        K out = 0;
        u32 ex = 0;
        for (K m = g0.hi_mask; m;) {                             // qubit 0 first (stabilizer.py:311-319)
          const int bit = KeyOps<K>::highest(m);
          m ^= (K)1 << bit;
          const u32 d = (u32)((key0 >> bit) & 3u) - 1u, pick = (u32)(choice >> bit) & 3u;
          v *= sm.tb.w[bit >> 1][d][pick];
          const u32 ax = sm.tb.axis[bit >> 1][d][pick];
          if (FUSED) compose<K>(out, ex, sm.im.img[bit >> 1][ax - 1], sm.im.imx[bit >> 1][ax - 1], sm.im.e[bit >> 1][ax - 1]);
          else out |= (K)ax << bit;
        }
        sm.p_hi[e] = v;
        sm.k_hi[e] = out;
        if (FUSED) sm.e_hi[e] = (unsigned char)(ex & 3u);
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kEmitPer; ++k) {
        const u32 idx = (u32)k * kThreads + threadIdx.x;
        if (idx < n_out) {
          const u32 t = bl0 + idx;
          const u32 e = (t * magic) >> 16;                       // t / L
          const u32 bl = t - e * g0.L;
          double v = sm.p_hi[e];
          v *= sm.low_w[bl][2];                                  // ((p_hi * w2) * w1) * w0, absent = 1.0
          v *= sm.low_w[bl][1];
          v *= sm.low_w[bl][0];
          K out = sm.k_hi[e];
          if (FUSED) {
            u32 ex = (u32)sm.e_hi[e];
            compose<K>(out, ex, sm.low_word[bl], sm.low_imx[bl], sm.low_e[bl]);
            if (composed_sign<K>(out, ex)) v = -v;               // sign flips are exact
          } else {
            out |= sm.low_word[bl];
          }
          st_stream(keys_out + r0 + idx, (KO)out);
          st_stream(lam_out + r0 + idx, v);
        }
      }
      continue;
    }
    __syncthreads();                                             // previous tile fully consumed
    if (threadIdx.x == 0) sm.lohi[0] = last_le(roff, total_in, r0);
    if (threadIdx.x == 32) sm.lohi[1] = last_le(roff, total_in, r1 - 1);
    __syncthreads();
    const int64_t lo = sm.lohi[0], hi = sm.lohi[1];
    const int span = (int)(hi - lo) + 1;                          // sources feeding this tile
    for (int i = threadIdx.x; i <= span; i += kThreads) sm.win[i] = roff[lo + i];
    __syncthreads();

    // ---- 1. blocks per source, exclusive prefix (chunks of kThreads sources)
    u32 carried = 0;
    for (int base = 0; base < span; base += kThreads) {
      const int rel = base + threadIdx.x;
      u32 nb = 0;
      if (rel < span) {
        const LowGroup<K> g = low_group<K>((K)keys_in[lo + rel], sm.tb);
        const u64 bb = (rel == 0 ? r0 : sm.win[rel]) - sm.win[rel];
        const u64 be = min(sm.win[rel + 1], r1) - sm.win[rel];     // exclusive, > bb
        const u64 hf = bb / g.L;
        nb = (u32)((be - 1) / g.L - hf) + 1u;
        if (rel == 0) sm.hfirst0 = hf;
      }
      u32 total;
      const u32 excl = block_exclusive_sum<u32>(nb, sm.scan, total);
      if (rel < span) sm.blk[rel] = carried + excl;
      carried += total;
    }
    if (threadIdx.x == 0) sm.blk[span] = carried;
    __syncthreads();

    // ---- 2. fold the high digits of every block once
    const int n_blocks = (int)sm.blk[span];
    for (int e = threadIdx.x; e < n_blocks; e += kThreads) {
      int a = 0, z = span;                                        // last rel with blk[rel] <= e
      while (z - a > 1) {
        const int mid = (a + z) >> 1;
        if (sm.blk[mid] <= (u32)e) a = mid; else z = mid;
      }
      const K key = (K)keys_in[lo + a];
      const LowGroup<K> g = low_group<K>(key, sm.tb);
      K h = (K)(a == 0 ? sm.hfirst0 : 0ull) + (K)((u32)e - sm.blk[a]);
      // decode h over the high digits (least significant first), remember the picks
      K choice = 0;
      for (K m = g.hi_mask; m;) {
        const int bit = KeyOps<K>::lowest(m);
        m &= m - 1;
        u32 pick;
        divmod_small<K>(h, sm.tb.cnt[bit >> 1][(u32)((key >> bit) & 3u) - 1u], h, pick);
        choice |= (K)pick << bit;
      }
      // fold: qubit 0 (most significant digit) first, like stabilizer.py:311-319
      double v = lam_in[lo + a];
      K out = 0;
      u32 ex = 0;
      for (K m = g.hi_mask; m;) {
        const int bit = KeyOps<K>::highest(m);
        m ^= (K)1 << bit;
        const u32 d = (u32)((key >> bit) & 3u) - 1u, pick = (u32)(choice >> bit) & 3u;
        v *= sm.tb.w[bit >> 1][d][pick];
        const u32 ax = sm.tb.axis[bit >> 1][d][pick];
        if (FUSED) compose<K>(out, ex, sm.im.img[bit >> 1][ax - 1], sm.im.imx[bit >> 1][ax - 1], sm.im.e[bit >> 1][ax - 1]);
        else out |= (K)ax << bit;
      }
      sm.p_hi[e] = v;
      sm.k_hi[e] = out;
      if (FUSED) sm.e_hi[e] = (unsigned char)(ex & 3u);
    }
    __syncthreads();

    // ---- 3. one raw term per thread per round, consecutive lanes = consecutive terms
    const bool one_source = span == 1;                 // hoist its digits
    const K keyf = (K)keys_in[lo];
    const LowGroup<K> gf = low_group<K>(keyf, sm.tb);
#pragma unroll 2
    for (int k = 0; k < kEmitPer; ++k) {
      const u64 r = r0 + (u64)k * kThreads + threadIdx.x;
      if (r >= r1) break;
      const int rel = one_source ? 0 : (int)last_le(sm.win, span, r);
      const K key = one_source ? keyf : (K)keys_in[lo + rel];
      const LowGroup<K> g = one_source ? gf : low_group<K>(key, sm.tb);
      K q = (K)(r - sm.win[rel]);
      u32 pick[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) divmod_small<K>(q, g.rad[j], q, pick[j]);
      const u32 e = sm.blk[rel] + (u32)(q - (K)(rel == 0 ? sm.hfirst0 : 0ull));
      double v = sm.p_hi[e];
      K out = sm.k_hi[e];
      u32 ex = FUSED ? (u32)sm.e_hi[e] : 0u;
#pragma unroll
      for (int j = 2; j >= 0; --j) {
        if (g.bit[j] >= 0) {
          const int p = g.bit[j] >> 1;
          v *= sm.tb.w[p][g.dig[j]][pick[j]];
          const u32 ax = sm.tb.axis[p][g.dig[j]][pick[j]];
          if (FUSED) compose<K>(out, ex, sm.im.img[p][ax - 1], sm.im.imx[p][ax - 1], sm.im.e[p][ax - 1]);
          else out |= (K)ax << g.bit[j];
        }
      }
      if (FUSED && composed_sign<K>(out, ex)) v = -v;     // sign flips are exact
      st_stream(keys_out + r, (KO)out);
      st_stream(lam_out + r, v);
    }
  }
}

int fill_table(const qx_store* s, const int32_t* counts, const int32_t* axes, const double* weights,
               OperatorTable* tb) {
  for (int p = 0; p < QX_MAX_QUBITS; ++p)
    for (int a = 0; a < 3; ++a) {
      tb->cnt[p][a] = 1;
      for (int b = 0; b < 3; ++b) {
        tb->axis[p][a][b] = (unsigned char)(a + 1);
        tb->w[p][a][b] = (b == 0) ? 1.0 : 0.0;
      }
    }
  for (int j = 0; j < s->n_qubits; ++j) {
    const int p = s->n_qubits - 1 - j;
    for (int a = 0; a < 3; ++a) {
      const int c = counts[j * 3 + a];
      QX_REQUIRE(c >= 1 && c <= 3, "qubit %d axis %d: %d nonzero weights (need 1..3)", j, a + 1, c);
      tb->cnt[p][a] = (unsigned char)c;
      if (!axes || !weights) continue;
      int prev = 0;
      for (int b = 0; b < c; ++b) {
        const int ax = axes[(j * 3 + a) * 3 + b];
        QX_REQUIRE(ax > prev && ax <= 3, "qubit %d axis %d: output axes must ascend within 1..3", j, a + 1);
        prev = ax;
        tb->axis[p][a][b] = (unsigned char)ax;
        tb->w[p][a][b] = weights[(j * 3 + a) * 3 + b];
      }
    }
  }
  return QX_OK;
}

int prepare_lookback(qx_store* s, int64_t tiles, u64** status, u32** ticket) {
  // layout in scratch: [ticket (8 bytes)] [status u64 * tiles]
  const int64_t bytes = 8 + 8 * (tiles + 1);
  QX_TRY(qx_store_scratch(s, bytes));
  QX_CUDA(cudaMemsetAsync(s->scratch, 0, (size_t)bytes, s->stream));
  *ticket = reinterpret_cast<u32*>(s->scratch);
  *status = reinterpret_cast<u64*>(reinterpret_cast<char*>(s->scratch) + 8);
  return QX_OK;
}

}  // namespace

extern "C" int qx_apply_split(qx_store* s, int32_t qubit, const int32_t a1[4], const double w1[4],
                              const int32_t a2[4], const double w2[4]) {
  QX_REQUIRE(s && a1 && w1 && a2 && w2, "NULL argument");
  QX_NARROW_ONLY(s, "qx_apply_split");
  QX_REQUIRE(qubit >= 0 && qubit < s->n_qubits, "qubit %d out of range for n=%d", qubit, s->n_qubits);
  SplitTable tb;
  tb.shift = 2u * (u32)(s->n_qubits - 1 - qubit);
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
  const int64_t tiles = std::max<int64_t>(1, (s->ub_total + kTile - 1) / kTile);
  u64* status;
  u32* ticket;
  QX_TRY(prepare_lookback(s, tiles, &status, &ticket));
  const int in = s->cur, out = s->cur ^ 1;
  {
    QxProfileScope prof(QX_K_SPLIT, s->stream, 16.0 * 3.0 * (double)s->ub_total);
    k_split<<<(unsigned)tiles, kThreads, 0, s->stream>>>(s->keys[in], s->lam[in], s->seg[in], s->n_seg,
                                                         s->keys[out], s->lam[out], s->seg[out], status,
                                                         ticket, tb);
    QX_CUDA(cudaGetLastError());
  }
  qx_store_flip(s);
  s->exact = false;
  s->ub_total = 2 * ub_in;
  s->ub_seg = 2 * s->ub_seg;
  return QX_OK;
}

static int count_pass(qx_store* s, const OperatorTable& tb, u64** roff_out) {
  // needs exact input size: the count array is indexed by input term
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  const int64_t total = s->h_seg[s->n_seg];
  const int64_t tiles = std::max<int64_t>(1, (total + kTile - 1) / kTile);
  const int64_t lb_bytes = 8 + 8 * (tiles + 1);
  const int64_t roff_at = (lb_bytes + 255) / 256 * 256;
  QX_TRY(qx_store_scratch(s, roff_at + 8 * (total + 1)));
  QX_CUDA(cudaMemsetAsync(s->scratch, 0, (size_t)lb_bytes, s->stream));
  u32* ticket = reinterpret_cast<u32*>(s->scratch);
  u64* status = reinterpret_cast<u64*>(reinterpret_cast<char*>(s->scratch) + 8);
  u64* roff = reinterpret_cast<u64*>(reinterpret_cast<char*>(s->scratch) + roff_at);
  {
    QxProfileScope prof(QX_K_EXPAND_COUNT, s->stream, 16.0 * (double)total);
    k_expand_count<<<(unsigned)tiles, kThreads, 0, s->stream>>>(s->keys[s->cur], s->seg[s->cur],
                                                                s->n_seg, roff, status, ticket, tb);
    QX_CUDA(cudaGetLastError());
  }
  *roff_out = roff;
  return QX_OK;
}

// ---- source order of the reference's ragged flatten ---------------------------------------------
// One CTA per segment of at most kOrdCap terms: pattern word (branch count minus one of every
// digit, two bits each, qubit 0 most significant: numeric order = lexicographic order of the
// count vectors np.unique(axis=0) produces, stabilizer.py:294), bitonic sort on (pattern, tie) in
// shared memory, terms written back in place.  Segments already in that order are not touched.
constexpr int kOrdCap = 2048;
constexpr int kOrdThreads = 256;
struct OrdSmem {
  u64 pat[kOrdCap];
  u64 tie[kOrdCap];
  u64 key[kOrdCap];
  double lam[kOrdCap];
};

__global__ void __launch_bounds__(kOrdThreads)
k_order_by_pattern(u64* __restrict__ keys, double* __restrict__ lam, const int64_t* __restrict__ seg, int by_key,
                   const __grid_constant__ OperatorTable tb) {
  extern __shared__ __align__(16) unsigned char ord_raw[];
  OrdSmem& sm = *reinterpret_cast<OrdSmem*>(ord_raw);
  __shared__ unsigned char s_cnt[QX_MAX_QUBITS][3];
  const int64_t lo = seg[blockIdx.x], len64 = seg[blockIdx.x + 1] - lo;
  if (len64 < 3 || len64 > kOrdCap) return;       // two contributions add up the same in either order
  for (int i = threadIdx.x; i < QX_MAX_QUBITS * 3; i += kOrdThreads) s_cnt[i / 3][i % 3] = tb.cnt[i / 3][i % 3];
  __syncthreads();
  const int len = (int)len64;
  int m = 32;
  while (m < len) m <<= 1;
  for (int e = threadIdx.x; e < m; e += kOrdThreads) {
    u64 key = ~0ull, pat = ~0ull;                // padding sorts behind every term
    double l = 0.0;
    if (e < len) {
      key = keys[lo + e];
      l = lam[lo + e];
      pat = 0;
      for (u64 sup = support_mask(key); sup;) {
        const int b = __ffsll((long long)sup) - 1;
        sup &= sup - 1;
        pat |= (u64)(s_cnt[b >> 1][((key >> b) & 3ull) - 1] - 1) << b;
      }
    }
    sm.pat[e] = pat;
    sm.key[e] = key;
    sm.lam[e] = l;
    sm.tie[e] = by_key ? key : (u64)e;
  }
  __syncthreads();
  int bad = 0;
  for (int e = threadIdx.x + 1; e < len; e += kOrdThreads)
    bad |= sm.pat[e - 1] > sm.pat[e] || (sm.pat[e - 1] == sm.pat[e] && sm.tie[e - 1] > sm.tie[e]);
  if (!__syncthreads_or(bad)) return;
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (m >> 1); t += kOrdThreads) {
        const int a = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int b = a | j;
        const u64 pa = sm.pat[a], pb = sm.pat[b], ta = sm.tie[a], tb2 = sm.tie[b];
        const bool greater = pa > pb || (pa == pb && ta > tb2);
        if (greater == ((a & k) == 0)) {
          sm.pat[a] = pb; sm.pat[b] = pa;
          sm.tie[a] = tb2; sm.tie[b] = ta;
          const u64 ka = sm.key[a]; sm.key[a] = sm.key[b]; sm.key[b] = ka;
          const double la = sm.lam[a]; sm.lam[a] = sm.lam[b]; sm.lam[b] = la;
        }
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < len; e += kOrdThreads) {
    keys[lo + e] = sm.key[e];
    lam[lo + e] = sm.lam[e];
  }
}

extern "C" int qx_store_order_for_operator(qx_store* s, const int32_t* counts, int32_t by_key) {
  QX_REQUIRE(s && counts, "NULL argument");
  QX_NARROW_ONLY(s, "qx_store_order_for_operator");
  OperatorTable tb;
  QX_TRY(fill_table(s, counts, nullptr, nullptr, &tb));
  if (s->ub_seg < 3 || s->n_seg == 0) return QX_OK;
  QX_CUDA(cudaSetDevice(s->device));
  static bool attr_set = false;
  if (!attr_set) {
    QX_CUDA(cudaFuncSetAttribute(k_order_by_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(OrdSmem)));
    attr_set = true;
  }
  k_order_by_pattern<<<s->n_seg, kOrdThreads, sizeof(OrdSmem), s->stream>>>(s->keys[s->cur], s->lam[s->cur],
                                                                         s->seg[s->cur], by_key ? 1 : 0, tb);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  return QX_OK;
}

extern "C" int qx_count_operator(qx_store* s, const int32_t* counts, int64_t* raw_per_segment) {
  QX_REQUIRE(s && counts && raw_per_segment, "NULL argument");
  QX_NARROW_ONLY(s, "qx_count_operator");
  OperatorTable tb;
  QX_TRY(fill_table(s, counts, nullptr, nullptr, &tb));
  QX_CUDA(cudaSetDevice(s->device));
  u64* roff;
  QX_TRY(count_pass(s, tb, &roff));
  // borrow the dead offsets array for the gathered raw offsets
  int64_t* tmp = s->seg[s->cur ^ 1];
  k_gather_offsets<<<(s->n_seg + 256) / 256, 256, 0, s->stream>>>(s->seg[s->cur], s->n_seg, roff, tmp);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  QX_TRY(qx_readback(s->stream, s->h_pinned, tmp, (int64_t)s->n_seg + 1));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  for (int g = 0; g < s->n_seg; ++g) raw_per_segment[g] = s->h_pinned[g + 1] - s->h_pinned[g];
  return QX_OK;
}

// ---- host side of the fused path -----------------------------------------------------------
namespace {

// one op of a sign-permutation program on one word (same encoding as clifford.cu apply_op)
void host_apply_op(u32 op, u64& key, u32& neg, u32 cx_c, u32 cx_t, u32 cx_s) {
  const u32 s0 = (op >> 2) & 63u;
  const u32 d0 = (u32)(key >> s0) & 3u;
  if ((op & 3u) == 0u) {
    const u32 nd = (op >> (16u + 2u * d0)) & 3u;
    neg ^= (op >> (24u + d0)) & 1u;
    key ^= (u64)(d0 ^ nd) << s0;
  } else {
    const u32 s1 = (op >> 8) & 63u;
    const u32 d1 = (u32)(key >> s1) & 3u;
    const u32 e = d0 * 4u + d1;
    const u32 n0 = (cx_c >> (2u * e)) & 3u, n1 = (cx_t >> (2u * e)) & 3u;
    neg ^= (cx_s >> e) & 1u;
    key ^= ((u64)(d0 ^ n0) << s0) | ((u64)(d1 ^ n1) << s1);
  }
}

// Images of the 3n single-digit words under a sign-permutation program.  The same programs recur
// (every run of a cached circuit plan, every step of a benchmark loop) and pushing 3n words
// through a few hundred ops costs more host time than the kernel that uses the table takes on
// the small configs, so the last tables are kept, found by an FNV-1a hash of the program and
// verified against a copy of it.
struct ImageCacheEntry {
  u64 hash = 0;
  int n_qubits = 0;
  u32 cx_c = 0, cx_t = 0, cx_s = 0;
  std::vector<uint32_t> program;
  u64 img[QX_MAX_QUBITS][3];
  unsigned char e[QX_MAX_QUBITS][3];
  bool used = false;
};
constexpr int kImageCache = 64;

template <typename K>
void fill_images(int n_qubits, const uint32_t* program, int n_ops, u32 cx_c, u32 cx_t, u32 cx_s,
                 ImageTable<K>* im) {
  memset(im, 0, sizeof(*im));
  const u64 lo = 0x5555555555555555ull;
  static thread_local ImageCacheEntry cache[kImageCache];
  u64 h = 1469598103934665603ull ^ (u64)n_qubits;
  for (int i = 0; i < n_ops; ++i) h = (h ^ program[i]) * 1099511628211ull;
  ImageCacheEntry& ce = cache[h % kImageCache];
  const bool hit = ce.used && ce.hash == h && ce.n_qubits == n_qubits && ce.cx_c == cx_c && ce.cx_t == cx_t &&
                   ce.cx_s == cx_s && (int)ce.program.size() == n_ops &&
                   (n_ops == 0 || memcmp(ce.program.data(), program, sizeof(uint32_t) * (size_t)n_ops) == 0);
  if (!hit) {
    for (int p = 0; p < n_qubits; ++p)
      for (u32 a = 1; a <= 3; ++a) {
        u64 w = (u64)a << (2 * p);
        u32 neg = 0;
        for (int i = 0; i < n_ops; ++i) host_apply_op(program[i], w, neg, cx_c, cx_t, cx_s);
        const u32 ny = (u32)__builtin_popcountll((w >> 1) & ~w & lo);
        ce.img[p][a - 1] = w;
        ce.e[p][a - 1] = (unsigned char)((ny + 2u * neg) & 3u);
      }
    ce.hash = h;
    ce.n_qubits = n_qubits;
    ce.cx_c = cx_c;
    ce.cx_t = cx_t;
    ce.cx_s = cx_s;
    ce.program.assign(program, program + n_ops);
    ce.used = true;
  }
  for (int p = 0; p < n_qubits; ++p)
    for (int a = 0; a < 3; ++a) {
      const u64 w = ce.img[p][a];
      im->img[p][a] = (K)w;
      im->imx[p][a] = (K)((w ^ (w >> 1)) & lo);
      im->e[p][a] = ce.e[p][a];
    }
}

}  // namespace

namespace qxe {
void fill_images_u32(int n_qubits, const uint32_t* program, int n_ops, u32 cx_c, u32 cx_t, u32 cx_s,
                     ImageTable<u32>* im) {
  fill_images<u32>(n_qubits, program, n_ops, cx_c, cx_t, cx_s, im);
}
void fill_images_u64(int n_qubits, const uint32_t* program, int n_ops, u32 cx_c, u32 cx_t, u32 cx_s,
                     ImageTable<u64>* im) {
  fill_images<u64>(n_qubits, program, n_ops, cx_c, cx_t, cx_s, im);
}
}  // namespace qxe

// dense.cu: the grouped dense operator step
int qx_dense_operator_step(qx_store* s, const OperatorTable& nz, const uint32_t* program, int n_ops,
                           u32 cx_c, u32 cx_t, u32 cx_s, double eps, int64_t* slots_total,
                           int64_t probe_fanout, bool* done, int part = 0, int parts = 1);

namespace {

template <typename K, typename KO, bool FUSED>
int launch_emit(qx_store* s, const OperatorTable& tb, const ImageTable<K>& im, const u64* roff,
                int64_t total_in, int64_t raw, int in, int out) {
  const int64_t tiles = (raw + kEmitTile - 1) / kEmitTile;
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)s->sm_count * 8);
  static bool attr_set = false;
  if (!attr_set) {
    QX_CUDA(cudaFuncSetAttribute(k_expand_emit<K, KO, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(EmitSmem<K>)));
    attr_set = true;
  }
  k_expand_emit<K, KO, FUSED><<<grid, kThreads, sizeof(EmitSmem<K>), s->stream>>>(
      s->keys[in], s->lam[in], roff, total_in, reinterpret_cast<KO*>(s->keys[out]), s->lam[out], tb, im);
  QX_CUDA(cudaGetLastError());
  return QX_OK;
}

// U_k (+ an optional Clifford run folded in).  narrow_ok: the caller merges right away with the
// large path, so for 2n <= 32 the raw keys may be written as 32-bit words; *narrow says whether
// they were.
// dense_eps > 0: the caller merges right away with this drop threshold, so an operator with a
// large fan-out may take the grouped dense path (dense.cu), which leaves the store canonical;
// *went_dense says whether it did.
int expand(qx_store* s, const OperatorTable& tb, const uint32_t* program, int n_ops, u32 cx_c,
           u32 cx_t, u32 cx_s, bool narrow_ok, int64_t term_limit, int64_t* raw_total, bool* narrow,
           double dense_eps = -1.0, bool* went_dense = nullptr, int part = 0, int parts = 1) {
  QX_CUDA(cudaSetDevice(s->device));
  u64* roff;
  QX_TRY(count_pass(s, tb, &roff));
  const int64_t total_in = s->h_seg[s->n_seg];
  k_gather_offsets<<<(s->n_seg + 256) / 256, 256, 0, s->stream>>>(s->seg[s->cur], s->n_seg, roff,
                                                                  s->seg[s->cur ^ 1]);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  QX_TRY(qx_readback(s->stream, s->h_pinned, s->seg[s->cur ^ 1], (int64_t)s->n_seg + 1));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  const int64_t raw = s->h_pinned[s->n_seg];
  if (raw_total) *raw_total = raw;
  if (term_limit > 0 && raw > term_limit)
    return qx_fail(QX_ERR_RESOURCE, "operator would expand %lld terms into %lld raw terms (limit %lld)",
                   (long long)total_in, (long long)raw, (long long)term_limit);
  int64_t ub_seg = 0;
  for (int g = 0; g < s->n_seg; ++g) ub_seg = std::max(ub_seg, s->h_pinned[g + 1] - s->h_pinned[g]);
  if (went_dense) *went_dense = false;
  static const bool no_dense = getenv("QX_NO_DENSE") != nullptr;
  static const int64_t dense_fanout = getenv("QX_DENSE_FANOUT") ? atoll(getenv("QX_DENSE_FANOUT")) : 16;
  if (dense_eps > 0.0 && !no_dense && ub_seg > QX_SMALL_MAX && raw >= dense_fanout * total_in) {
    bool done = false;
    QX_TRY(qx_dense_operator_step(s, tb, program, n_ops, cx_c, cx_t, cx_s, dense_eps, nullptr, 0, &done, part, parts));
    if (went_dense) *went_dense = true;
    return QX_OK;
  }
  if (raw > s->cap) {
    // growing moves the live terms; the count array (scratch) and the gathered offsets stay valid
    std::vector<int64_t> raw_off(s->h_pinned, s->h_pinned + s->n_seg + 1);
    QX_TRY(qx_store_reserve(s, raw, true));
    QX_CUDA(cudaMemcpyAsync(s->seg[s->cur ^ 1], raw_off.data(), sizeof(int64_t) * (size_t)(s->n_seg + 1),
                            cudaMemcpyHostToDevice, s->stream));
    QX_CUDA(cudaStreamSynchronize(s->stream));
  }
  const bool small_keys = s->n_qubits <= 16;
  const bool go_narrow = narrow_ok && small_keys && ub_seg > QX_SMALL_MAX;
  if (narrow) *narrow = go_narrow;
  const int in = s->cur, out = s->cur ^ 1;
  if (raw > 0) {
    const double key_bytes = go_narrow ? 4.0 : 8.0;
    QxProfileScope prof(QX_K_EXPAND_EMIT, s->stream, 16.0 * (double)total_in + (8.0 + key_bytes) * (double)raw);
    if (small_keys) {
      ImageTable<u32> im;
      if (n_ops > 0) fill_images<u32>(s->n_qubits, program, n_ops, cx_c, cx_t, cx_s, &im);
      if (n_ops > 0 && go_narrow) QX_TRY((launch_emit<u32, u32, true>(s, tb, im, roff, total_in, raw, in, out)));
      else if (n_ops > 0) QX_TRY((launch_emit<u32, u64, true>(s, tb, im, roff, total_in, raw, in, out)));
      else if (go_narrow) QX_TRY((launch_emit<u32, u32, false>(s, tb, im, roff, total_in, raw, in, out)));
      else QX_TRY((launch_emit<u32, u64, false>(s, tb, im, roff, total_in, raw, in, out)));
    } else {
      ImageTable<u64> im;
      if (n_ops > 0) {
        fill_images<u64>(s->n_qubits, program, n_ops, cx_c, cx_t, cx_s, &im);
        QX_TRY((launch_emit<u64, u64, true>(s, tb, im, roff, total_in, raw, in, out)));
      } else {
        QX_TRY((launch_emit<u64, u64, false>(s, tb, im, roff, total_in, raw, in, out)));
      }
    }
  }
  qx_store_flip(s);
  for (int g = 0; g <= s->n_seg; ++g) s->h_seg[g] = s->h_pinned[g];
  s->exact = true;
  s->ub_total = raw;
  s->ub_seg = ub_seg;
  return QX_OK;
}


// ---- small stores: expansion + Clifford run + merge in ONE launch --------------------------------
// Configs 1, 2, 3, 5 hold a few thousand terms: their cost is launches and host round trips, not
// bandwidth.  When every generator's raw expansion fits shared memory (<= QX_SMALL_MAX terms, known
// on the host from the rank bound and the operator's largest fan-out), one CTA per generator does
// the whole operator step: branch counts + scan, raw terms into shared memory (products qubit 0
// first, images of the run composed in), bitonic sort on (key, raw position), in-order run sums,
// drop rule, compaction by look-back across the generators -- the reference's
// flatten + apply_cx + canonicalize (stabilizer.py:289-363) with one launch and one read-back.
constexpr int kSoThreads = 256;
constexpr int kSoWarps = kSoThreads / 32;
constexpr int kSoSrcMax = 4096;

__global__ void __launch_bounds__(kSoThreads)
k_small_operator(const u64* __restrict__ keys_in, const double* __restrict__ lam_in,
                 const int64_t* __restrict__ seg_in, int n_seg, u64* __restrict__ keys_out,
                 double* __restrict__ lam_out, int64_t* __restrict__ seg_out, u64* status, int* error,
                 int src_cap, int raw_cap, double eps, const __grid_constant__ OperatorTable tb,
                 const __grid_constant__ ImageTable<u64> im) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* rkey = reinterpret_cast<u64*>(smem_raw);                            // raw_cap
  double* rlam = reinterpret_cast<double*>(rkey + raw_cap);                // raw_cap
  u32* soff = reinterpret_cast<u32*>(rlam + raw_cap);                      // src_cap + 1
  unsigned short* ridx = reinterpret_cast<unsigned short*>(soff + src_cap + 1);   // raw_cap
  __shared__ OperatorTable s_tb;
  __shared__ ImageTable<u64> s_im;
  __shared__ u64 s_scan[kSoWarps + 1];
  __shared__ u64 s_base;
  const int g = qx_tile_id(reinterpret_cast<u32*>(error) + 1);   // in-order dispatch, see qx_device.cuh (error[1]: a zeroed spare word)
  const int tid = threadIdx.x;
  {
    const u32* src = reinterpret_cast<const u32*>(&tb);
    u32* dst = reinterpret_cast<u32*>(&s_tb);
    for (int i = tid; i < (int)(sizeof(OperatorTable) / 4); i += kSoThreads) dst[i] = src[i];
    const u32* isrc = reinterpret_cast<const u32*>(&im);
    u32* idst = reinterpret_cast<u32*>(&s_im);
    for (int i = tid; i < (int)(sizeof(ImageTable<u64>) / 4); i += kSoThreads) idst[i] = isrc[i];
  }
  const int64_t start = seg_in[g];
  int len = (int)min((int64_t)0x7fffffff, seg_in[g + 1] - start);
  bool bad = len > src_cap;
  if (bad) len = 0;
  __syncthreads();
  // branch counts -> exclusive raw offsets (consecutive sources per thread)
  const int per = (len + kSoThreads - 1) / kSoThreads;
  const int e0 = tid * per, e1 = min(len, e0 + per);
  u64 mine = 0;
  for (int e = e0; e < e1; ++e) mine += branch_count(keys_in[start + e], s_tb.cnt);
  u64 total;
  u64 run = block_exclusive_sum<u64>(mine, s_scan, total);
  if (total > (u64)raw_cap) {              // host bound was wrong: flag it, keep the chain alive
    bad = true;
    total = 0;
    len = 0;
  }
  for (int e = e0; e < e1 && !bad; ++e) {
    soff[e] = (u32)run;
    run += branch_count(keys_in[start + e], s_tb.cnt);
  }
  if (tid == 0) {
    soff[len] = (u32)total;
    if (bad) atomicExch(error, 1);
    else atomicAdd(reinterpret_cast<unsigned long long*>(error) + 1, (unsigned long long)total);   // raw terms of the step
  }
  __syncthreads();
  const int raw = (int)total;
  int m = 32;
  while (m < raw) m <<= 1;
  // raw terms: source by bisection of the offsets, picks by mixed-radix decode (lowest digit
  // fastest), product and image composition qubit 0 first (stabilizer.py:311-319)
  for (int r = tid; r < m; r += kSoThreads) {
    u64 out = ~0ull;
    double v = 0.0;
    if (r < raw) {
      int lo = 0, hi = len;                // soff[lo] <= r < soff[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (soff[mid] <= (u32)r) lo = mid; else hi = mid;
      }
      const u64 key = keys_in[start + lo];
      u32 b = (u32)r - soff[lo];
      u64 picks = 0;
      for (u64 mask = support_mask(key); mask;) {
        const int bit = __ffsll((long long)mask) - 1;
        mask &= mask - 1;
        const u32 c = s_tb.cnt[bit >> 1][(u32)((key >> bit) & 3ull) - 1u];
        const u32 q = b / c;
        picks |= (u64)(b - q * c) << bit;
        b = q;
      }
      v = lam_in[start + lo];
      out = 0;
      u32 ex = 0;
      for (u64 mask = support_mask(key); mask;) {
        const int bit = 63 - __clzll((long long)mask);
        mask ^= 1ull << bit;
        const int p = bit >> 1;
        const u32 d = (u32)((key >> bit) & 3ull) - 1u, pick = (u32)(picks >> bit) & 3u;
        v = __dmul_rn(v, s_tb.w[p][d][pick]);
        const u32 ax = s_tb.axis[p][d][pick];
        compose<u64>(out, ex, s_im.img[p][ax - 1], s_im.imx[p][ax - 1], s_im.e[p][ax - 1]);
      }
      if (composed_sign<u64>(out, ex)) v = -v;     // sign flips are exact
    }
    rkey[r] = out;
    rlam[r] = v;
    ridx[r] = (unsigned short)r;
  }
  __syncthreads();
  // bitonic network on (key, raw position): equal keys stay in raw order, padding ends up last
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < (m >> 1); t += kSoThreads) {
        const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int hi = lo | j;
        const u64 ka = rkey[lo], kb = rkey[hi];
        const unsigned short ia = ridx[lo], ib = ridx[hi];
        const bool greater = ka > kb || (ka == kb && ia > ib);
        if (greater == ((lo & k) == 0)) {
          rkey[lo] = kb; rkey[hi] = ka;
          ridx[lo] = ib; ridx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  // run sums (sequential, raw order), drop rule, ordered compaction row by row
  const int rows = (raw + kSoThreads - 1) / kSoThreads;
  u64 my_count = 0;
  for (int r = 0; r < rows; ++r) {
    const int e = r * kSoThreads + tid;
    if (e < raw) {
      const u64 key = rkey[e];
      if (e == 0 || rkey[e - 1] != key) {
        double sum = rlam[ridx[e]];
        for (int j = e + 1; j < raw && rkey[j] == key; ++j) sum += rlam[ridx[j]];
        if (fabs(sum) >= eps) ++my_count;
      }
    }
  }
  u64 seg_total;
  block_exclusive_sum<u64>(my_count, s_scan, seg_total);
  if ((tid >> 5) == 0) {
    const u64 excl = lookback_exclusive(status, g, seg_total);
    if (lane_id() == 0) s_base = excl;
  }
  __syncthreads();
  const int64_t base = (int64_t)s_base;
  u64 kept_before = 0;
  for (int r = 0; r < rows; ++r) {
    const int e = r * kSoThreads + tid;
    bool kept = false;
    u64 key = 0;
    double sum = 0.0;
    if (e < raw) {
      key = rkey[e];
      if (e == 0 || rkey[e - 1] != key) {
        sum = rlam[ridx[e]];
        for (int j = e + 1; j < raw && rkey[j] == key; ++j) sum += rlam[ridx[j]];
        kept = fabs(sum) >= eps;
      }
    }
    u64 row_total;
    const u64 excl = block_exclusive_sum<u64>(kept ? 1ull : 0ull, s_scan, row_total);
    if (kept) {
      const int64_t pos = base + (int64_t)(kept_before + excl);
      keys_out[pos] = key;
      lam_out[pos] = sum;
    }
    kept_before += row_total;
  }
  if (tid == 0) {
    seg_out[g] = base;
    if (g == n_seg - 1) seg_out[n_seg] = base + (int64_t)seg_total;
  }
}

// Host side: *done = false (and nothing touched) when the bounds do not fit.
int small_operator_run(qx_store* s, const OperatorTable& tb, const uint32_t* program, int n_ops, u32 cx_c,
                       u32 cx_t, u32 cx_s, double eps, int64_t max_fanout, bool* done, int64_t* raw_total) {
  *done = false;
  static const bool off = getenv("QX_NO_SMALL_OPERATOR") != nullptr;
  if (off || s->n_words > 1 || s->n_seg < 1) return QX_OK;
  const int64_t src_ub = s->ub_seg;
  if (src_ub < 1 || src_ub > kSoSrcMax || src_ub * max_fanout > QX_SMALL_MAX) return QX_OK;
  QX_CUDA(cudaSetDevice(s->device));
  int raw_cap = 32;
  while (raw_cap < src_ub * max_fanout) raw_cap <<= 1;
  const int src_cap = (int)src_ub;
  QX_TRY(qx_store_reserve(s, std::min<int64_t>(s->ub_total * max_fanout, (int64_t)s->n_seg * raw_cap) + 2, true));
  const int64_t bytes = 16 + 8 * ((int64_t)s->n_seg + 1);
  QX_TRY(qx_store_scratch(s, bytes));
  QX_CUDA(cudaMemsetAsync(s->scratch, 0, (size_t)bytes, s->stream));
  int* error = reinterpret_cast<int*>(s->scratch);
  u64* status = reinterpret_cast<u64*>(reinterpret_cast<char*>(s->scratch) + 16);
  ImageTable<u64> im;
  fill_images<u64>(s->n_qubits, program, n_ops, cx_c, cx_t, cx_s, &im);
  const size_t smem = (size_t)raw_cap * 18 + 4 * ((size_t)src_cap + 1) + 16;
  static size_t attr_smem = 0;
  if (smem > attr_smem) {
    QX_CUDA(cudaFuncSetAttribute(k_small_operator, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 QX_SMALL_MAX * 18 + 4 * (kSoSrcMax + 1) + 16));
    attr_smem = QX_SMALL_MAX * 18 + 4 * (kSoSrcMax + 1) + 16;
  }
  const int in = s->cur, out = s->cur ^ 1;
  {
    QxProfileScope prof(QX_K_SMALL_MERGE, s->stream, 32.0 * (double)s->ub_total * (double)max_fanout);
    k_small_operator<<<s->n_seg, kSoThreads, smem, s->stream>>>(s->keys[in], s->lam[in], s->seg[in], s->n_seg,
                                                               s->keys[out], s->lam[out], s->seg[out], status,
                                                               error, src_cap, raw_cap, eps, tb, im);
    QX_CUDA(cudaGetLastError());
  }
  // one round trip: the error word, then the new offsets
  QX_CUDA(cudaMemcpyAsync(s->h_pinned, error, 16, cudaMemcpyDeviceToHost, s->stream));
  QX_TRY(qx_readback(s->stream, s->h_seg, s->seg[out], (int64_t)s->n_seg + 1));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  if (*reinterpret_cast<int*>(s->h_pinned) != 0) {
    // a bound was wrong (cannot happen with exact ranks): the input buffer is untouched, so the
    // general path can still run; the host mirror of the offsets is restored first
    s->exact = false;
    QX_TRY(qx_store_refresh(s));
    return QX_OK;
  }
  s->cur = out;
  s->exact = true;
  s->ub_total = s->h_seg[s->n_seg];
  int64_t mx = 0;
  for (int g = 0; g < s->n_seg; ++g) mx = std::max(mx, s->h_seg[g + 1] - s->h_seg[g]);
  s->ub_seg = mx;
  if (raw_total) *raw_total = s->h_pinned[1];
  *done = true;
  return QX_OK;
}

#include "program.cuh"

}  // namespace

// ---- circuit programs (program.cuh) ----------------------------------------------------------------
struct qx_program {
  int device = 0;
  int n_qubits = 0;
  int n_steps = 0;
  int n_rows = 0;             // oprun steps = rows of the ranks table
  PgStep* d_steps = nullptr;
  int small_fits = -1;        // what the last run found: 1 = the small kernel variant is enough, 0 = it is not
};

extern "C" int qx_program_create(int device, int32_t n_qubits, int32_t n_steps, const int32_t* kinds,
                                 const int32_t* order, const int32_t* counts, const int32_t* axes,
                                 const double* weights, const uint32_t* ops, const int64_t* ops_off,
                                 qx_program** out) {
  QX_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  QX_REQUIRE(n_qubits >= 1 && n_qubits <= QX_MAX_QUBITS, "circuit programs need one-word keys (1 <= n <= %d), got %d",
             QX_MAX_QUBITS, n_qubits);
  QX_REQUIRE(n_steps >= 1 && kinds && ops_off, "bad step list");
  qx_store shape;                        // fill_table / qx_check_program only look at the qubit count
  shape.n_qubits = n_qubits;
  u32 cx_c, cx_t, cx_s;
  qx_standard_cx(&cx_c, &cx_t, &cx_s);
  std::vector<PgStep> steps((size_t)n_steps);
  int rows = 0;
  for (int i = 0; i < n_steps; ++i) {
    PgStep& st = steps[i];
    memset(&st, 0, sizeof(st));
    st.kind = kinds[i];
    QX_REQUIRE(st.kind == PG_CLIFFORD || st.kind == PG_OPRUN || st.kind == PG_SORT, "step %d: unknown kind %d", i, st.kind);
    const int64_t o0 = ops_off[i], o1 = ops_off[i + 1];
    QX_REQUIRE(o0 >= 0 && o1 >= o0 && o1 - o0 < (1ll << 30) && (o1 == o0 || ops), "step %d: bad op range", i);
    if (st.kind == PG_SORT) continue;
    const uint32_t* prog = o1 > o0 ? ops + o0 : nullptr;
    QX_TRY(qx_check_program(&shape, prog, (int32_t)(o1 - o0)));
    fill_images<u64>(n_qubits, prog, (int)(o1 - o0), cx_c, cx_t, cx_s, &st.im);
    if (st.kind == PG_OPRUN) {
      QX_REQUIRE(counts && axes && weights, "step %d: operator tables missing", i);
      QX_TRY(fill_table(&shape, counts + (size_t)i * n_qubits * 3, axes + (size_t)i * n_qubits * 9,
                        weights + (size_t)i * n_qubits * 9, &st.tb));
      st.order = order ? (order[i] != 0) : 0;
      st.rank_row = rows++;
    }
  }
  QX_CUDA(cudaSetDevice(device));
  qx_program* p = new qx_program;
  p->device = device;
  p->n_qubits = n_qubits;
  p->n_steps = n_steps;
  p->n_rows = rows;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p->d_steps), sizeof(PgStep) * (size_t)n_steps);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_steps, steps.data(), sizeof(PgStep) * (size_t)n_steps, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (p->d_steps) cudaFree(p->d_steps);
    delete p;
    return qx_fail(QX_ERR_CUDA, "uploading a circuit program failed: %s", cudaGetErrorString(e));
  }
  *out = p;
  return QX_OK;
}

extern "C" int qx_program_destroy(qx_program* p) {
  if (!p) return QX_OK;
  if (p->d_steps) {
    cudaSetDevice(p->device);
    cudaFree(p->d_steps);
  }
  delete p;
  return QX_OK;
}

extern "C" int qx_program_rows(const qx_program* p, int32_t* rows) {
  QX_REQUIRE(p && rows, "NULL argument");
  *rows = p->n_rows;
  return QX_OK;
}

// One launch for the whole program.  *fitted = 0: some generator outgrew shared memory; the store
// is as it was before the call and `ranks` is undefined.  *fitted = 1: the store holds the result
// (canonical if the program ends in an oprun or a sort step), ranks[row * n_segments + g] = terms
// of generator g after the row-th branching step (a 0 = collapsed there; later rows of it are 0).
extern "C" int qx_store_run_program(qx_store* s, const qx_program* p, const int32_t* init_qubits, double eps,
                                    int64_t* ranks, int64_t* raw_total, int32_t* fitted, int64_t* offsets,
                                    uint64_t* host_keys, double* host_lambdas, int64_t host_cap,
                                    int32_t* host_filled, double* device_ms, int32_t max_steps,
                                    int32_t* stopped_step) {
  QX_REQUIRE(s && p && fitted, "NULL argument");
  QX_NARROW_ONLY(s, "qx_store_run_program");
  QX_REQUIRE(p->n_qubits == s->n_qubits && p->device == s->device, "program was compiled for n=%d on device %d",
             p->n_qubits, p->device);
  QX_REQUIRE(eps >= 0.0, "eps must be non-negative");
  QX_REQUIRE(p->n_rows == 0 || ranks, "ranks is NULL");
  QX_REQUIRE((host_keys == nullptr) == (host_lambdas == nullptr), "host_keys and host_lambdas go together");
  *fitted = 0;
  if (host_filled) *host_filled = 0;
  if (stopped_step) *stopped_step = 0;
  QX_REQUIRE(max_steps >= 0 && max_steps <= p->n_steps, "max_steps %d out of range (program has %d steps)", max_steps,
             p->n_steps);
  const int run_steps = max_steps > 0 ? max_steps : p->n_steps;
  static const bool off = getenv("QX_NO_PROGRAM") != nullptr;
  if (off || s->n_seg < 1) return QX_OK;
  PgInit init;
  memset(&init, 0, sizeof(init));
  init.n_qubits = s->n_qubits;
  if (init_qubits) {
    QX_REQUIRE(s->n_seg <= QX_MAX_QUBITS, "init_qubits: at most %d generators", QX_MAX_QUBITS);
    init.on = 1;
    init.n_qubits = s->n_qubits;
    for (int g = 0; g < s->n_seg; ++g) {
      QX_REQUIRE(init_qubits[g] >= 0 && init_qubits[g] < s->n_qubits, "qubit %d out of range for n=%d", init_qubits[g],
                 s->n_qubits);
      init.qubit[g] = init_qubits[g];
    }
  }
  QX_CUDA(cudaSetDevice(s->device));
  if (!init.on) {
    if (!s->exact) QX_TRY(qx_store_refresh(s));
    if (s->ub_seg > kPgSrcCap) return QX_OK;
  }
  QX_TRY(qx_store_reserve(s, (int64_t)s->n_seg * kPgSrcCap + 2, !init.on));
  const int64_t status_bytes = 8 * ((int64_t)s->n_seg + 1);
  QX_TRY(qx_store_scratch(s, status_bytes));
  u64* status = reinterpret_cast<u64*>(s->scratch);
  // what the kernel reports, in page-locked host memory
  const int64_t rank_words = (int64_t)p->n_rows * s->n_seg;
  const int64_t need = 5 * (int64_t)s->n_seg + 1 + rank_words;
  int64_t* h = s->h_pinned;
  void* h_big = nullptr;
  if (need > s->h_pinned_words) {
    QX_TRY(qx_pinned_alloc(&h_big, 8 * need));
    h = reinterpret_cast<int64_t*>(h_big);
  }
  struct ReleasePinned {
    void* p;
    ~ReleasePinned() { if (p) qx_pinned_free(p); }
  } relp{h_big};
  PgHost host;
  host.flags = h;
  host.raw = h + s->n_seg;
  host.seg = h + 2 * s->n_seg;
  host.clock = h + 3 * s->n_seg + 1;
  host.ranks = h + 5 * s->n_seg + 1;
  host.keys = reinterpret_cast<u64*>(host_keys);
  host.lam = host_lambdas;
  host.cap = host_keys ? host_cap : 0;
  static bool attr_set = false;
  if (!attr_set) {
    QX_CUDA(cudaFuncSetAttribute(k_small_circuit<PgSmem>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PgSmem)));
    attr_set = true;
  }
  const int in = s->cur, out = s->cur ^ 1;
  // the small variant first unless the last run of this program outgrew it (a circuit's ranks do
  // not change from run to run); the full one if it does not fit
  qx_program* pm = const_cast<qx_program*>(p);
  int64_t flags = 0, raw = 0;
  for (int variant = (pm->small_fits == 0 || s->ub_seg > PgSmemSmall::kSrcCap) ? 1 : 0; variant < 2; ++variant) {
    memset(h, 0, 8 * (size_t)need);
    QX_CUDA(cudaMemsetAsync(s->scratch, 0, (size_t)status_bytes, s->stream));
    {
      QxProfileScope prof(QX_K_SMALL_MERGE, s->stream, 32.0 * (double)std::max<int64_t>(s->ub_total, s->n_seg));
      if (variant == 0)
        k_small_circuit<PgSmemSmall><<<s->n_seg, kPgThreads, sizeof(PgSmemSmall), s->stream>>>(
            s->keys[in], s->lam[in], s->seg[in], s->n_seg, p->d_steps, run_steps, s->keys[out], s->lam[out],
            s->seg[out], status, eps, init, host);
      else
        k_small_circuit<PgSmem><<<s->n_seg, kPgThreads, sizeof(PgSmem), s->stream>>>(
            s->keys[in], s->lam[in], s->seg[in], s->n_seg, p->d_steps, run_steps, s->keys[out], s->lam[out],
            s->seg[out], status, eps, init, host);
      QX_CUDA(cudaGetLastError());
    }
    QX_CUDA(cudaStreamSynchronize(s->stream));
    flags = 0;
    raw = 0;
    for (int g = 0; g < s->n_seg; ++g) {
      flags |= host.flags[g];
      raw += host.raw[g];
    }
    if (variant == 0) pm->small_fits = (flags & 1) ? 0 : 1;
    if (!(flags & 1)) break;
  }
  if (flags & 1) {
    if (stopped_step) {
      // the first step some generator outgrew shared memory at: the steps in front of it fit
      int64_t first = p->n_steps;
      for (int g = 0; g < s->n_seg; ++g)
        if (host.flags[g] & 1) first = std::min<int64_t>(first, host.flags[g] >> 8);
      *stopped_step = (int32_t)first;
    }
    // did not fit: the live buffer is untouched -- unless there was none (init_qubits): make it
    if (init.on) return qx_store_init_z(s, init_qubits);
    return QX_OK;
  }
  for (int g = 0; g <= s->n_seg; ++g) s->h_seg[g] = host.seg[g];
  if (offsets)
    for (int g = 0; g <= s->n_seg; ++g) offsets[g] = host.seg[g];
  for (int64_t i = 0; i < rank_words; ++i) ranks[i] = host.ranks[i];
  if (raw_total) *raw_total = raw;
  if (host_filled) *host_filled = (host_keys && !(flags & 2)) ? 1 : 0;
  if (device_ms) {
    // first CTA in to last CTA out, on the GPU's own nanosecond clock
    int64_t first = host.clock[0], last = host.clock[s->n_seg];
    for (int g = 1; g < s->n_seg; ++g) {
      first = std::min(first, host.clock[g]);
      last = std::max(last, host.clock[s->n_seg + g]);
    }
    *device_ms = (double)(last - first) * 1e-6;
  }
  s->cur = out;
  s->exact = true;
  s->narrow_keys = false;
  s->pack_bnd = nullptr;
  s->ub_total = s->h_seg[s->n_seg];
  int64_t mx = 0;
  for (int g = 0; g < s->n_seg; ++g) mx = std::max(mx, s->h_seg[g + 1] - s->h_seg[g]);
  s->ub_seg = mx;
  *fitted = 1;
  return QX_OK;
}

extern "C" int qx_apply_operator(qx_store* s, const int32_t* counts, const int32_t* axes,
                                 const double* weights, int64_t term_limit, int64_t* raw_total) {
  QX_REQUIRE(s && counts && axes && weights, "NULL argument");
  QX_NARROW_ONLY(s, "qx_apply_operator (branching U_k)");
  OperatorTable tb;
  QX_TRY(fill_table(s, counts, axes, weights, &tb));
  return expand(s, tb, nullptr, 0, 0, 0, 0, false, term_limit, raw_total, nullptr);
}

static int operator_run(qx_store* s, const int32_t* counts, const int32_t* axes, const double* weights,
                        const uint32_t* program, int32_t n_ops, uint32_t cx_c, uint32_t cx_t, uint32_t cx_s,
                        double eps, int64_t term_limit, int64_t* raw_total, int64_t* ranks, int part, int parts,
                        int* partitioned);

extern "C" int qx_apply_operator_run(qx_store* s, const int32_t* counts, const int32_t* axes,
                                     const double* weights, const uint32_t* program, int32_t n_ops,
                                     uint32_t cx_c, uint32_t cx_t, uint32_t cx_s, double eps,
                                     int64_t term_limit, int64_t* raw_total, int64_t* ranks) {
  return operator_run(s, counts, axes, weights, program, n_ops, cx_c, cx_t, cx_s, eps, term_limit, raw_total,
                      ranks, 0, 1, nullptr);
}

extern "C" int qx_apply_operator_run_part(qx_store* s, const int32_t* counts, const int32_t* axes,
                                          const double* weights, const uint32_t* program, int32_t n_ops,
                                          uint32_t cx_c, uint32_t cx_t, uint32_t cx_s, double eps,
                                          int32_t part, int32_t parts, int64_t* ranks, int32_t* partitioned) {
  QX_REQUIRE(parts >= 1 && part >= 0 && part < parts, "bad part %d of %d", part, parts);
  QX_REQUIRE(partitioned != nullptr, "partitioned is NULL");
  int flag = 0;
  QX_TRY(operator_run(s, counts, axes, weights, program, n_ops, cx_c, cx_t, cx_s, eps, 0, nullptr, ranks, part,
                      parts, &flag));
  *partitioned = flag;
  return QX_OK;
}

static int operator_run(qx_store* s, const int32_t* counts, const int32_t* axes, const double* weights,
                        const uint32_t* program, int32_t n_ops, uint32_t cx_c, uint32_t cx_t, uint32_t cx_s,
                        double eps, int64_t term_limit, int64_t* raw_total, int64_t* ranks, int part, int parts,
                        int* partitioned) {
  if (partitioned) *partitioned = 0;
  QX_REQUIRE(s && counts && axes && weights, "NULL argument");
  QX_NARROW_ONLY(s, "qx_apply_operator_run (branching U_k)");
  QX_REQUIRE(n_ops >= 0 && (n_ops == 0 || program), "bad program");
  QX_REQUIRE(eps >= 0.0, "eps must be non-negative");
  OperatorTable tb;
  QX_TRY(fill_table(s, counts, axes, weights, &tb));
  QX_TRY(qx_check_program(s, program, n_ops));
  u32 std_c, std_t, std_s;
  qx_standard_cx(&std_c, &std_t, &std_s);
  static const bool no_fuse = getenv("QX_NO_FUSE") != nullptr;
  if (no_fuse || cx_c != std_c || cx_t != std_t || cx_s != std_s) {
    // tables that are not the CX conjugation (mutation tests) are not a homomorphism: run the
    // three steps one after the other, table-driven
    QX_TRY(expand(s, tb, nullptr, 0, 0, 0, 0, false, term_limit, raw_total, nullptr));
    QX_TRY(qx_apply_clifford(s, program, n_ops, cx_c, cx_t, cx_s));
    return qx_merge(s, eps, ranks);
  }
  // Few sources: group them first instead of counting raw branches -- the same single host
  // round trip then already yields the slot counts the grouped path needs.
  static const bool no_dense = getenv("QX_NO_DENSE") != nullptr;
  static const int64_t dense_fanout = getenv("QX_DENSE_FANOUT") ? atoll(getenv("QX_DENSE_FANOUT")) : 16;
  if (eps > 0.0 && !no_dense && term_limit <= 0) {
    QX_CUDA(cudaSetDevice(s->device));
    if (!s->exact) QX_TRY(qx_store_refresh(s));
    const int64_t total_in = s->h_seg[s->n_seg];
    // what one term can branch into at most: operators that touch a few qubits never qualify
    int64_t max_fanout = 1;
    for (int p = 0; p < s->n_qubits && max_fanout < (1 << 20); ++p)
      max_fanout *= std::max({tb.cnt[p][0], tb.cnt[p][1], tb.cnt[p][2]});
    if (total_in > 0 && total_in <= (1 << 16) && max_fanout >= dense_fanout) {
      bool done = false;
      int64_t slots = 0;
      QX_TRY(qx_dense_operator_step(s, tb, program, n_ops, cx_c, cx_t, cx_s, eps, &slots, dense_fanout, &done,
                                    part, parts));
      if (done) {
        if (partitioned) *partitioned = parts > 1;
        if (raw_total) *raw_total = slots;
        if (ranks)
          for (int g = 0; g < s->n_seg; ++g) ranks[g] = s->h_seg[g + 1] - s->h_seg[g];
        return QX_OK;
      }
    }
  }
  if (term_limit <= 0 && parts == 1) {
    // small stores: the whole step in one launch
    QX_CUDA(cudaSetDevice(s->device));
    if (!s->exact) QX_TRY(qx_store_refresh(s));
    int64_t fan = 1;
    for (int p = 0; p < s->n_qubits && fan <= QX_SMALL_MAX; ++p)
      fan *= std::max({tb.cnt[p][0], tb.cnt[p][1], tb.cnt[p][2]});
    bool done = false;
    QX_TRY(small_operator_run(s, tb, program, n_ops, cx_c, cx_t, cx_s, eps, fan, &done, raw_total));
    if (done) {
      if (ranks)
        for (int g = 0; g < s->n_seg; ++g) ranks[g] = s->h_seg[g + 1] - s->h_seg[g];
      return QX_OK;
    }
  }
  static const bool no_narrow = getenv("QX_NO_NARROW") != nullptr;
  bool narrow = false, dense = false;
  QX_TRY(expand(s, tb, program, n_ops, cx_c, cx_t, cx_s, !no_narrow, term_limit, raw_total, &narrow, eps, &dense,
                part, parts));
  if (dense && partitioned) *partitioned = parts > 1;
  if (!dense) QX_TRY(qx_run_merge(s, eps, false, narrow));
  if (ranks)
    for (int g = 0; g < s->n_seg; ++g) ranks[g] = s->h_seg[g + 1] - s->h_seg[g];
  return QX_OK;
}
