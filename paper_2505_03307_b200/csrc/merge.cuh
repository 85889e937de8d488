// a6: the duplicate-term merge (reference stabilizer.py:325-337 canonicalize;
// measure.py:76-91 _merge for the complex read-out accumulator).
//
//   unique-sort by key  ->  in-order sum of each run of equal keys  ->  drop  ->  ascending
//
// Two device paths, same semantics, both deterministic (no floating-point atomics:
// the sort is stable and every run is summed sequentially in input order, which is
// the order np.add.at uses):
//
//   small  every segment <= QX_SMALL_MAX raw terms: ONE launch, one CTA per segment;
//          bitonic sort on (key, input position) in shared memory, run sums, and a
//          look-back across segments so the output is written compacted.  This is the
//          latency path (configs 1, 2, 3, 5: a few thousand terms, hundreds of merges).
//   large  segmented onesweep LSD radix sort, 8 bits per pass over the 2n significant
//          key bits only (n = 16 -> 4 passes, not 8): one histogram pass, then per digit
//          one pass that ranks a 4608-term tile in shared memory (warp match + per-warp
//          counters), resolves its global offsets by decoupled look-back, and scatters
//          through shared memory so runs of equal digit leave as coalesced stores.
//          Tiles are segment-aligned, so generators never mix and no generator-id pass
//          is needed.  A final reduce-by-key pass sums runs, applies the drop rule and
//          compacts with a second look-back.  HBM-bound: 32 B per term per sort pass.
//
// Templated on the coefficient type: double (evolution, keep |sum| >= eps) and
// double2 (read-out, complex, keep sum != 0).
#pragma once

#include <algorithm>
#include <type_traits>

#include "qx_device.cuh"

namespace qxm {

// ---------------------------------------------------------------------------------
// coefficient traits
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void acc(double& a, double b) { a += b; }
__device__ __forceinline__ void acc(double2& a, double2 b) { a.x += b.x; a.y += b.y; }
__device__ __forceinline__ bool keep(double v, double eps) { return fabs(v) >= eps; }
__device__ __forceinline__ bool keep(double2 v, double) { return v.x != 0.0 || v.y != 0.0; }

constexpr int kSortThreads = QX_SORT_THREADS;
constexpr int kSortItems = QX_SORT_ITEMS;
constexpr int kSortTile = QX_SORT_TILE;
constexpr int kSortWarps = kSortThreads / 32;
constexpr u32 kFlagAgg = 1u << 30;
constexpr u32 kFlagInc = 2u << 30;
constexpr u32 kFlagVal = (1u << 30) - 1;

// ---------------------------------------------------------------------------------
// plan: segment-aligned tile table
// ---------------------------------------------------------------------------------
// tile_prefix[g] = sort tiles owned by segments before g; [n_seg] = total tiles.
static __global__ void k_sort_plan(const int64_t* __restrict__ seg, int n_seg,
                                   int64_t* __restrict__ tile_prefix, u32* ticket, int tile_terms) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t run = 0;
    for (int g = 0; g < n_seg; ++g) {
      tile_prefix[g] = run;
      run += (seg[g + 1] - seg[g] + tile_terms - 1) / tile_terms;
    }
    tile_prefix[n_seg] = run;
    *ticket = 0u;
  }
}

// largest g with tile_prefix[g] <= tile < tile_prefix[g+1]
__device__ __forceinline__ int tile_segment(const int64_t* tile_prefix, int n_seg, int64_t tile) {
  int lo = 0, hi = n_seg;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tile_prefix[mid] <= tile) lo = mid; else hi = mid;
  }
  return lo;
}

// One record per sort tile, filled once per merge: the passes (and the histogram) read it with a
// single broadcast load instead of every thread bisecting the segment table in global memory
// (6 % of the pass's instructions and the head of its critical path, profiles/r01g).
struct __align__(16) TileInfo {
  int64_t off;        // first term of the tile, relative to the start of its segment
  int count;          // terms in the tile (<= tile_terms)
  int seg;            // segment; bit 31 set iff this is the segment's first tile
  int64_t start0;     // absolute first term in the FIRST pass's input (base_in[seg] + off)
  int64_t start;      // absolute first term in every later pass's input (seg[seg] + off)
};
// A pass reads segment g at base_in[g] + off.  base_in is the offset array itself except for the
// first pass after the grouped operator step (dense.cu), whose output sits at the slot offsets of
// the generators with gaps behind the kept terms; every pass WRITES the compact layout seg[g].

static __global__ void k_sort_tilemap(const int64_t* __restrict__ seg, const int64_t* __restrict__ base0, int n_seg,
                                      const int64_t* __restrict__ tile_prefix, TileInfo* __restrict__ info,
                                      int tile_terms) {
  const int64_t total_tiles = tile_prefix[n_seg];
  for (int64_t tile = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; tile < total_tiles;
       tile += (int64_t)gridDim.x * blockDim.x) {
    const int g = tile_segment(tile_prefix, n_seg, tile);
    TileInfo ti;
    ti.off = (tile - tile_prefix[g]) * tile_terms;
    ti.count = (int)min((int64_t)tile_terms, seg[g + 1] - seg[g] - ti.off);
    ti.seg = g | (tile == tile_prefix[g] ? (int)0x80000000 : 0);
    ti.start0 = base0[g] + ti.off;
    ti.start = seg[g] + ti.off;
    info[tile] = ti;
  }
}

// ---------------------------------------------------------------------------------
// histogram: hist[g][pass][digit], all passes in one read of the keys
// ---------------------------------------------------------------------------------
constexpr int kMaxPasses = 8;

template <typename K>
static __global__ void __launch_bounds__(kSortThreads)
k_sort_hist(const K* __restrict__ keys, const int64_t* __restrict__ base_in, const TileInfo* __restrict__ info,
            const int64_t* __restrict__ n_tiles, u32* __restrict__ hist, int passes) {
  __shared__ u32 sh[kMaxPasses][QX_RADIX];
  for (int i = threadIdx.x; i < kMaxPasses * QX_RADIX; i += kSortThreads) (&sh[0][0])[i] = 0u;
  __syncthreads();
  const int64_t total_tiles = *n_tiles;
  int cur_g = -1;
  for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const TileInfo ti = info[tile];
    const int g = ti.seg & 0x7fffffff;
    if (g != cur_g) {
      if (cur_g >= 0) {
        __syncthreads();
        for (int i = threadIdx.x; i < passes * QX_RADIX; i += kSortThreads) {
          const u32 c = (&sh[0][0])[i];
          if (c) atomicAdd(hist + (size_t)cur_g * passes * QX_RADIX + i, c);
          (&sh[0][0])[i] = 0u;
        }
        __syncthreads();
      }
      cur_g = g;
    }
    const int64_t start = base_in[g] + ti.off;
    const int count = ti.count;
    {   // this CTA's next tile: have it in L2 by then
      const int64_t nt = tile + gridDim.x;
      if (nt < total_tiles) {
        const TileInfo tn = info[nt];
        prefetch_l2(keys + base_in[tn.seg & 0x7fffffff] + tn.off, tn.count);
      }
    }
    const int rounds = (count + kSortThreads - 1) / kSortThreads;
#pragma unroll 4
    for (int k = 0; k < rounds; ++k) {
      const int idx = k * kSortThreads + threadIdx.x;
      const bool live = idx < count;
      const K key = live ? ld_stream(keys + start + idx) : (K)0;
      const u32 alive = __ballot_sync(QX_FULL_MASK, live);
      for (int p = 0; p < passes; ++p) {
        const u32 d = (u32)(key >> (QX_RADIX_BITS * p)) & (QX_RADIX - 1);
        // Pauli words are sparse: whole warps often share a digit; count those once.
        const u32 d0 = __shfl_sync(QX_FULL_MASK, d, __ffs(alive | 0x80000000u) - 1);
        const bool same = __all_sync(QX_FULL_MASK, !live || d == d0);
        if (same) {
          if (live && lane_id() == (u32)(__ffs(alive) - 1)) atomicAdd(&sh[p][d], (u32)__popc(alive));
        } else if (live) {
          atomicAdd(&sh[p][d], 1u);
        }
      }
    }
  }
  if (cur_g >= 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < passes * QX_RADIX; i += kSortThreads) {
      const u32 c = (&sh[0][0])[i];
      if (c) atomicAdd(hist + (size_t)cur_g * passes * QX_RADIX + i, c);
    }
  }
}

// counts -> exclusive digit offsets inside the segment, in place; one block per (g, pass)
static __global__ void __launch_bounds__(QX_RADIX) k_sort_scan_hist(u32* __restrict__ hist) {
  __shared__ u32 s_scan[QX_RADIX / 32 + 1];
  u32* row = hist + (size_t)blockIdx.x * QX_RADIX;
  const u32 c = row[threadIdx.x];
  u32 total;
  const u32 excl = block_exclusive_sum<u32>(c, s_scan, total);
  row[threadIdx.x] = excl;
}

// ---------------------------------------------------------------------------------
// one onesweep pass
// ---------------------------------------------------------------------------------
template <typename K, typename V, int THREADS, int ITEMS>
struct SortSmem {
  u32 whist[THREADS / 32][QX_RADIX];  // per-warp digit counters -> exclusive warp offsets
  u32 gbase[QX_RADIX];                // index inside the segment of slot 0 of each digit, minus tile_start (mod 2^32)
  u32 scan[THREADS / 32 + 1];
  V vals[THREADS * ITEMS];
  K keys[THREADS * ITEMS];
};

// THREADS x ITEMS terms per tile, warp-striped; LB = predecessors read per look-back round trip.
// Lanes of the warp whose 8-bit digit equals mine.  Hand-scheduled: one R2P moves the digit's
// bits into predicates, then per bit one VOTE and two logic ops (the compiler's version of the
// same loop spends six instructions per bit; this kernel is issue-bound, profiles/r01b).
__device__ __forceinline__ u32 match_digit8(u32 d) {
  u32 peers;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      ".reg .b32 v, t;\n"
      "mov.b32 %0, 0xffffffff;\n"
#define QX_MATCH_BIT(m)                                  \
      "and.b32 t, %1, " #m ";\n"                         \
      "setp.ne.b32 p, t, 0;\n"                           \
      "vote.sync.ballot.b32 v, p, 0xffffffff;\n"         \
      "@!p not.b32 v, v;\n"                              \
      "and.b32 %0, %0, v;\n"
      QX_MATCH_BIT(1) QX_MATCH_BIT(2) QX_MATCH_BIT(4) QX_MATCH_BIT(8)
      QX_MATCH_BIT(16) QX_MATCH_BIT(32) QX_MATCH_BIT(64) QX_MATCH_BIT(128)
#undef QX_MATCH_BIT
      "}\n"
      : "=r"(peers)
      : "r"(d));
  return peers;
}

// digit = byte `which` of the key: one PRMT on the right half instead of a 64-bit shift + mask
__device__ __forceinline__ u32 key_byte(u64 key, int which) {
  const u32 half = which < 4 ? (u32)key : (u32)(key >> 32);
  return __byte_perm(half, 0u, 0x4440u | (u32)(which & 3));
}
// narrow keys (2n <= 32 bits): the whole word is one register
__device__ __forceinline__ u32 key_byte(u32 key, int which) {
  return __byte_perm(key, 0u, 0x4440u | (u32)(which & 3));
}

// KO = type of the keys written: the last pass over narrow (32-bit) keys of a sort-only merge
// widens them to the store's 64-bit words on the way out.
template <typename K, typename V, int THREADS, int ITEMS, int LB, int MINB = (THREADS <= 256 ? 3 : 2),
          typename KO = K>
__global__ void __launch_bounds__(THREADS, MINB)
k_onesweep(const K* __restrict__ keys_in, const V* __restrict__ vals_in,
           KO* __restrict__ keys_out, V* __restrict__ vals_out,
           const int64_t* __restrict__ seg, const int64_t* __restrict__ base_in,
           const TileInfo* __restrict__ info,
           const int64_t* __restrict__ n_tiles, const u32* __restrict__ digit_base, int base_stride,
           u32* status, int which, int ahead, int debug, u32* __restrict__ bnd) {
  constexpr int WARPS = THREADS / 32;
  constexpr int TILE = THREADS * ITEMS;
  static_assert(THREADS >= QX_RADIX, "one thread per digit in the scan");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem<K, V, THREADS, ITEMS>& sm = *reinterpret_cast<SortSmem<K, V, THREADS, ITEMS>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();

  // Tile = blockIdx.x: CTAs of a 1-D grid are dispatched in index order, so a tile's predecessors
  // are resident or done when it looks back (the assumption cub::DeviceScan makes).  No ticket
  // atomic, no dependent offset-table load: the record holds the absolute start.
  for (int i = tid; i < WARPS * QX_RADIX / 4; i += THREADS)
    reinterpret_cast<uint4*>(&sm.whist[0][0])[i] = make_uint4(0u, 0u, 0u, 0u);
  const int64_t tile = qx_tile_id(status + (size_t)gridDim.x * QX_RADIX);   // the word behind the tiles' status words
  const int64_t total_tiles = *n_tiles;
  if (tile >= total_tiles) return;
  const TileInfo ti = info[tile];
  const bool pass0 = base_in != seg;
  const int g = ti.seg & 0x7fffffff;
  const bool first = ti.seg < 0;
  const int64_t start = pass0 ? ti.start0 : ti.start;
  const int count = ti.count;
  const bool full = count == TILE;
  const K* kin = keys_in + start;
  const V* vin = vals_in + start;
  // ---- load, warp-striped: warp w owns tile slots [w*32*ITEMS, (w+1)*32*ITEMS)
  K key[ITEMS];
  const int wslot = warp * (32 * ITEMS) + lane;
  if (full) {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) key[k] = ld_stream(kin + wslot + k * 32);
  } else {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int idx = wslot + k * 32;
      key[k] = idx < count ? ld_stream(kin + idx) : (K)~(K)0;       // padding sorts last
    }
  }
  // ---- L2 prefetch of the tile `ahead` positions behind this one (every tile is prefetched
  // exactly once): with ahead ~ resident CTAs the lines arrive in L2 just before use and the
  // loads above pay L2 latency instead of HBM latency.  Issued after this tile's own loads so
  // that the look-up of the far tile's record does not delay them.
  if (ahead > 0 && tile + ahead < total_tiles) {
    const TileInfo tp = info[tile + ahead];
    const int64_t sp = pass0 ? tp.start0 : tp.start;
    const int cp = tp.count;
    for (int i = tid * 16; i < cp; i += THREADS * 16) {      // one 128-byte line of doubles per step
      if (sizeof(K) == 8 || (i & 16) == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(keys_in + sp + i));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(vals_in + sp + i));
      if (sizeof(V) > 8) asm volatile("prefetch.global.L2 [%0];" ::"l"(vals_in + sp + i + 8));
    }
  }
  __syncthreads();

  // ---- early counts: per-warp digit histogram with fire-and-forget shared atomics.  Order
  // does not matter for counts, so the tile's aggregate can be published for the tiles behind
  // us BEFORE the (much longer) stable ranking -- their look-back then overlaps our ranking
  // instead of waiting for it (look-back stalls were 26 % of the pass, profiles/r01d).
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) atomicAdd(&sm.whist[warp][key_byte(key[k], which)], 1u);
  __syncthreads();

  // ---- per digit: exclusive offsets over warps, tile totals, exclusive scan over digits
  u32 digit_total = 0;
  u32 wcount[WARPS];
  if (tid < QX_RADIX) {
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      wcount[w] = sm.whist[w][tid];
      digit_total += wcount[w];
    }
  }
  u32 tile_sum;
  const u32 dstart = block_exclusive_sum<u32>(digit_total, sm.scan, tile_sum);
  // whist[w][d] <- first tile-sorted slot of warp w's terms with digit d: the digit's start in
  // the tile is folded in here, once per (warp, digit), so the ranking below needs no second
  // table look-up per term (random digits: 3.5 bank-conflict wavefronts per look-up, 12 % of the
  // pass's shared-memory wavefronts, and the LSU data pipe is its busiest unit, profiles/r01h)
  if (tid < QX_RADIX) {
    u32 running = dstart;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      sm.whist[w][tid] = running;
      running += wcount[w];
    }
  }
  // padding keys all carry digit 255 and sit behind the live ones
  const u32 live_total = digit_total - ((tid == QX_RADIX - 1) ? (u32)(TILE - count) : 0u);
  u32* mine = status + (size_t)tile * QX_RADIX + tid;
  const bool solo = first || (debug & 1);
  if (tid < QX_RADIX) st_volatile_u32(mine, (solo ? kFlagInc : kFlagAgg) | live_total);
  __syncthreads();

  // ---- stable rank inside the warp, straight into the tile-sorted slot.  Lanes with equal
  // digits form a group (match_digit8); the lowest lane advances the warp's running offset
  // for that digit with one shared atomic and everyone takes old + position in group.  The
  // shuffle that broadcasts `old` also orders item k's update before item k+1's (different
  // lanes may lead), which is what makes the ranking stable.
  u32 slot[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const u32 d = key_byte(key[k], which);
    const u32 peers = match_digit8(d);     // (the MATCH.ANY instruction is 1.4x slower per pass)
    const u32 below = __popc(peers & lanemask_lt());
    u32 old = 0;
    if (below == 0) old = atomicAdd(&sm.whist[warp][d], (u32)__popc(peers));
    slot[k] = __shfl_sync(QX_FULL_MASK, old, __ffs(peers) - 1) + below;
    sm.keys[slot[k]] = key[k];
  }
  // coefficients: cp.async straight into the tile-sorted slot -- no register staging and, above
  // all, no wait for the loads before the look-back below starts (with plain loads every thread
  // sat on its first coefficient for an L2/HBM round trip first: 0.787 -> 0.760 ms per pass)
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int idx = wslot + k * 32;
    if (full || idx < count) {
      const u32 dst = (u32)__cvta_generic_to_shared(&sm.vals[slot[k]]);
      if (sizeof(V) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(vin + idx) : "memory");
      else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(vin + idx) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");

  // ---- decoupled look-back, one chain per digit, confined to this segment's tiles.  Eight
  // predecessors are read per round trip: with ~300 tiles in flight the nearest inclusive
  // prefix is typically a dozen tiles back, and walking there one dependent L2 load at a
  // time was the critical path of the kernel.
  if (tid < QX_RADIX) {
    u32 excl = 0;
    if (!solo) {
      constexpr int W = LB;
      // predecessor j sits j * QX_RADIX words below sp: constant offsets, one compare per load
      const u32* sp = status + (size_t)(tile - 1) * QX_RADIX + tid;
      int avail = (int)(ti.off / TILE);           // predecessors inside this segment
      bool done = false;
      while (!done) {
        u32 w[W];
#pragma unroll
        for (int j = 0; j < W; ++j) w[j] = j < avail ? ld_volatile_u32(sp - j * QX_RADIX) : kFlagInc;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          if (!done) {
            while ((w[j] >> 30) == 0u) w[j] = ld_volatile_u32(sp - j * QX_RADIX);
            excl += w[j] & kFlagVal;
            done = (w[j] >> 30) == 2u;
          }
        }
        sp -= W * QX_RADIX;
        avail -= W;
      }
      st_volatile_u32(mine, kFlagInc | (excl + live_total));
    }
    sm.gbase[tid] = digit_base[(size_t)g * base_stride + tid] + excl - dstart;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  // ---- coalesced write-out: consecutive slots of one digit are consecutive in HBM.  Offsets are
  // 32-bit and relative to the segment (a segment holds < 2^30 terms): one IMAD.WIDE per store
  // instead of 64-bit index arithmetic per item.
  KO* kout = keys_out + seg[g];
  V* vout = vals_out + seg[g];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int slot = k * THREADS + tid;
    if (full || slot < count) {
      const K kk = sm.keys[slot];
      const u32 dst = sm.gbase[key_byte(kk, which)] + (u32)slot;
      st_stream(kout + dst, (KO)kk);
      st_stream(vout + dst, sm.vals[slot]);
      if (sizeof(KO) == 2) {
        // packed download format (last pass only): the key leaves as its low 16 bits; the high
        // 16 are recovered from bucket boundaries, bnd[g][h] = first position in generator g of
        // a key with high half h.  Tile-sorted order agrees with the final order, so a term whose
        // tile predecessor has the same high half is never the first of its bucket: ~300
        // candidates per tile, one RED.MIN each.
        const u32 hi = (u32)((u64)kk >> 16);
        if (slot == 0 || (u32)((u64)sm.keys[slot - 1] >> 16) != hi)
          atomicMin(bnd + (size_t)g * (QX_PACK_BUCKETS + 1) + hi, dst);
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// reduce-by-key + drop + compaction over the sorted segments
// ---------------------------------------------------------------------------------
template <typename K, typename V, int kRedThreads, int kRedItems>
struct ReduceSmem {
  static constexpr int kRedTile = kRedThreads * kRedItems;
  static constexpr int kRedWarps = kRedThreads / 32;
  alignas(16) V val[kRedTile];
  alignas(16) K key[kRedTile + 4];   // [kKeyAt - 1] = key before the tile, [kKeyAt ..] = tile (16-byte aligned: bulk copies)
  u32 opens[kRedTile / 32];    // bit j: tile slot j is the first term of a non-empty segment
  u64 scan[kRedWarps + 1];
  u64 base;
  alignas(8) u64 mbar;         // completion of the tile's bulk copies
  int tile;
  static constexpr int kKeyAt = 16 / (int)sizeof(K);   // 2 (64-bit keys) or 4 (32-bit keys)
};

// ---- TMA-style bulk copies (cp.async.bulk, sm_90+): a contiguous, 16-byte aligned block moves from
// global to shared memory without passing through registers or the LSU's per-thread path; one
// thread issues it, completion is counted in bytes on an mbarrier that every thread waits on.
__device__ __forceinline__ u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 arrivals) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(arrivals));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src_global, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst_smem)),
               "l"(src_global), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "QX_MBAR_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra QX_MBAR_DONE;\n"
      "bra QX_MBAR_WAIT;\n"
      "QX_MBAR_DONE:\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// One pass over the sorted segments: a term is a head if it opens a segment or its key differs
// from its predecessor's; the head sums its run sequentially (input order = np.add.at order),
// applies the drop rule, and kept heads are compacted with a ballot prefix + tile look-back.
// The tile (keys, coefficients, one halo key) is staged in shared memory with coalesced
// streaming loads, so every term is read from HBM exactly once and no thread searches the
// offset table; only runs that cross the tile end touch global memory again.
template <typename K, typename V, int kRedThreads, int kRedItems>
__global__ void __launch_bounds__(kRedThreads, (sizeof(V) == 8 && kRedThreads == 256) ? 6 : 1)
k_reduce(const K* __restrict__ keys_in, const V* __restrict__ vals_in,
         const int64_t* __restrict__ seg_in, int n_seg, u64* __restrict__ keys_out,
         V* __restrict__ vals_out, int64_t* __restrict__ seg_out, u64* status, u32* ticket,
         double eps, int debug) {
  constexpr int kRedTile = kRedThreads * kRedItems;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ReduceSmem<K, V, kRedThreads, kRedItems>& sm =
      *reinterpret_cast<ReduceSmem<K, V, kRedThreads, kRedItems>*>(smem_raw);
  if (threadIdx.x < kRedTile / 32) sm.opens[threadIdx.x] = 0u;
  const int tile = qx_tile_id(ticket);              // in-order dispatch, see qx_device.cuh
  const int64_t total = seg_in[n_seg];
  const int64_t ntiles = total > 0 ? (total + kRedTile - 1) / kRedTile : 1;
  if (tile >= ntiles) return;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t t0 = (int64_t)tile * kRedTile;
  const int cnt = (int)min((int64_t)kRedTile, total - t0);
  {
    const int64_t far = ((int64_t)tile + kPrefetchAhead) * kRedTile;
    if (far < total) {
      const int fc = (int)min((int64_t)kRedTile, total - far);
      prefetch_l2(keys_in + far, fc);
      prefetch_l2(vals_in + far, fc);
    }
  }

  constexpr int kKeyAt = ReduceSmem<K, V, kRedThreads, kRedItems>::kKeyAt;
#ifndef QX_NO_BULK_COPY
  // full tiles: two bulk copies (keys, coefficients) issued by one thread; the tile starts at a
  // multiple of kRedTile terms, so both sides are 16-byte aligned.  The last, partial tile takes
  // the per-thread loads.
  const bool bulk = cnt == kRedTile;
  if (bulk && threadIdx.x == 0) {
    mbar_init(&sm.mbar, 1);
    mbar_expect(&sm.mbar, (u32)(kRedTile * (sizeof(K) + sizeof(V))));
    bulk_load(&sm.key[kKeyAt], keys_in + t0, (u32)(kRedTile * sizeof(K)), &sm.mbar);
    bulk_load(&sm.val[0], vals_in + t0, (u32)(kRedTile * sizeof(V)), &sm.mbar);
  }
#else
  const bool bulk = false;
#endif
  if (!bulk) {
    for (int j = threadIdx.x; j < cnt; j += kRedThreads) {
      sm.key[kKeyAt + j] = ld_stream(keys_in + t0 + j);
      sm.val[j] = ld_stream(vals_in + t0 + j);
    }
  }
  if (threadIdx.x == 0) sm.key[kKeyAt - 1] = t0 > 0 ? keys_in[t0 - 1] : (K)0;
  {   // segments that start inside this tile
    int lo = 0, hi = n_seg;                         // first g with seg_in[g] >= t0
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (seg_in[mid] < t0) lo = mid + 1; else hi = mid;
    }
    for (int g = lo + threadIdx.x; g < n_seg; g += kRedThreads) {
      const int64_t at = seg_in[g];
      if (at >= t0 + cnt) break;
      if (seg_in[g + 1] > at) atomicOr(&sm.opens[(at - t0) >> 5], 1u << ((at - t0) & 31));
    }
  }
  __syncthreads();                                  // (also: the barrier's init is visible to the waiters)
  if (bulk) mbar_wait(&sm.mbar, 0);

  // A kept head leaves its sum in sm.val[j] (no other thread's run contains a head) and its key
  // stays in sm.key: the write-out re-reads both, so only `pre` and the flags live across the
  // look-back -- 40 registers instead of 62, six CTAs per SM instead of four (the kernel waits on
  // barriers and the look-back, occupancy is what hides that).
  u32 pre[kRedItems];          // kept heads before this item inside the warp
  u32 flags = 0;               // bit k: item k is a kept head; bit 16+k: item k opens a segment
  u32 running = 0;
#pragma unroll
  for (int k = 0; k < kRedItems; ++k) {
    const int j = warp * (32 * kRedItems) + k * 32 + lane;
    bool kept = false;
    if (j < cnt) {
      const K key = sm.key[kKeyAt + j];
      const bool opens = (sm.opens[j >> 5] >> (j & 31)) & 1u;
      if (opens) flags |= 1u << (16 + k);
      if (opens || sm.key[kKeyAt - 1 + j] != key) {
        V s = sm.val[j];
        int e = j + 1;
        while (e < cnt && sm.key[kKeyAt + e] == key && !((sm.opens[e >> 5] >> (e & 31)) & 1u)) {
          acc(s, sm.val[e]);
          ++e;
        }
        if (e == cnt && t0 + cnt < total) {          // the run may continue past the tile
          const int g = segment_of(seg_in, n_seg, t0 + j);
          const int64_t end = seg_in[g + 1];
          for (int64_t i = t0 + cnt; i < end && keys_in[i] == key; ++i) acc(s, vals_in[i]);
        }
        sm.val[j] = s;
        kept = keep(s, eps);
      }
    }
    if (kept) flags |= 1u << k;
    const u32 votes = __ballot_sync(QX_FULL_MASK, kept);
    pre[k] = running + __popc(votes & lanemask_lt());
    running += __popc(votes);
  }
  u64 tile_total;
  const u64 mine = (lane == 0) ? (u64)running : 0ull;
  u64 warp_excl = block_exclusive_sum<u64>(mine, sm.scan, tile_total);
  warp_excl = __shfl_sync(QX_FULL_MASK, warp_excl, 0);
  if (warp == 0) {
    const u64 excl = (debug & 2) ? (u64)tile * kRedTile : lookback_exclusive(status, tile, tile_total);
    if (lane == 0) sm.base = excl;
  }
  __syncthreads();
  const int64_t base = (int64_t)(sm.base + warp_excl);
#pragma unroll
  for (int k = 0; k < kRedItems; ++k) {
    const int64_t pos = base + pre[k];
    if (flags & (1u << k)) {
      const int j = warp * (32 * kRedItems) + k * 32 + lane;
      st_stream(keys_out + pos, (u64)sm.key[kKeyAt + j]);
      st_stream(vals_out + pos, sm.val[j]);
    }
    if (flags & (1u << (16 + k))) {
      const int64_t i = t0 + warp * (32 * kRedItems) + k * 32 + lane;
      open_offsets(seg_in, seg_out, segment_of(seg_in, n_seg, i), i, pos);
    }
  }
  if (tile == ntiles - 1 && threadIdx.x == 0)
    close_offsets(seg_in, seg_out, n_seg, total, (int64_t)(sm.base + tile_total));
}

// ---------------------------------------------------------------------------------
// small path: one CTA per segment, everything in shared memory
// ---------------------------------------------------------------------------------
constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;

template <typename V>
__global__ void __launch_bounds__(kSmallThreads)
k_small_merge(const u64* __restrict__ keys_in, const V* __restrict__ vals_in,
              const int64_t* __restrict__ seg_in, int n_seg, u64* __restrict__ keys_out,
              V* __restrict__ vals_out, int64_t* __restrict__ seg_out, u64* status, u32* ticket,
              int* error, int cap, double eps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* skey = reinterpret_cast<u64*>(smem_raw);                       // cap
  unsigned short* sidx = reinterpret_cast<unsigned short*>(skey + cap);   // cap
  __shared__ int s_g;
  __shared__ u64 s_scan[kSmallWarps + 1];
  __shared__ u64 s_base;
  const int g = qx_tile_id(ticket);      // in-order dispatch, see qx_device.cuh
  if (g >= n_seg) return;
  const int64_t start = seg_in[g];
  int len = (int)min((int64_t)0x7fffffff, seg_in[g + 1] - start);
  if (len > cap) {                       // host bound was wrong: flag it, keep the chain alive
    if (threadIdx.x == 0) atomicExch(error, 1);
    len = 0;
  }
  int m = 32;
  while (m < len) m <<= 1;
  for (int e = threadIdx.x; e < m; e += kSmallThreads) {
    skey[e] = e < len ? keys_in[start + e] : ~0ull;
    sidx[e] = (unsigned short)e;
  }
  __syncthreads();
  // bitonic network on (key, input position): position breaks ties, so equal keys
  // stay in input order and padding (key = max, position >= len) ends up last
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (m >> 1); t += kSmallThreads) {
        const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int hi = lo | j;
        const u64 ka = skey[lo], kb = skey[hi];
        const unsigned short ia = sidx[lo], ib = sidx[hi];
        const bool greater = ka > kb || (ka == kb && ia > ib);
        const bool ascending = (lo & k) == 0;
        if (greater == ascending) {
          skey[lo] = kb; skey[hi] = ka;
          sidx[lo] = ib; sidx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  // run sums (sequential, input order), drop rule, ordered compaction row by row
  const int rows = (len + kSmallThreads - 1) / kSmallThreads;
  u64 kept_before = 0;                   // kept heads in earlier rows
  // first sweep: count, so that the segment's output base is known before writing
  u64 my_count = 0;
  for (int r = 0; r < rows; ++r) {
    const int e = r * kSmallThreads + threadIdx.x;
    if (e < len) {
      const u64 key = skey[e];
      if (e == 0 || skey[e - 1] != key) {
        V s = vals_in[start + sidx[e]];
        for (int j = e + 1; j < len && skey[j] == key; ++j) acc(s, vals_in[start + sidx[j]]);
        if (keep(s, eps)) ++my_count;
      }
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
  for (int r = 0; r < rows; ++r) {
    const int e = r * kSmallThreads + threadIdx.x;
    bool kept = false;
    u64 key = 0;
    V s;
    if (e < len) {
      key = skey[e];
      if (e == 0 || skey[e - 1] != key) {
        s = vals_in[start + sidx[e]];
        for (int j = e + 1; j < len && skey[j] == key; ++j) acc(s, vals_in[start + sidx[j]]);
        kept = keep(s, eps);
      }
    }
    u64 row_total;
    const u64 excl = block_exclusive_sum<u64>(kept ? 1ull : 0ull, s_scan, row_total);
    if (kept) {
      const int64_t pos = base + (int64_t)(kept_before + excl);
      keys_out[pos] = key;
      vals_out[pos] = s;
    }
    kept_before += row_total;
  }
  if (threadIdx.x == 0) {
    seg_out[g] = base;
    if (g == n_seg - 1) seg_out[n_seg] = base + (int64_t)seg_total;
  }
}

// ---------------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------------
template <typename V>
struct MergeBuffers {
  u64* keys[2];
  V* vals[2];
  int64_t* seg[2];
  int cur;            // live buffer on entry; updated to the live buffer on exit
  int n_seg;
  int64_t ub_total;   // host upper bounds on the raw sizes
  int64_t ub_seg;
};

inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

template <typename V>
int merge_small(QxArena* ar, MergeBuffers<V>& mb, double eps, int cls) {
  int cap = 32;
  while (cap < mb.ub_seg) cap <<= 1;
  const size_t smem = (size_t)cap * (sizeof(u64) + sizeof(unsigned short));
  const int64_t bytes = 16 + 8 * ((int64_t)mb.n_seg + 1);
  QX_TRY(qx_arena_scratch(ar, bytes));
  QX_CUDA(cudaMemsetAsync(ar->scratch, 0, (size_t)bytes, ar->stream));
  u32* ticket = reinterpret_cast<u32*>(ar->scratch);
  int* error = reinterpret_cast<int*>(reinterpret_cast<char*>(ar->scratch) + 8);
  u64* status = reinterpret_cast<u64*>(reinterpret_cast<char*>(ar->scratch) + 16);
  static bool attr_set[2] = {false, false};
  const int which = sizeof(V) == 8 ? 0 : 1;
  if (!attr_set[which]) {
    QX_CUDA(cudaFuncSetAttribute(k_small_merge<V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 QX_SMALL_MAX * (int)(sizeof(u64) + sizeof(unsigned short))));
    attr_set[which] = true;
  }
  const int in = mb.cur, out = mb.cur ^ 1;
  {
    QxProfileScope prof(cls, ar->stream, (16.0 + sizeof(V)) * (double)mb.ub_total);
    k_small_merge<V><<<mb.n_seg, kSmallThreads, smem, ar->stream>>>(
        mb.keys[in], mb.vals[in], mb.seg[in], mb.n_seg, mb.keys[out], mb.vals[out], mb.seg[out],
        status, ticket, error, cap, eps);
    QX_CUDA(cudaGetLastError());
  }
  QX_CUDA(cudaMemcpyAsync(ar->h_pinned, error, sizeof(int), cudaMemcpyDeviceToHost, ar->stream));
  mb.cur = out;
  return QX_OK;     // caller synchronises and checks *(int*)h_pinned
}

struct SortVariant {
  int tile_terms;
  const char* name;
};

inline int sort_prefetch_distance(int sm_count) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("QX_SORT_PREFETCH");
    v = e ? atoi(e) : -1;
  }
  return v >= 0 ? v : 2 * sm_count;     // ~ resident CTAs (two per SM)
}

template <typename K, typename V, int THREADS, int ITEMS, int LB, int MINB = (THREADS <= 256 ? 3 : 2),
          typename KO = K>
int launch_pass(QxArena* ar, MergeBuffers<V>& mb, int cur, int64_t tiles_ub, const TileInfo* info,
                const int64_t* n_tiles, const u32* digit_base, int base_stride, int which,
                const int64_t* base_in, u32* bnd = nullptr) {
  using Smem = SortSmem<K, V, THREADS, ITEMS>;
  static bool attr_set = false;
  if (!attr_set) {
    QX_CUDA(cudaFuncSetAttribute(k_onesweep<K, V, THREADS, ITEMS, LB, MINB, KO>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
    attr_set = true;
  }
  k_onesweep<K, V, THREADS, ITEMS, LB, MINB, KO><<<(unsigned)tiles_ub, THREADS, sizeof(Smem), ar->stream>>>(
      reinterpret_cast<const K*>(mb.keys[cur]), mb.vals[cur], reinterpret_cast<KO*>(mb.keys[cur ^ 1]),
      mb.vals[cur ^ 1], mb.seg[cur], base_in ? base_in : mb.seg[cur], info, n_tiles,
      digit_base, base_stride, ar->status, which, sort_prefetch_distance(ar->sm_count),
      getenv("QX_SORT_DEBUG") ? atoi(getenv("QX_SORT_DEBUG")) : 0, bnd);
  QX_CUDA(cudaGetLastError());
  return QX_OK;
}

// Bucket table of the packed download: exclusive positions, entry QX_PACK_BUCKETS = rank.  The
// passes left bnd[g][h] = first position of a key with high half h (or ~0 for an empty bucket);
// a backward running minimum turns that into "first position of a key with high half >= h".
static __global__ void __launch_bounds__(1024) k_pack_bounds(u32* __restrict__ bnd, const int64_t* __restrict__ seg) {
  __shared__ u32 s_min[1024];
  constexpr int PER = QX_PACK_BUCKETS / 1024;
  u32* row = bnd + (size_t)blockIdx.x * (QX_PACK_BUCKETS + 1);
  const u32 rank = (u32)(seg[blockIdx.x + 1] - seg[blockIdx.x]);
  const int t = threadIdx.x;
  u32 m = 0xffffffffu;
  for (int i = 0; i < PER; ++i) m = min(m, row[t * PER + i]);
  s_min[t] = m;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {                 // suffix minimum over the chunks
    const u32 o = t + d < 1024 ? s_min[t + d] : 0xffffffffu;
    __syncthreads();
    s_min[t] = min(s_min[t], o);
    __syncthreads();
  }
  u32 carry = t + 1 < 1024 ? min(s_min[t + 1], rank) : rank;
  for (int i = PER - 1; i >= 0; --i) {
    carry = min(carry, row[t * PER + i]);
    row[t * PER + i] = carry;
  }
  if (t == 0) row[QX_PACK_BUCKETS] = rank;
}

// Tile geometry of the sort pass; QX_SORT_VARIANT picks one for A/B runs on the GPU.
inline int sort_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QX_SORT_VARIANT");
    v = e ? atoi(e) : 0;
    if (v < 0 || v > 6) v = 0;
  }
  return v;
}

inline int sort_tile_terms(int variant, size_t value_bytes) {
  if (value_bytes > 8) return 256 * 12;            // complex coefficients: one geometry
  switch (variant) {
    case 2: return 256 * 12;
    case 3: return 256 * 16;
    case 4: return 512 * 8;
    case 5: return 384 * 8;
    case 6: return 384 * 10;
    default: return 384 * 12;
  }
}

// WIDEN: the pass reads narrow keys and writes 64-bit ones (last pass of a narrow sort-only merge)
template <typename K, typename V, bool WIDEN = false>
int dispatch_pass(int variant, QxArena* ar, MergeBuffers<V>& mb, int cur, int64_t tiles_ub,
                  const TileInfo* info, const int64_t* n_tiles, const u32* digit_base, int base_stride,
                  int which, const int64_t* base_in = nullptr) {
  using KO = typename std::conditional<WIDEN, u64, K>::type;
  if (sizeof(V) > 8)
    return launch_pass<K, V, 256, 12, 8>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
  if constexpr (sizeof(K) == 4) {
    // narrow keys: 56 registers and 68 KB of shared memory per CTA -> three CTAs (36 warps) per SM
    // instead of two; the pass is latency-bound, not HBM-bound (profiles/r01g), so occupancy pays.
    // (if constexpr: these occupancies are never instantiated for 64-bit keys, where 56 registers
    // would spill -- the 64-bit variants below run two CTAs per SM at 85 registers, no stack)
    switch (variant) {
      case 2: return launch_pass<K, V, 256, 12, 8, 4, KO>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      case 3: return launch_pass<K, V, 256, 16, 8, 3, KO>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      case 4: return launch_pass<K, V, 512, 8, 8, 2, KO>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      case 5: return launch_pass<K, V, 384, 8, 8, 4, KO>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      case 6: return launch_pass<K, V, 384, 10, 8, 3, KO>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      default: return launch_pass<K, V, 384, 12, 8, 3, KO>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
    }
  } else {
    switch (variant) {
      case 2: return launch_pass<K, V, 256, 12, 8>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      case 3: return launch_pass<K, V, 256, 16, 8>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      case 4: return launch_pass<K, V, 512, 8, 8>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      case 5: return launch_pass<K, V, 384, 8, 8, 2>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      case 6: return launch_pass<K, V, 384, 10, 8>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
      default: return launch_pass<K, V, 384, 12, 8>(ar, mb, cur, tiles_ub, info, n_tiles, digit_base, base_stride, which, base_in);
    }
  }
}

// do_reduce = false: sort only (keys known unique and nothing to drop, e.g. after a run of
// Clifford gates) -- the segment offsets do not change and no rank read-back is needed.
// K = u32: the live buffer holds NARROW keys (one 32-bit word per term, 2n <= 32) as written by
// the fused expansion kernel; every pass then moves 12 B per term instead of 16 and the reduce
// widens back to the store's 64-bit keys.  Narrow keys never leave a merge.
// cls_pass / cls_hist: instrumentation classes of the passes (the dense operator path sorts its
// few source terms with this routine too and books them separately).
template <typename V, typename K = u64>
int merge_large(QxArena* ar, MergeBuffers<V>& mb, double eps, int cls_reduce, bool do_reduce = true,
                int cls_pass = QX_K_SORT_PASS, int cls_hist = QX_K_SORT_HIST,
                const int64_t* first_base_in = nullptr, const u32* pre_hist = nullptr, bool widen_last = true,
                u32* pack_bnd = nullptr, int key_bits = 0) {
  const int n_seg = mb.n_seg;
  // key_bits: bits of the key that can be set (default: the 2n of a one-word Pauli word)
  if (key_bits <= 0) key_bits = 2 * ar->n_qubits;
  const int passes = std::min(kMaxPasses, (key_bits + QX_RADIX_BITS - 1) / QX_RADIX_BITS);
  if (mb.ub_seg >= (int64_t)kFlagVal)
    return qx_fail(QX_ERR_RESOURCE, "a generator with %lld raw terms exceeds the sort's 2^30 limit",
                   (long long)mb.ub_seg);
  const int variant = sort_variant();
  const int tile_terms = sort_tile_terms(variant, sizeof(V));
  const int64_t tiles_ub = (mb.ub_total + tile_terms - 1) / tile_terms + n_seg;
  static const int red_variant = getenv("QX_REDUCE_VARIANT") ? atoi(getenv("QX_REDUCE_VARIANT")) : 0;
  const int red_tile = sizeof(V) > 8 ? 2048 : (red_variant == 1 ? 1024 : red_variant == 2 ? 2048 : red_variant == 3 ? 4096 : 2048);
  const int64_t red_tiles = std::max<int64_t>(1, (mb.ub_total + red_tile - 1) / red_tile);
  // scratch layout: ticket | tile_prefix | hist | reduce look-back | tile records
  const int64_t off_prefix = 256;
  const int64_t off_hist = align_up(off_prefix + 8 * ((int64_t)n_seg + 1), 256);
  const int64_t hist_bytes = 4ll * n_seg * passes * QX_RADIX;
  const int64_t off_red = align_up(off_hist + hist_bytes, 256);
  const int64_t off_info = align_up(off_red + 8 * (red_tiles + 1), 256);
  const int64_t zero_bytes = off_info;                       // the tile records are written, not cleared
  const int64_t total_bytes = off_info + (int64_t)sizeof(TileInfo) * tiles_ub;
  QX_TRY(qx_arena_scratch(ar, total_bytes));
  QX_TRY(qx_arena_status(ar, tiles_ub * QX_RADIX + 1));      // + the ticket word of QX_TICKETED_LOOKBACK builds
  char* base = reinterpret_cast<char*>(ar->scratch);
  u32* ticket = reinterpret_cast<u32*>(base);
  int64_t* tile_prefix = reinterpret_cast<int64_t*>(base + off_prefix);
  u32* hist = reinterpret_cast<u32*>(base + off_hist);
  u64* red_status = reinterpret_cast<u64*>(base + off_red);
  TileInfo* info = reinterpret_cast<TileInfo*>(base + off_info);
  const int64_t* n_tiles = tile_prefix + n_seg;
  QX_CUDA(cudaMemsetAsync(base, 0, (size_t)zero_bytes, ar->stream));

  int cur = mb.cur;
  k_sort_plan<<<1, 32, 0, ar->stream>>>(mb.seg[cur], n_seg, tile_prefix, ticket, tile_terms);
  k_sort_tilemap<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((tiles_ub + 255) / 256, 4096)), 256, 0, ar->stream>>>(
      mb.seg[cur], first_base_in ? first_base_in : mb.seg[cur], n_seg, tile_prefix, info, tile_terms);
  qx_count_launches(2);
  QX_CUDA(cudaGetLastError());
  if (pre_hist) {
    // the producer of the keys counted their digits already (dense.cu); its buffer is scanned
    // in place and outlives the passes (no device-to-device copy: a copy engine may be busy
    // with another store's download)
    hist = const_cast<u32*>(pre_hist);
  } else {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_ub, (int64_t)ar->sm_count * 4));
    QxProfileScope prof(cls_hist, ar->stream, (double)sizeof(K) * (double)mb.ub_total);
    k_sort_hist<K><<<grid, kSortThreads, 0, ar->stream>>>(reinterpret_cast<const K*>(mb.keys[cur]),
                                                          first_base_in ? first_base_in : mb.seg[cur], info,
                                                          n_tiles, hist, passes);
    QX_CUDA(cudaGetLastError());
  }
  k_sort_scan_hist<<<n_seg * passes, QX_RADIX, 0, ar->stream>>>(hist);
  qx_count_launches(1);
  QX_CUDA(cudaGetLastError());
  // the offsets do not change under a sort; both buffers need them for the ping-pong
  QX_CUDA(cudaMemcpyAsync(mb.seg[cur ^ 1], mb.seg[cur], sizeof(int64_t) * (size_t)(n_seg + 1),
                          cudaMemcpyDeviceToDevice, ar->stream));
  for (int p = 0; p < passes; ++p) {
    QX_CUDA(cudaMemsetAsync(ar->status, 0, sizeof(u32) * (size_t)(tiles_ub * QX_RADIX + 1), ar->stream));
    QxProfileScope prof(cls_pass, ar->stream, 2.0 * (sizeof(K) + sizeof(V)) * (double)mb.ub_total);
    if (!do_reduce && sizeof(K) == 4 && p == passes - 1 && pack_bnd) {
      // packed download: 16-bit keys + bucket table (see k_onesweep's write-out)
      if constexpr (sizeof(K) == 4 && sizeof(V) == 8) {
        QX_CUDA(cudaMemsetAsync(pack_bnd, 0xff, sizeof(u32) * (size_t)n_seg * (QX_PACK_BUCKETS + 1), ar->stream));
        QX_TRY((launch_pass<u32, V, 384, 12, 8, 3, unsigned short>(
            ar, mb, cur, tiles_ub, info, n_tiles, hist + (size_t)p * QX_RADIX, passes * QX_RADIX, p,
            p == 0 ? first_base_in : nullptr, pack_bnd)));
        k_pack_bounds<<<n_seg, 1024, 0, ar->stream>>>(pack_bnd, mb.seg[cur]);
        qx_count_launches(1);
        QX_CUDA(cudaGetLastError());
      }
    } else if (!do_reduce && sizeof(K) == 4 && p == passes - 1 && widen_last)
      QX_TRY((dispatch_pass<K, V, true>(variant, ar, mb, cur, tiles_ub, info, n_tiles, hist + (size_t)p * QX_RADIX,
                                        passes * QX_RADIX, p, p == 0 ? first_base_in : nullptr)));
    else
      QX_TRY((dispatch_pass<K, V>(variant, ar, mb, cur, tiles_ub, info, n_tiles, hist + (size_t)p * QX_RADIX,
                                  passes * QX_RADIX, p, p == 0 ? first_base_in : nullptr)));
    cur ^= 1;
  }
  if (!do_reduce) {
    mb.cur = cur;
    return QX_OK;
  }
  QX_CUDA(cudaMemsetAsync(ticket, 0, sizeof(u32), ar->stream));
  {
    QxProfileScope prof(cls_reduce, ar->stream, (sizeof(K) + 8.0 + 2.0 * sizeof(V)) * (double)mb.ub_total);
#define QX_LAUNCH_REDUCE(T, I)                                                                        \
  do {                                                                                                \
    static bool attr = false;                                                                         \
    if (!attr) {                                                                                      \
      QX_CUDA(cudaFuncSetAttribute(k_reduce<K, V, T, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                   (int)sizeof(ReduceSmem<K, V, T, I>)));                             \
      attr = true;                                                                                    \
    }                                                                                                 \
    k_reduce<K, V, T, I><<<(unsigned)red_tiles, T, sizeof(ReduceSmem<K, V, T, I>), ar->stream>>>(     \
        reinterpret_cast<const K*>(mb.keys[cur]), mb.vals[cur], mb.seg[cur], n_seg, mb.keys[cur ^ 1], \
        mb.vals[cur ^ 1],                                                                             \
        mb.seg[cur ^ 1], red_status, ticket, eps,                                                     \
        getenv("QX_SORT_DEBUG") ? atoi(getenv("QX_SORT_DEBUG")) : 0);                                 \
  } while (0)
    if (sizeof(V) > 8 || red_variant == 0) QX_LAUNCH_REDUCE(256, 8);
    else if (red_variant == 1) QX_LAUNCH_REDUCE(128, 8);
    else if (red_variant == 2) QX_LAUNCH_REDUCE(128, 16);
    else QX_LAUNCH_REDUCE(512, 8);
#undef QX_LAUNCH_REDUCE
    QX_CUDA(cudaGetLastError());
  }
  mb.cur = cur ^ 1;
  return QX_OK;
}

}  // namespace qxm
