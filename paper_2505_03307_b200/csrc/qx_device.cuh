// Device-side building blocks: warp/block scans, decoupled look-back, segment lookup.
#pragma once

#include "qx_internal.cuh"

#define QX_FULL_MASK 0xffffffffu

// ---- streaming loads/stores -------------------------------------------------
// Term arrays are touched once per pass: keep them out of L1 so the 126 MB L2
// and the look-back words are not evicted by them.
__device__ __forceinline__ u64 ld_stream(const u64* p) { return __ldcs(p); }
__device__ __forceinline__ u32 ld_stream(const u32* p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(u64* p, u64 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(u32* p, u32 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(unsigned short* p, unsigned short v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }

__device__ __forceinline__ u32 ld_volatile_u32(const u32* p) {
  u32 v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ u64 ld_volatile_u64(const u64* p) {
  u64 v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile_u32(u32* p, u32 v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ void st_volatile_u64(u64* p, u64 v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- warp / block scans -------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(QX_FULL_MASK, v, d);
    if (lane_id() >= (u32)d) v += o;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(QX_FULL_MASK, v, d);
  return v;
}

// Exclusive prefix of `v` over the block in thread order; `total` = block sum.
// `smem` needs (blockDim.x / 32) + 1 entries.  Two __syncthreads.
template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* smem, T& total) {
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  T incl = warp_inclusive_sum(v);
  if (lane_id() == 31) smem[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = (lane_id() < (u32)nwarps) ? smem[lane_id()] : T(0);
    T wi = warp_inclusive_sum(w);
    if (lane_id() < (u32)nwarps) smem[lane_id()] = wi - w;
    if (lane_id() == 31) smem[nwarps] = wi;
  }
  __syncthreads();
  T out = smem[warp] + incl - v;
  total = smem[nwarps];
  __syncthreads();   // smem may be reused by the caller right away
  return out;
}

// ---- decoupled look-back over tiles, one 64-bit value per tile ------------------
// status word: bits 63-62 = 0 not ready, 1 tile aggregate, 2 inclusive prefix.
// Tiles must be taken in ticket order so that every predecessor is already running.
constexpr u64 QX_LB_AGG = 1ull << 62;
constexpr u64 QX_LB_INC = 2ull << 62;
constexpr u64 QX_LB_VAL = (1ull << 62) - 1;

// Called by all 32 lanes of ONE warp; returns the exclusive prefix of `aggregate`.
// R status words per lane per round trip (32 * R predecessors): with hundreds of tiles in
// flight a new tile starts every ~10-25 ns, so a walker that consumes only 32 predecessors
// per L2 round trip (~0.4 us) cannot catch up with the frontier of resolved tiles.
template <int R = 1>
__device__ __forceinline__ u64 lookback_exclusive(u64* status, int tile, u64 aggregate) {
  if (tile == 0) {
    if (lane_id() == 0) st_volatile_u64(status, QX_LB_INC | aggregate);
    return 0;
  }
  if (lane_id() == 0) st_volatile_u64(status + tile, QX_LB_AGG | aggregate);
  u64 excl = 0;
  int base = tile - 1;
  bool done = false;
  while (!done) {
    u64 w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int t = base - r * 32 - (int)lane_id();
      w[r] = t >= 0 ? ld_volatile_u64(status + t) : QX_LB_INC;   // before tile 0: inclusive 0
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!done) {
        const int t = base - r * 32 - (int)lane_id();
        while ((w[r] >> 62) == 0) w[r] = ld_volatile_u64(status + t);
        const u32 inc = __ballot_sync(QX_FULL_MASK, (w[r] >> 62) == 2);
        u64 v = w[r] & QX_LB_VAL;
        if (inc) {
          const int first = __ffs(inc) - 1;     // nearest tile holding an inclusive prefix
          if ((int)lane_id() > first) v = 0;
          done = true;
        }
        excl += warp_sum(v);
      }
    }
    base -= 32 * R;
  }
  if (lane_id() == 0) st_volatile_u64(status + tile, QX_LB_INC | (excl + aggregate));
  return excl;
}

// ---- segment lookup ---------------------------------------------------------------
// Largest g in [0, n_seg) with off[g] <= i, skipping empty segments (off[g+1] > i).
__device__ __forceinline__ int segment_of(const int64_t* off, int n_seg, int64_t i) {
  int lo = 0, hi = n_seg;                   // invariant: off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// ---- Pauli-word helpers --------------------------------------------------------------
// bit 2p set iff the digit at bit position 2p is not the identity
__device__ __forceinline__ u64 support_mask(u64 key) {
  return (key | (key >> 1)) & 0x5555555555555555ull;
}
// true iff the word has no X or Y digit (x bit = hi ^ lo)
__device__ __forceinline__ bool zi_only(u64 key) {
  return (((key >> 1) ^ key) & 0x5555555555555555ull) == 0;
}

// ---- tile tickets and segment-offset bookkeeping of the single-pass kernels ------------
// Dynamic tile id: tiles are handed out in launch order so look-back never waits on
// a tile that has not started.
// Tile id of a look-back kernel: blockIdx.x.  CTAs of a 1-D grid are dispatched in index order,
// so every predecessor a tile may wait for is resident or finished (the assumption
// cub::DeviceScan makes); an atomic ticket per CTA cost a ~700-cycle round trip at the head of
// every tile.  That order is observed hardware behaviour, not a documented guarantee: building
// with -DQX_TICKETED_LOOKBACK hands the ids out by an atomic counter instead (every launch site
// zeroes one), which is correct under ANY dispatch order; the GPU suite is run once with that
// build (profiles/r02_ticketed_lookback.txt).
__device__ __forceinline__ int qx_tile_id(u32* ticket) {
#ifdef QX_TICKETED_LOOKBACK
  __shared__ int s_ticketed_tile;
  if (threadIdx.x == 0) s_ticketed_tile = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  return s_ticketed_tile;
#else
  (void)ticket;
  return (int)blockIdx.x;
#endif
}
// The barrier is kept: callers publish shared state before it.
__device__ __forceinline__ int take_ticket(u32* ticket, int*) {
  const int tile = qx_tile_id(ticket);
  __syncthreads();
  return tile;
}

// L2 prefetch of `count` elements starting at p (whole 128-byte lines, all threads of the CTA)
template <typename T>
__device__ __forceinline__ void prefetch_l2(const T* p, int count) {
  constexpr int kPerLine = 128 / (int)sizeof(T);
  for (int i = (int)threadIdx.x * kPerLine; i < count; i += (int)blockDim.x * kPerLine)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + i));
}
constexpr int kPrefetchAhead = 592;     // tiles: about the CTAs resident on the device

// After the last real term: every segment starting at `total_in` (trailing empties
// and the end sentinel) starts at `total_out`.
__device__ __forceinline__ void close_offsets(const int64_t* seg_in, int64_t* seg_out, int n_seg,
                                              int64_t total_in, int64_t total_out) {
  for (int g = n_seg; g >= 0 && seg_in[g] == total_in; --g) seg_out[g] = total_out;
}

// Segment g starts at input index i and lands at output index pos; empty segments
// that start at the same index land there too.
__device__ __forceinline__ void open_offsets(const int64_t* seg_in, int64_t* seg_out, int g,
                                             int64_t i, int64_t pos) {
  seg_out[g] = pos;
  for (int h = g - 1; h >= 0 && seg_in[h] == i; --h) seg_out[h] = pos;
}

