// Term hash-partition for multi-GPU rebalancing.  Not in the
// reference (it is single-process); this is the device half of the all-to-all-v that
// re-homes terms by owner = mix(key) % world before a merge, used when there are
// fewer generators than GPUs or one generator dominates.
//
//   qx_store_partition_by_owner  live terms -> [owner 0: seg 0..S-1][owner 1: ...] + counts
//   qx_store_assemble            received  [source 0: seg 0..S-1][source 1: ...] -> store
//
// One stable compaction pass per owner (warp ballot prefix + look-back, like the v1
// split), so terms keep their relative order and the following merge stays deterministic.
#include <algorithm>
#include <vector>

#include "qx_device.cuh"

namespace {

constexpr int kThreads = QX_SCAN_THREADS;
constexpr int kItems = QX_SCAN_ITEMS;
constexpr int kTile = QX_SCAN_TILE;
constexpr int kWarps = kThreads / 32;

__host__ __device__ __forceinline__ u64 mix64(u64 z) {      // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// totals[0] = terms already placed (owners < rank); the last tile adds this owner's total.
__global__ void __launch_bounds__(kThreads)
k_partition_select(const u64* __restrict__ keys_in, const double* __restrict__ lam_in,
                   const int64_t* __restrict__ seg_in, int n_seg, u64* __restrict__ keys_out,
                   double* __restrict__ lam_out, int64_t* __restrict__ seg_pos, int64_t* totals,
                   u64* status, u32* ticket, u32 world, u32 rank) {
  __shared__ int s_tile;
  __shared__ u64 s_scan[kWarps + 1];
  __shared__ u64 s_base;
  const int tile = take_ticket(ticket, &s_tile);
  const int64_t total = seg_in[n_seg];
  const int64_t ntiles = total > 0 ? (total + kTile - 1) / kTile : 1;
  if (tile >= ntiles) return;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t wbase = (int64_t)tile * kTile + (int64_t)warp * (32 * kItems);
  const int64_t placed = totals[rank];
  u64 key[kItems];
  u32 pre[kItems];
  u32 mineflags = 0, running = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    key[k] = i < total ? ld_stream(keys_in + i) : 0ull;
    const bool sel = i < total && (u32)(mix64(key[k]) % world) == rank;
    if (sel) mineflags |= 1u << k;
    const u32 votes = __ballot_sync(QX_FULL_MASK, sel);
    pre[k] = running + __popc(votes & lanemask_lt());
    running += __popc(votes);
  }
  u64 tile_total;
  const u64 mine = (lane == 0) ? (u64)running : 0ull;
  u64 warp_excl = block_exclusive_sum<u64>(mine, s_scan, tile_total);
  warp_excl = __shfl_sync(QX_FULL_MASK, warp_excl, 0);
  if (warp == 0) {
    const u64 excl = lookback_exclusive(status, tile, tile_total);
    if (lane == 0) s_base = excl;
  }
  __syncthreads();
  const int64_t base = (int64_t)(s_base + warp_excl);
  // one segment search per warp instead of one per term (see k_split): almost no warp holds a boundary
  const int g_warp = segment_of(seg_in, n_seg, min(wbase, total - 1));
  const bool no_opens = seg_in[g_warp] < wbase && seg_in[g_warp + 1] >= wbase + 32 * kItems;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = wbase + k * 32 + lane;
    if (i >= total) continue;
    const int64_t rel = base + pre[k];               // selected terms before i
    if (mineflags & (1u << k)) {
      keys_out[placed + rel] = key[k];
      lam_out[placed + rel] = lam_in[i];
    }
    if (!no_opens) {
      const int g = segment_of(seg_in, n_seg, i);
      if (seg_in[g] == i) open_offsets(seg_in, seg_pos, g, i, rel);
    }
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) {
    const int64_t sel_total = (int64_t)(s_base + tile_total);
    close_offsets(seg_in, seg_pos, n_seg, total, sel_total);
    totals[rank + 1] = placed + sel_total;
  }
}

}  // namespace

extern "C" int qx_store_partition_by_owner(qx_store* s, int32_t world, int64_t* send_counts) {
  if (s) QX_NARROW_ONLY(s, "qx_store_partition_by_owner");
  QX_REQUIRE(s && send_counts, "NULL argument");
  QX_REQUIRE(world >= 1 && world <= 64, "world size %d out of range", world);
  QX_CUDA(cudaSetDevice(s->device));
  if (!s->exact) QX_TRY(qx_store_refresh(s));
  const int64_t total = s->h_seg[s->n_seg];
  const int64_t tiles = std::max<int64_t>(1, (total + kTile - 1) / kTile);
  // scratch: ticket | status[tiles+1] | totals[world+1] | seg_pos[world][n_seg+1]
  const int64_t off_status = 8;
  const int64_t off_totals = off_status + 8 * (tiles + 1);
  const int64_t off_pos = off_totals + 8 * ((int64_t)world + 1);
  const int64_t bytes = off_pos + 8ll * world * (s->n_seg + 1);
  QX_TRY(qx_store_scratch(s, bytes));
  char* base = reinterpret_cast<char*>(s->scratch);
  u32* ticket = reinterpret_cast<u32*>(base);
  u64* status = reinterpret_cast<u64*>(base + off_status);
  int64_t* totals = reinterpret_cast<int64_t*>(base + off_totals);
  int64_t* seg_pos = reinterpret_cast<int64_t*>(base + off_pos);
  QX_CUDA(cudaMemsetAsync(base, 0, (size_t)bytes, s->stream));
  const int in = s->cur, out = s->cur ^ 1;
  for (int r = 0; r < world; ++r) {
    if (r > 0) QX_CUDA(cudaMemsetAsync(base, 0, (size_t)off_totals, s->stream));
    QxProfileScope prof(QX_K_PARTITION, s->stream, 8.0 * (double)total + 32.0 * (double)total / world);
    k_partition_select<<<(unsigned)tiles, kThreads, 0, s->stream>>>(
        s->keys[in], s->lam[in], s->seg[in], s->n_seg, s->keys[out], s->lam[out],
        seg_pos + (size_t)r * (s->n_seg + 1), totals, status, ticket, (u32)world, (u32)r);
    QX_CUDA(cudaGetLastError());
  }
  std::vector<int64_t> pos((size_t)world * (s->n_seg + 1));
  QX_CUDA(cudaMemcpyAsync(pos.data(), seg_pos, sizeof(int64_t) * pos.size(), cudaMemcpyDeviceToHost,
                          s->stream));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  for (int r = 0; r < world; ++r)
    for (int g = 0; g < s->n_seg; ++g)
      send_counts[(size_t)r * s->n_seg + g] =
          pos[(size_t)r * (s->n_seg + 1) + g + 1] - pos[(size_t)r * (s->n_seg + 1) + g];
  // the partitioned image is the live buffer now; offsets describe it as ONE run per
  // segment no longer -- callers must follow with qx_store_assemble (or upload).
  qx_store_flip(s);
  QX_CUDA(cudaMemcpyAsync(s->seg[s->cur], s->seg[in], sizeof(int64_t) * (size_t)(s->n_seg + 1),
                          cudaMemcpyDeviceToDevice, s->stream));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  return QX_OK;
}

extern "C" int qx_store_assemble(qx_store* s, const uint64_t* d_keys, const double* d_lambdas,
                                 int32_t world, const int64_t* recv_counts) {
  if (s) QX_NARROW_ONLY(s, "qx_store_assemble");
  QX_REQUIRE(s && recv_counts, "NULL argument");
  QX_REQUIRE(world >= 1 && world <= 64, "world size %d out of range", world);
  QX_CUDA(cudaSetDevice(s->device));
  const int S = s->n_seg;
  int64_t total = 0;
  for (int i = 0; i < world * S; ++i) {
    QX_REQUIRE(recv_counts[i] >= 0, "negative chunk count");
    total += recv_counts[i];
  }
  QX_REQUIRE(total == 0 || (d_keys && d_lambdas), "device pointers are NULL");
  // never assemble in place: the source may alias the live buffer (loop-back, world = 1)
  QX_TRY(qx_store_reserve(s, total, true));
  const int out = s->cur ^ 1;
  std::vector<int64_t> src_off((size_t)world * S + 1, 0);
  for (int i = 0; i < world * S; ++i) src_off[i + 1] = src_off[i] + recv_counts[i];
  int64_t at = 0;
  for (int g = 0; g < S; ++g) {
    s->h_seg[g] = at;
    for (int q = 0; q < world; ++q) {
      const int64_t n = recv_counts[(size_t)q * S + g];
      if (n == 0) continue;
      const int64_t from = src_off[(size_t)q * S + g];
      QX_CUDA(cudaMemcpyAsync(s->keys[out] + at, d_keys + from, sizeof(u64) * (size_t)n,
                              cudaMemcpyDeviceToDevice, s->stream));
      QX_CUDA(cudaMemcpyAsync(s->lam[out] + at, d_lambdas + from, sizeof(double) * (size_t)n,
                              cudaMemcpyDeviceToDevice, s->stream));
      at += n;
    }
  }
  s->h_seg[S] = at;
  QX_CUDA(cudaMemcpyAsync(s->seg[out], s->h_seg, sizeof(int64_t) * (size_t)(S + 1),
                          cudaMemcpyHostToDevice, s->stream));
  QX_CUDA(cudaStreamSynchronize(s->stream));
  qx_store_flip(s);
  s->exact = true;
  s->ub_total = at;
  s->ub_seg = 0;
  for (int g = 0; g < S; ++g) s->ub_seg = std::max(s->ub_seg, s->h_seg[g + 1] - s->h_seg[g]);
  return QX_OK;
}
