// a2 + Clifford part of a3: fused gate-apply for sign-permutation gates.
//
// Replaces apply_cx (reference stabilizer.py:340-363, tables lut.py:108-134) and
// the H/S/X/SX cases of _apply_1q_terms (engine.py:183-218), plus every composed
// U_k block that is a signed axis permutation (v3 path, stabilizer.py:264-270).
// One launch pushes each term through the WHOLE run of gates in registers: the
// term is read once and written once however long the run is (2 * 16 B per term
// per run instead of per gate).  Conjugation by a Clifford is a bijection on
// Pauli words and leaves |lambda| unchanged, so the merge the reference performs
// after these gates can only re-sort; it is deferred to the next real merge.
//
// HBM-bound elementwise kernel: 128-bit loads/stores (two terms per thread per
// step), gate program broadcast from shared memory, grid = SMs * resident CTAs.
#include <string.h>

#include <algorithm>

#include "qx_device.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kProgChunk = 960;     // ops per launch: the program travels as a kernel parameter

// The gate program sits in the parameter (constant) bank: every thread reads the same word,
// so the field decode (kind, shifts, table) runs once per warp on the uniform datapath
// instead of once per thread.
struct Program {
  u32 n_ops;
  u32 ops[kProgChunk];
};

struct CxTables {
  u32 c, t, s;
};

// K = u32 when the word fits 32 bits (n <= 16): the kernel is ALU-bound and 64-bit variable
// shifts cost two to three instructions each.
template <typename K>
__device__ __forceinline__ void apply_op(u32 op, K& key, u32& neg, const CxTables cx) {
  const u32 s0 = (op >> 2) & 63u;
  const u32 d0 = (u32)(key >> s0) & 3u;
  if ((op & 3u) == 0u) {
    const u32 nd = (op >> (16u + 2u * d0)) & 3u;
    neg ^= (op >> (24u + d0)) & 1u;
    key ^= (K)(d0 ^ nd) << s0;
  } else {
    const u32 s1 = (op >> 8) & 63u;
    const u32 d1 = (u32)(key >> s1) & 3u;
    const u32 e = d0 * 4u + d1;
    const u32 n0 = (cx.c >> (2u * e)) & 3u;
    const u32 n1 = (cx.t >> (2u * e)) & 3u;
    neg ^= (cx.s >> e) & 1u;
    key ^= ((K)(d0 ^ n0) << s0) | ((K)(d1 ^ n1) << s1);
  }
}

template <typename K>
__global__ void __launch_bounds__(kThreads)
k_clifford_run(u64* __restrict__ keys, double* __restrict__ lam,
               const int64_t* __restrict__ seg_off, int n_seg,
               const __grid_constant__ Program pg, const CxTables cx) {
  const int n_ops = (int)pg.n_ops;
  const u32* prog = pg.ops;
  const int64_t total = seg_off[n_seg];
  const int64_t pairs = total >> 1;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  ulonglong2* keys2 = reinterpret_cast<ulonglong2*>(keys);
  double2* lam2 = reinterpret_cast<double2*>(lam);
  for (int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x; p < pairs; p += stride) {
    ulonglong2 k = __ldcs(keys2 + p);
    K ka = (K)k.x, kb = (K)k.y;
    u32 na = 0, nb = 0;
    for (int i = 0; i < n_ops; ++i) {
      const u32 op = prog[i];
      apply_op<K>(op, ka, na, cx);
      apply_op<K>(op, kb, nb, cx);
    }
    __stcs(keys2 + p, make_ulonglong2((u64)ka, (u64)kb));
    if (na | nb) {                       // sign flips are exact: only touch lambda when needed
      double2 l = lam2[p];
      if (na) l.x = -l.x;
      if (nb) l.y = -l.y;
      lam2[p] = l;
    }
  }
  if ((total & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t i = total - 1;
    K k = (K)keys[i];
    u32 neg = 0;
    for (int j = 0; j < n_ops; ++j) apply_op<K>(prog[j], k, neg, cx);
    keys[i] = (u64)k;
    if (neg) lam[i] = -lam[i];
  }
}

}  // namespace

extern "C" int qx_apply_clifford(qx_store* s, const uint32_t* program, int32_t n_ops, uint32_t cx_c,
                                 uint32_t cx_t, uint32_t cx_s) {
  QX_REQUIRE(s != nullptr, "store is NULL");
  QX_REQUIRE(n_ops >= 0, "negative op count");
  if (n_ops == 0) return QX_OK;
  QX_REQUIRE(program != nullptr, "program is NULL");
  const u32 max_shift = 2u * (u32)(s->n_qubits - 1);
  for (int i = 0; i < n_ops; ++i) {
    const u32 op = program[i], kind = op & 3u, s0 = (op >> 2) & 63u, s1 = (op >> 8) & 63u;
    QX_REQUIRE(kind <= 1u, "op %d: unknown kind %u", i, kind);
    QX_REQUIRE(s0 <= max_shift && (s0 & 1u) == 0, "op %d: wire out of range for n=%d", i, s->n_qubits);
    if (kind == 1u) {
      QX_REQUIRE(s1 <= max_shift && (s1 & 1u) == 0, "op %d: wire out of range for n=%d", i, s->n_qubits);
      QX_REQUIRE(s0 != s1, "op %d: control and target must differ", i);
    }
  }
  QX_CUDA(cudaSetDevice(s->device));
  const int64_t ub = std::max<int64_t>(s->ub_total, 1);
  const int64_t want = (ub / 2 + kThreads - 1) / kThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)s->sm_count * 8));
  const CxTables cx = {cx_c, cx_t, cx_s};
  static Program pg;       // host staging; the launch copies it into the parameter buffer
  for (int done = 0; done < n_ops; done += kProgChunk) {
    const int chunk = std::min(kProgChunk, n_ops - done);
    pg.n_ops = (u32)chunk;
    memcpy(pg.ops, program + done, sizeof(u32) * (size_t)chunk);
    QxProfileScope prof(QX_K_CLIFFORD, s->stream, 32.0 * (double)s->ub_total);
    if (s->n_qubits <= 16)
      k_clifford_run<u32><<<grid, kThreads, 0, s->stream>>>(s->keys[s->cur], s->lam[s->cur], s->seg[s->cur],
                                                            s->n_seg, pg, cx);
    else
      k_clifford_run<u64><<<grid, kThreads, 0, s->stream>>>(s->keys[s->cur], s->lam[s->cur], s->seg[s->cur],
                                                            s->n_seg, pg, cx);
    QX_CUDA(cudaGetLastError());
  }
  return QX_OK;
}
