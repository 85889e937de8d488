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
#include <stdlib.h>
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

// ---------------------------------------------------------------------------------------
// bit-sliced variant for runs of three or more gates
// ---------------------------------------------------------------------------------------
// Each thread takes 32 terms, transposes their words into bit planes (plane p = bit p of all
// 32 words, one 32-bit register per plane) and runs the gate program on whole planes: a CX is
// four plane loads, eight logic ops and three plane stores for 32 terms at once, instead of
// ~14 instructions per term.  The planes live in shared memory ([plane][thread], conflict
// free) because the program addresses them by run-time index.  Cost per term: ~30
// instructions for the two transposes plus ~0.6 per gate -- the per-term kernel above needs
// ~14 per gate and was ALU-bound at 1.9 TB/s on the 15-CX ladders of the ansatz circuits.
constexpr int kSlicedThreads = 128;

// main-diagonal transpose of a 32x32 bit matrix held in 32 registers (an involution)
__device__ __forceinline__ void transpose32(u32 (&a)[32]) {
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int j = 16 >> s;
    const u32 m = s == 0 ? 0x0000FFFFu : s == 1 ? 0x00FF00FFu : s == 2 ? 0x0F0F0F0Fu
                : s == 3 ? 0x33333333u : 0x55555555u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if ((k & j) == 0) {
        const u32 t = ((a[k] >> j) ^ a[k + j]) & m;
        a[k + j] ^= t;
        a[k] ^= t << j;
      }
    }
  }
}

template <int NW>      // 32-bit words per key: 1 for n <= 16, 2 otherwise
__global__ void __launch_bounds__(kSlicedThreads)
k_clifford_sliced(u64* __restrict__ keys, double* __restrict__ lam,
                  const int64_t* __restrict__ seg_off, int n_seg,
                  const __grid_constant__ Program pg, const CxTables cx) {
  extern __shared__ u32 planes[];                       // [32 * NW][kSlicedThreads]
  const int tid = threadIdx.x, lane = tid & 31;
  u32* mine = planes + tid;
  auto P = [&](u32 bit) -> u32& { return mine[bit * kSlicedThreads]; };
  const int64_t total = seg_off[n_seg];
  const int64_t chunks = (total + 1023) >> 10;          // 1024 terms per warp per round
  const int warps = kSlicedThreads / 32;
  for (int64_t c = (int64_t)blockIdx.x * warps + (tid >> 5); c < chunks; c += (int64_t)gridDim.x * warps) {
    const int64_t base = (c << 10) + lane;              // term i of this thread = base + 32 * i
    // L2 prefetch (no registers held): this chunk's coefficients, touched only at the end of the
    // round, and the keys of the chunk this warp takes next.  The kernel is latency-bound at 128
    // registers per thread (profiles/r01h: issue 17 %, long-scoreboard stalls 18 warps per issue);
    // both dependent round trips of a round now end in L2 instead of HBM.
#ifndef QX_EXP_NO_CLPF
    {
      const int64_t cn = c + (int64_t)gridDim.x * warps;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t t = (c << 10) + h * 512 + lane * 16;           // one 128-byte line per lane
        if (t < total) asm volatile("prefetch.global.L2 [%0];" ::"l"(lam + t));
        const int64_t tn = (cn << 10) + h * 512 + lane * 16;
        if (tn < total) asm volatile("prefetch.global.L2 [%0];" ::"l"(keys + tn));
      }
    }
#endif
    u32 row[32];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int64_t t = base + 32 * i;
        const u64 k = t < total ? keys[t] : 0ull;
        row[i] = w == 0 ? (u32)k : (u32)(k >> 32);
      }
      transpose32(row);
#pragma unroll
      for (int b = 0; b < 32; ++b) P(32 * w + b) = row[b];
    }
    u32 neg = 0;                                        // bit i: term i changes sign
    for (u32 g = 0; g < pg.n_ops; ++g) {
      const u32 op = pg.ops[g];
      const u32 s0 = (op >> 2) & 63u;
      if ((op & 3u) == 0u) {
        // signed axis permutation: new code bits and sign as functions of the old (hi, lo)
        const u32 hi = P(s0 + 1), lo = P(s0);
        const u32 is_x = ~hi & lo, is_y = hi & ~lo, is_z = hi & lo;
        const u32 tab = op >> 16;
        const u32 ix = (tab >> 2) & 3u, iy = (tab >> 4) & 3u, iz = (tab >> 6) & 3u;
        P(s0 + 1) = (is_x & (0u - (ix >> 1))) | (is_y & (0u - (iy >> 1))) | (is_z & (0u - (iz >> 1)));
        P(s0) = (is_x & (0u - (ix & 1u))) | (is_y & (0u - (iy & 1u))) | (is_z & (0u - (iz & 1u)));
        neg ^= (is_x & (0u - ((tab >> 9) & 1u))) | (is_y & (0u - ((tab >> 10) & 1u))) |
               (is_z & (0u - ((tab >> 11) & 1u)));
      } else {
        // CX on code bits (hi = z, lo = x ^ z): z_c ^= z_t, x_t ^= x_c,
        // sign flips iff x_c & z_t & ~(x_t ^ z_c) on the inputs
        const u32 s1 = (op >> 8) & 63u;
        const u32 hc = P(s0 + 1), lc = P(s0), ht = P(s1 + 1), lt = P(s1);
        neg ^= (hc ^ lc) & ht & ~(ht ^ lt ^ hc);
        P(s0 + 1) = hc ^ ht;
        P(s0) = lc ^ ht;
        P(s1) = lt ^ hc ^ lc;
      }
    }
    u64 out[32];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int b = 0; b < 32; ++b) row[b] = P(32 * w + b);
      transpose32(row);
#pragma unroll
      for (int i = 0; i < 32; ++i) out[i] = w == 0 ? (u64)row[i] : (out[i] | ((u64)row[i] << 32));
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int64_t t = base + 32 * i;
      if (t < total) {
        keys[t] = out[i];
        if ((neg >> i) & 1u) lam[t] = -lam[t];          // sign flips are exact
      }
    }
  }
}

}  // namespace

void qx_standard_cx(u32* cx_c, u32* cx_t, u32* cx_s) {
  u32 std_c = 0, std_t = 0, std_s = 0;
  for (u32 dc = 0; dc < 4; ++dc)
    for (u32 dt = 0; dt < 4; ++dt) {
      const u32 hc = dc >> 1, lc = dc & 1, ht = dt >> 1, lt = dt & 1, e = dc * 4 + dt;
      std_c |= ((((hc ^ ht) << 1) | (lc ^ ht)) << (2 * e));
      std_t |= (((ht << 1) | (lt ^ hc ^ lc)) << (2 * e));
      std_s |= (((hc ^ lc) & ht & (1u ^ ht ^ lt ^ hc)) << e);
    }
  *cx_c = std_c;
  *cx_t = std_t;
  *cx_s = std_s;
}

int qx_check_program(const qx_store* s, const uint32_t* program, int32_t n_ops) {
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
  return QX_OK;
}

extern "C" int qx_apply_clifford(qx_store* s, const uint32_t* program, int32_t n_ops, uint32_t cx_c,
                                 uint32_t cx_t, uint32_t cx_s) {
  QX_TRY(qx_check_program(s, program, n_ops));
  QX_NARROW_ONLY(s, "qx_apply_clifford");
  if (n_ops == 0) return QX_OK;
  QX_CUDA(cudaSetDevice(s->device));
  const int64_t ub = std::max<int64_t>(s->ub_total, 1);
  const int64_t want = (ub / 2 + kThreads - 1) / kThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)s->sm_count * 8));
  const CxTables cx = {cx_c, cx_t, cx_s};
  static Program pg;       // host staging; the launch copies it into the parameter buffer
  // the sliced kernel evaluates CX from the x/z rule, which equals the reference's tables
  // (lut.py:108-134); a caller passing other tables (mutation tests) gets the table-driven kernel
  u32 std_c, std_t, std_s;
  qx_standard_cx(&std_c, &std_t, &std_s);
  static const bool per_term_only = getenv("QX_CLIFFORD_PER_TERM") != nullptr;
  const bool no_slice = per_term_only || cx_c != std_c || cx_t != std_t || cx_s != std_s;
  for (int done = 0; done < n_ops; done += kProgChunk) {
    const int chunk = std::min(kProgChunk, n_ops - done);
    pg.n_ops = (u32)chunk;
    memcpy(pg.ops, program + done, sizeof(u32) * (size_t)chunk);
    QxProfileScope prof(QX_K_CLIFFORD, s->stream, 32.0 * (double)s->ub_total);
    if (chunk >= 3 && !no_slice) {
      const int64_t chunks = (ub + 1023) / 1024;
      const int sgrid = (int)std::max<int64_t>(1, std::min<int64_t>((chunks + 3) / 4, (int64_t)s->sm_count * 8));
      if (s->n_qubits <= 16) {
        k_clifford_sliced<1><<<sgrid, kSlicedThreads, 32 * kSlicedThreads * 4, s->stream>>>(
            s->keys[s->cur], s->lam[s->cur], s->seg[s->cur], s->n_seg, pg, cx);
      } else {
        static bool attr = false;
        if (!attr) {
          QX_CUDA(cudaFuncSetAttribute(k_clifford_sliced<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       64 * kSlicedThreads * 4));
          attr = true;
        }
        k_clifford_sliced<2><<<sgrid, kSlicedThreads, 64 * kSlicedThreads * 4, s->stream>>>(
            s->keys[s->cur], s->lam[s->cur], s->seg[s->cur], s->n_seg, pg, cx);
      }
      QX_CUDA(cudaGetLastError());
      continue;
    }
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
