// Shared device-side pieces of the operator kernels (branch.cu: raw expansion; dense.cu:
// grouped dense accumulation): branch tables, Clifford-image composition, two-level decode.
#pragma once

#include "qx_device.cuh"

namespace qxe {

// Indexed by digit position p = n-1-qubit (p = 0 is the least significant digit).
struct OperatorTable {
  double w[QX_MAX_QUBITS][3][3];
  unsigned char axis[QX_MAX_QUBITS][3][3];
  unsigned char cnt[QX_MAX_QUBITS][3];
};

static __device__ __forceinline__ u64 branch_count(u64 key, const unsigned char (*cnt)[3]) {
  u64 m = support_mask(key), c = 1;
  while (m) {
    const int b = __ffsll((long long)m) - 1;
    m &= m - 1;
    c *= cnt[b >> 1][((key >> b) & 3ull) - 1];
  }
  return c;
}

// index of the last entry <= r in a strictly increasing array a[0..n)
static __device__ __forceinline__ int64_t last_le(const u64* a, int64_t n, u64 r) {
  int64_t lo = 0, hi = n;                  // a[lo] <= r < a[hi] (a[n] = +inf)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// ---- working-key width ------------------------------------------------------------------
// For n <= 16 a word fits 32 bits and a term has at most 3^16 < 2^32 branches, so the whole
// enumeration runs on 32-bit registers (these kernels are ALU-bound: half the instructions).
template <typename K> struct KeyOps;
template <> struct KeyOps<u32> {
  static __device__ __forceinline__ int lowest(u32 m) { return __ffs((int)m) - 1; }
  static __device__ __forceinline__ int highest(u32 m) { return 31 - __clz((int)m); }
  static __device__ __forceinline__ u32 support(u32 k) { return (k | (k >> 1)) & 0x55555555u; }
};
template <> struct KeyOps<u64> {
  static __device__ __forceinline__ int lowest(u64 m) { return __ffsll((long long)m) - 1; }
  static __device__ __forceinline__ int highest(u64 m) { return 63 - __clzll((long long)m); }
  static __device__ __forceinline__ u64 support(u64 k) { return support_mask(k); }
};

// ---- Clifford run folded into the expansion ---------------------------------------------------
// In v2/v3 every U_k is followed by a run of sign-permutation ops (the CX group V_k, Clifford
// blocks of later U's).  Conjugation by the run is a group homomorphism on Pauli operators, so the
// image of a raw term is the ordered product of the images of its single-digit factors: the host
// pushes the 3n single-digit words through the run once (ImageTable) and the expansion kernel
// composes images instead of OR-ing digits -- the raw terms leave the kernel already conjugated
// and the separate read+write pass of the Clifford kernel disappears.
// Bookkeeping in "XZ form": a Hermitian word with sign s is i^e X^x Z^z with e = #Y + 2s, and
//   (i^ea X^xa Z^za)(i^eb X^xb Z^zb) = i^(ea + eb + 2|za & xb|) X^(xa^xb) Z^(za^zb);
// on the packed base-4 code (hi = z, lo = x ^ z) the word part is one XOR, the exponent one
// popcount.  Factors of one term act on different qubits, so they commute and the final
// exponent minus #Y of the final word is 0 or 2: the sign, applied to lambda exactly.
template <typename K>
struct ImageTable {
  K img[QX_MAX_QUBITS][3];             // image word of axis a+1 at digit position p
  K imx[QX_MAX_QUBITS][3];             // its x plane ((w ^ w >> 1) & 0x55..), precomputed
  unsigned char e[QX_MAX_QUBITS][3];   // (#Y of the image + 2 * sign) mod 4
};

template <typename K> struct Plane;
template <> struct Plane<u32> {
  static constexpr u32 lo = 0x55555555u;
  static __device__ __forceinline__ u32 popc(u32 v) { return (u32)__popc(v); }
};
template <> struct Plane<u64> {
  static constexpr u64 lo = 0x5555555555555555ull;
  static __device__ __forceinline__ u32 popc(u64 v) { return (u32)__popcll(v); }
};

template <typename K>
static __device__ __forceinline__ void compose(K& word, u32& e, K img, K imx, u32 ie) {
  e += ie + 2u * Plane<K>::popc((word >> 1) & imx);
  word ^= img;
}
// 1 iff the composed operator is MINUS the Hermitian word
template <typename K>
static __device__ __forceinline__ u32 composed_sign(K word, u32 e) {
  const u32 ny = Plane<K>::popc((word >> 1) & ~word & Plane<K>::lo);
  return ((e - ny) >> 1) & 1u;
}

// ---- two-level branch decode --------------------------------------------------------------
// A source term with non-identity digits d_0 < d_1 < ... (least significant first) and radices
// c_i expands into prod c_i raw terms, branch id b = mixed-radix number with d_0 fastest.
// Split the digits into a LOW group (d_0, d_1, d_2: L = c0*c1*c2 <= 27 branches) and the HIGH
// rest.  All L branches of one "block" h = b / L share the high digits, i.e. the partial
// product p_hi = lambda * w(top) * ... * w(d_3) and the partial word k_hi.  Per output tile:
//   1. every source that feeds the tile counts the blocks it touches (prefix sum in smem);
//   2. one thread per BLOCK decodes h and folds the high digits once into (p_hi, k_hi) in smem
//      -- the only loops over digits, amortised over up to 27 outputs;
//   3. one thread per OUTPUT (consecutive lanes = consecutive raw terms, so stores are fully
//      coalesced) splits b into (h, three low picks), reads its block's (p_hi, k_hi) and does
//      three multiplies, in the reference's order: ((p_hi * w2) * w1) * w0 with qubit 0 first.
// Control flow in step 3 is uniform across the warp: no loops, no data-dependent branches.
template <typename K>
struct LowGroup {
  int bit[3];      // digit positions (bit offsets), -1 if absent
  u32 rad[3];      // radices (1 if absent)
  u32 dig[3];      // input axis - 1 at those positions
  K hi_mask;       // support bits above the group
  u32 L;           // rad[0] * rad[1] * rad[2]
};

template <typename K>
static __device__ __forceinline__ LowGroup<K> low_group(K key, const OperatorTable& tb) {
  LowGroup<K> g;
  K m = KeyOps<K>::support(key);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    g.bit[j] = -1;
    g.rad[j] = 1;
    g.dig[j] = 0;
    if (m) {
      const int bit = KeyOps<K>::lowest(m);
      m &= m - 1;
      g.bit[j] = bit;
      g.dig[j] = (u32)((key >> bit) & 3u) - 1u;
      g.rad[j] = tb.cnt[bit >> 1][g.dig[j]];
    }
  }
  g.hi_mask = m;
  g.L = g.rad[0] * g.rad[1] * g.rad[2];
  return g;
}

// q = b / c, r = b % c for c in {1, 2, 3} without a divide
template <typename K>
static __device__ __forceinline__ void divmod_small(K b, u32 c, K& q, u32& r) {
  if (c == 1) { q = b; r = 0; }
  else if (c == 2) { q = b >> 1; r = (u32)(b & 1u); }
  else { q = b / 3u; r = (u32)(b - 3u * q); }
}

}  // namespace qxe
