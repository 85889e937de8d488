/*
 * qimax_b200.h -- C ABI of the B200 extended-stabilizer hot path (libqimax_b200.so).
 *
 * The reference (stabsim, pure Python/numpy) has no FFI; its boundary is the
 * public Python API.  Each entry point below names the reference function it
 * replaces (paths under /root/reference/pkg/src/stabsim/).  INTEGRATION.md shows
 * the ctypes binding a reference maintainer would add.
 *
 * Conventions
 *   - plain pointers and sizes only; every pointer is HOST memory unless the
 *     parameter name starts with d_ (then it is a device pointer on the store's device);
 *   - every call returns a qx_status; on failure qx_last_error() (thread-local)
 *     holds a message.  Python maps INVALID -> ValueError, RESOURCE ->
 *     ResourceLimitError, CONSISTENCY -> ConsistencyError, CUDA/UNSUPPORTED -> NativeError;
 *   - the caller owns handles; no pointer passed in is retained after return;
 *   - a handle is not thread-safe; distinct handles may be used from distinct threads.
 *
 * Term layout (both host side and in HBM): structure of arrays.
 *   key    uint64  base-4 Pauli word, 2 bits per qubit, qubit 0 most significant,
 *                  axis codes I=0 X=1 Y=2 Z=3 (reference pauli.py:24-30,67-86).  With
 *                  code bits (hi,lo): z = hi, x = hi ^ lo, so this *is* the packed
 *                  2-bit x/z form, ordered so that unsigned integer order equals the
 *                  reference's canonical order.  n_qubits <= 32 (one word); wider systems use
 *                  several words per key on a restricted path, see "more than 32 qubits" below.
 *   lambda float64 real coefficient (reference stabilizer.py:92).
 * A store holds n_segments generators back to back; offsets[s]..offsets[s+1] is
 * generator s.  16 bytes per term.
 */
#ifndef QIMAX_B200_H
#define QIMAX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QX_ABI_VERSION 1

typedef enum {
  QX_OK = 0,
  QX_ERR_INVALID = 1,      /* bad argument (reference raises ValueError) */
  QX_ERR_RESOURCE = 2,     /* a cap / budget / HBM limit would be exceeded (ResourceLimitError) */
  QX_ERR_CUDA = 3,         /* CUDA runtime failure or no usable device */
  QX_ERR_UNSUPPORTED = 4,  /* e.g. n_qubits > 32 */
  QX_ERR_CONSISTENCY = 5   /* internal invariant failed (ConsistencyError) */
} qx_status;

typedef struct qx_store qx_store;          /* term store: a1 */
typedef struct qx_expansion qx_expansion;  /* density-expansion accumulator: a9 */

/* ---- library ------------------------------------------------------------ */
int qx_abi_version(void);
const char* qx_last_error(void);
int qx_device_count(int* count);
int qx_device_info(int device, char* name, int name_cap, int* sm_count, int* cc_major,
                   int* cc_minor, int64_t* total_bytes, int64_t* free_bytes);

/* Page-locked host buffers so uploads/downloads run at full PCIe rate (optional). */
int qx_host_alloc(int64_t bytes, void** out);
int qx_host_free(void* ptr);
/* Return the library's cached (freed but retained) device blocks to the driver. */
int qx_trim(void);

/* ---- a1: term store (stabilizer.py:83-109 SimpleGenerator, :157-174 GeneratorSet/init_z) */
int qx_store_create(int device, int n_qubits, int n_segments, int64_t capacity_terms,
                    qx_store** out);
int qx_store_destroy(qx_store* s);
/* Launch on this CUDA stream (a cudaStream_t) instead of the legacy default stream. */
int qx_store_set_stream(qx_store* s, void* cuda_stream);
/* Segment i := 1.0 * Z on qubit qubits[i] (init_z, stabilizer.py:169-174); NULL = qubit i. */
int qx_store_init_z(qx_store* s, const int32_t* qubits);
/* Replace the whole content: offsets has n_segments+1 entries, offsets[0] == 0. */
int qx_store_upload(qx_store* s, const int64_t* offsets, const uint64_t* keys,
                    const double* lambdas);
/* Current term count per segment (synchronises). */
int qx_store_ranks(qx_store* s, int64_t* ranks);
/* Copy everything out: offsets (n_segments+1), then up to cap_terms keys/lambdas. */
int qx_store_download(qx_store* s, int64_t* offsets, uint64_t* keys, double* lambdas,
                      int64_t cap_terms);
/* Device views for zero-copy consumers (valid until the next mutating call). */
int qx_store_device_view(qx_store* s, const uint64_t** d_keys, const double** d_lambdas,
                         const int64_t** d_offsets);
int qx_store_capacity(qx_store* s, int64_t* capacity_terms, int64_t* hbm_bytes);
int qx_store_synchronize(qx_store* s);
/* Phase timers on the device (the reference's RunReport.timings keys partition / lut /
 * sub_flatten / cx, engine.py:92: the two device phases are measured with CUDA events on the
 * store's stream instead of a host clock around asynchronous launches).  record: a new event on
 * the stream, its index in *index.  elapsed: waits for event `second`, milliseconds between the
 * two.  Events live as long as the store. */
int qx_store_event_record(qx_store* s, int32_t* index);
int qx_store_event_elapsed(qx_store* s, int32_t first, int32_t second, double* ms);
/* Generators evolve independently (engine.py:113-116): a new store holding copies of segments
 * [seg_lo, seg_hi) of src (device-to-device), launching on a non-blocking stream of its own so
 * that its kernels and copies overlap those of other stores.  src is left untouched. */
int qx_store_slice(qx_store* src, int32_t seg_lo, int32_t seg_hi, int64_t capacity_terms,
                   qx_store** out);
/* qx_store_download without the final wait: offsets are returned at once (they are exact on
 * the host after any merge), the term copies are queued on the store's stream into keys /
 * lambdas, which should be page-locked (qx_host_alloc) and must stay valid until
 * qx_store_synchronize(s). */
int qx_store_download_async(qx_store* s, int64_t* offsets, uint64_t* keys, double* lambdas,
                            int64_t cap_terms);
/* For a store that is only downloaded next (n <= 16): on != 0 lets the next large operator step
 * leave 32-bit keys in HBM, so that 12 instead of 16 bytes per term cross PCIe.  Afterwards only
 * qx_store_download_narrow_async, qx_store_ranks, qx_store_synchronize and qx_store_destroy are
 * valid on the store. */
int qx_store_set_keep_narrow(qx_store* s, int on);
/* As qx_store_download_async for such a store: the 32-bit keys are copied into `staging`
 * (page-locked, cap_terms words) chunk by chunk and `threads` host threads widen every chunk into
 * `keys` as soon as it has landed, while later chunks and the coefficients are still on the wire.
 * qx_store_synchronize(s) waits for the copies AND the widening.  Falls back to
 * qx_store_download_async if the store holds 64-bit keys. */
int qx_store_download_narrow_async(qx_store* s, int64_t* offsets, uint64_t* keys, double* lambdas,
                                   int64_t cap_terms, uint32_t* staging, int32_t threads);
/* qx_store_set_keep_narrow(s, 2) additionally allows the PACKED form for large results: the last
 * sort pass writes only the low 16 bits of every key plus, per generator, a table of 65537 words
 * first[h] = position of the first key whose high half is >= h (keys are sorted, so the high
 * halves are the bucket index).  10 bytes per term cross PCIe.  This call downloads whichever
 * form the store holds (packed, 32-bit, 64-bit): `staging` (page-locked, staging_words 32-bit
 * words; cap_terms + 65537 * n_segments + 2 always suffices) receives the tables and the halves,
 * `threads` host threads rebuild the 64-bit keys bucket by bucket while the rest is on the wire.
 * *d2h_bytes (may be NULL) = bytes copied device -> host. */
int qx_store_download_packed_async(qx_store* s, int64_t* offsets, uint64_t* keys, double* lambdas,
                                   int64_t cap_terms, uint32_t* staging, int64_t staging_words,
                                   int32_t threads, int64_t* d2h_bytes);

/* ---- more than 32 qubits (reference stabilizer.py:40-59 switches to Python
 * big-int indices there).  qx_store_create accepts n_qubits <= 512; above 32 the store is WIDE:
 * W = ceil(2n/64) words per key.  Wide stores run the part of the path that such circuits use --
 * Clifford runs, v1 rotations (and with them branching v2/v3 operators, applied gate by gate),
 * merge/sort of generators of any size, ranks, norms --
 * through the calls below plus qx_store_init_z / qx_merge / qx_sort / qx_store_ranks /
 * qx_store_norms; every other entry point returns QX_ERR_UNSUPPORTED on a wide store.
 * Host layout of wide keys: term-major uint64[term][W], word 0 least significant. */
int qx_store_words(qx_store* s, int32_t* n_words);
int qx_store_upload_wide(qx_store* s, const int64_t* offsets, const uint64_t* words,
                         const double* lambdas);
int qx_store_download_wide(qx_store* s, int64_t* offsets, uint64_t* words, double* lambdas,
                           int64_t cap_terms);
/* The grouped operator step above 32 qubits (the reference's big-int path,
 * stabilizer.py:40-59, 289-322).  qx_store_support: per segment, OR of the support masks of its
 * terms -- n_segments x n_words words (bit 2p set: some term has a non-identity digit at bit
 * position 2p; works on one-word stores too).  qx_store_compact: the terms of the segments with
 * take[g] != 0 as one-word keys over the n_sel selected qubits (ascending; every taken term's
 * support must lie inside them) into `narrow`, a one-word store of n_sel qubits and as many
 * segments (the segments not taken are empty there); the order of the terms is kept, and so is
 * canonical order.  qx_store_expand: the inverse -- the taken segments of the multi-word store are
 * REPLACED by the one-word store's segments spread back over the selected qubits, the others keep
 * their terms.  Between the two the caller runs the one-word operator step
 * (qx_apply_operator_run) with the selected rows of the operator tables; identity digits
 * contribute a factor of exactly 1, so the result is what the reference computes at full width,
 * bit for bit. */
int qx_store_support(qx_store* s, uint64_t* words);
int qx_store_compact(qx_store* wide, const int32_t* qubits, int32_t n_sel, const uint8_t* take,
                     qx_store* narrow);
int qx_store_expand(qx_store* narrow, const int32_t* qubits, int32_t n_sel, const uint8_t* take,
                    qx_store* wide);

/* As qx_apply_clifford with 64-bit ops: low word as there (kind, image axes, signs; the shift
 * fields unused), bits 32-47 = bit position 2*(n-1-q) of the (control) digit, 48-63 of the target. */
int qx_apply_clifford_wide(qx_store* s, const uint64_t* ops, int32_t n_ops, uint32_t cx_c,
                           uint32_t cx_t, uint32_t cx_s);
/* As qx_apply_split; every term yields two entries (an absent second branch becomes a zero-weight
 * copy of the first), so the store doubles; qx_merge follows. */
int qx_apply_split_wide(qx_store* s, int32_t qubit, const int32_t a1[4], const double w1[4],
                        const int32_t a2[4], const double w2[4]);

/* ---- a2 + Clifford part of a3: fused run of sign-permutation gates ----------
 * Replaces apply_cx (stabilizer.py:340-363) and _apply_1q_terms (engine.py:183-218)
 * for H/S/X/SX and any composed U_k block that is a signed axis permutation.
 * One launch pushes every term through the whole program in registers; conjugation
 * by a Clifford is a bijection on words, so no merge is needed afterwards.
 * op word: bits 0-1 kind (0 = 1q permutation, 1 = CX); bits 2-7 shift of the
 * (control) digit = 2*(n-1-q); bits 8-13 shift of the CX target digit; for kind 0
 * bits 16-23 = image axis of input axis a at bits 16+2a, bits 24-27 = sign bit of axis a.
 * cx_c/cx_t: 2 bits per [control*4+target] entry; cx_s: 1 bit per entry
 * (LUT_C/LUT_T/LUT_SIGN, lut.py:108-134). */
int qx_apply_clifford(qx_store* s, const uint32_t* program, int32_t n_ops, uint32_t cx_c,
                      uint32_t cx_t, uint32_t cx_s);

/* ---- non-Clifford part of a3: split each term on one qubit (engine.py:190-217).
 * For input digit d: first branch (a1[d], w1[d]) always, second branch (a2[d], w2[d])
 * iff w2[d] != 0.  Output per segment is term-major: each term's first branch, then its
 * second branch if it has one (slots from a warp-ballot prefix sum + tile look-back).
 * A key only ever receives first branches or only second branches, so duplicates keep
 * the relative order of the reference's [firsts..., seconds...] list and the merge sums
 * them in the same order.  Unmerged; call qx_merge next. */
int qx_apply_split(qx_store* s, int32_t qubit, const int32_t a1[4], const double w1[4],
                   const int32_t a2[4], const double w2[4]);

/* ---- a4 + a5: substitute-and-flatten of one U_k (stabilizer.py:189-206, 289-322).
 * counts[j*3+p-1] = number of nonzero weights of input axis p on qubit j (1..3),
 * axes/weights[(j*3+p-1)*3+b] = b-th (axis, weight), ascending axis.  Every term
 * expands into the Cartesian product over its non-identity digits, branches in C
 * order with qubit 0 slowest, lambda * w_q0 * w_q1 * ... left to right.
 * Unmerged; raw_total receives the raw term count.  term_limit > 0 refuses
 * (QX_ERR_RESOURCE) a raw count above it before anything is written. */
int qx_apply_operator(qx_store* s, const int32_t* counts, const int32_t* axes,
                      const double* weights, int64_t term_limit, int64_t* raw_total);
/* ---- a4 + a5 + a2 + a6 in one call: U_k, the run of sign-permutation ops that follows it
 * (the CX group V_k and any Clifford blocks up to the next branching operator), then the merge
 * (engine.py:110-132: sub, flatten, apply_cx..., canonicalize).  Same result as
 * qx_apply_operator + qx_apply_clifford + qx_merge, but conjugation by the run is folded into the
 * expansion kernel (a Clifford run is a homomorphism: the image of a raw term is the product of
 * the images of its single-digit factors), so raw terms are written once, already conjugated,
 * and for 2n <= 32 as 32-bit keys that only the sort passes see.  program/n_ops/cx_*: as in
 * qx_apply_clifford (n_ops may be 0).  ranks (may be NULL): per-segment counts after the merge.
 * Operators with a large fan-out take the grouped dense path (csrc/dense.cu: sources grouped by
 * class word, one thread per output slot, sort only); raw_total then reports the slot count, an
 * upper bound of the merged size like the raw count. */
int qx_apply_operator_run(qx_store* s, const int32_t* counts, const int32_t* axes,
                          const double* weights, const uint32_t* program, int32_t n_ops,
                          uint32_t cx_c, uint32_t cx_t, uint32_t cx_s, double eps,
                          int64_t term_limit, int64_t* raw_total, int64_t* ranks);
/* Multi-GPU form of qx_apply_operator_run for the LAST branching operator of a circuit: every
 * device holds the same input terms and works off the part-th of `parts` contiguous ranges of
 * output slots (slots are independent: no communication).  *partitioned = 1: the store now holds
 * this part's share of every generator (canonical order, disjoint from the other parts' shares;
 * ranks are the share's counts -- sum them over the parts); 0: the operator did not take the
 * grouped path (few sources' worth of fan-out, eps == 0, ...) and the store holds the complete
 * result, identical on every device. */
int qx_apply_operator_run_part(qx_store* s, const int32_t* counts, const int32_t* axes,
                               const double* weights, const uint32_t* program, int32_t n_ops,
                               uint32_t cx_c, uint32_t cx_t, uint32_t cx_s, double eps,
                               int32_t part, int32_t parts, int64_t* ranks, int32_t* partitioned);
/* Host-only (no GPU work): the class decomposition qx_apply_operator_run uses for operators with
 * a large fan-out.  Per qubit, input axes that share an output axis (stabilizer.py:209-214: the
 * nonzero cells of a substituted row) form a class; terms whose words agree after every digit is
 * replaced by its class can collide in the merge, all others cannot.  Inputs as in
 * qx_apply_operator; outputs indexed [qubit*3 + axis-1]: class_id = smallest input axis of the
 * class (1..3), class_radix = number of output axes of the class; class_axes / class_weights
 * (may be NULL) [..*3 + b]: the class's output axes, ascending, and this input axis' weight on
 * each (0.0 where it does not reach that axis). */
int qx_operator_classes(int32_t n_qubits, const int32_t* counts, const int32_t* axes,
                        const double* weights, int32_t* class_id, int32_t* class_radix,
                        int32_t* class_axes, double* class_weights);
/* Host-only: what the last bucketed operator step of this process did (csrc/bucket.cuh: the
 * operator step of stabilizer.py:289-337 whose slots leave the kernel in canonical order, so that
 * canonicalize's sort disappears).  out[0..7] = groups, tiles, buckets, slots of the largest
 * bucket, slots, low key bits ranked inside a bucket, bucket capacity (0: the step did not
 * qualify and the grouped step + sort ran), CTAs per SM. */
int qx_bucket_last(int64_t out[8]);
/* Host-only: what the last grouped operator step of this process did (csrc/dense.cu).  out[0] =
 * groups (-1: the group list was not brought to the host), out[1] = groups whose sums were formed
 * mode by mode ahead of the slot kernel (k_group_kron: many sources on at most 8 digits),
 * out[2] = slots of those groups, out[3] = their sources. */
int qx_dense_last(int64_t out[4]);
/* Host-only: switch the bucketed step on or off for this process (tests and A/B runs compare it
 * with the grouped step + sort; results are bit-identical).  Returns the previous setting (1/0).
 * QX_NO_BUCKET in the environment starts the process with it off. */
int qx_bucket_enable(int32_t on);
/* Number of raw branches the same call would produce per segment, nothing written
 * (branch_counts, stabilizer.py:232-237). */
int qx_count_operator(qx_store* s, const int32_t* counts, int64_t* raw_per_segment);
/* Put the terms of every segment into the order in which the reference's ragged flatten walks
 * its strings (_flatten_ragged, stabilizer.py:294-296): strings grouped by their per-qubit branch
 * counts (count vectors ascending lexicographically, qubit 0 first), inside a group by word
 * (by_key = 1: the canonical order of engine.run's generators, whatever permutation the store
 * is in) or by input position (by_key = 0: the stable order of the kernel-level flatten).  Sums
 * of three or more contributions to one word are then added in the reference's order, so a
 * following qx_apply_operator(_run) + merge gives its coefficients bit for bit.  Segments of
 * more than 2048 terms are left as they are (large groups are summed in factored form anyway).
 * Asynchronous; nothing is read back. */
int qx_store_order_for_operator(qx_store* s, const int32_t* counts, int32_t by_key);

/* ---- a7 on the device: the reference's sequential chain (engine.py:110-132 for
 * v2/v3, :155-180 for v1) compiled into a device-resident step list and walked by ONE launch, one
 * CTA per generator, terms in shared memory from the first step to the last (csrc/program.cuh).
 * Steps (kinds[i]): 0 = a run of sign-permutation ops (apply_cx / fixed 1q gates,
 * stabilizer.py:340-363), 1 = a branching operator U_k + the run behind it + the merge (what
 * qx_apply_operator_run does: stabilizer.py:189-206, 289-337), with order[i] != 0 preceded by the
 * reference's string order (qx_store_order_for_operator with by_key = 1, stabilizer.py:294-296),
 * 2 = canonical order (what canonicalize amounts to after permutation steps).  ops[ops_off[i] ..
 * ops_off[i+1]) are step i's op words (as in qx_apply_clifford; standard CX tables);
 * counts/axes/weights hold n_steps operator tables of the qx_apply_operator layout back to back
 * (read for kind 1 only; may be NULL if there is none).  The program owns device memory on
 * `device` until qx_program_destroy. */
typedef struct qx_program qx_program;
int qx_program_create(int device, int32_t n_qubits, int32_t n_steps, const int32_t* kinds,
                      const int32_t* order, const int32_t* counts, const int32_t* axes,
                      const double* weights, const uint32_t* ops, const int64_t* ops_off,
                      qx_program** out);
int qx_program_destroy(qx_program* p);
/* Number of kind-1 steps = rows of the ranks table qx_store_run_program fills. */
int qx_program_rows(const qx_program* p, int32_t* rows);
/* Run the program on every generator of the store.  *fitted = 1: the store holds the result and
 * ranks[row * n_segments + g] = terms of generator g after the row-th kind-1 step (0 = all its
 * terms were dropped there -- the caller raises the reference's NumericalCollapseError,
 * engine.py:148-152 -- and its later rows stay 0); raw_total (may be NULL) = raw branches of all
 * kind-1 steps; offsets (may be NULL) = n_segments + 1 offsets of the result.  *fitted = 0: some
 * generator outgrew shared memory (more than 4096 terms between steps or 8192 raw branches in one
 * step); the store is exactly as before the call and the caller replays the steps one by one.
 * init_qubits != NULL (n_segments <= 32): the store's content is ignored and generator g starts as
 * Z on qubit init_qubits[g] -- what qx_store_init_z would have uploaded (init_z,
 * stabilizer.py:169-174; if the program then does not fit, the store is left as qx_store_init_z
 * leaves it).  host_keys / host_lambdas != NULL (PAGE-LOCKED memory from qx_host_alloc, room for
 * host_cap terms): the kernel also writes the result there, store layout; *host_filled = 1 if all
 * of it fit.  device_ms (may be NULL): duration of the launch on the GPU's own clock (first CTA in
 * to last CTA out, %globaltimer) -- the device phase timer of the run at no cost.  One launch and
 * one stream synchronize: ranks, offsets and the host copy of the result are written by the
 * kernel itself into page-locked memory.  max_steps > 0: only the first max_steps steps (a circuit
 * whose generators outgrow shared memory later starts with one launch and goes on step by step);
 * *stopped_step (may be NULL), when *fitted = 0: the first step that did not fit. */
int qx_store_run_program(qx_store* s, const qx_program* p, const int32_t* init_qubits, double eps,
                         int64_t* ranks, int64_t* raw_total, int32_t* fitted, int64_t* offsets,
                         uint64_t* host_keys, double* host_lambdas, int64_t host_cap,
                         int32_t* host_filled, double* device_ms, int32_t max_steps,
                         int32_t* stopped_step);

/* ---- a6: duplicate-term merge (canonicalize, stabilizer.py:325-337).
 * Per segment: stable sort by key, in-order segmented sum, keep |sum| >= eps,
 * ascending.  ranks (may be NULL) receives the new per-segment counts. */
int qx_merge(qx_store* s, double eps, int64_t* ranks);
/* Canonical order only: stable sort of every segment by key, nothing summed or dropped.
 * What canonicalize amounts to after Clifford gates (a bijection on words that keeps
 * |lambda|): term counts are unchanged, so nothing is read back.  Precondition: keys are
 * unique inside each segment (with duplicates, use qx_merge). */
int qx_sort(qx_store* s);

/* ---- north-star kernel (4): per segment, sum of lambda over Z/I-only words (any key width:
 * one-word stores and the multi-word stores above 32 qubits). */
int qx_store_zi_sums(qx_store* s, double* sums);
/* Per segment sum of lambda^2 (the P^2 = I self-check). */
int qx_store_norms(qx_store* s, double* sum_sq);

/* ---- a9/a10: density expansion 2^-n prod_j (I + P_j) (measure.py:40-91) ---- */
int qx_expansion_create(int device, int n_qubits, int64_t capacity_terms, qx_expansion** out);
int qx_expansion_destroy(qx_expansion* e);
int qx_expansion_reset(qx_expansion* e); /* acc := { I^n : 1 } */
/* acc := merge(acc U acc*g) for one generator given as host arrays; refuses with
 * QX_ERR_RESOURCE when |acc| * (1 + count) > term_budget (measure.py:59-62). */
int qx_expansion_multiply(qx_expansion* e, const uint64_t* keys, const double* lambdas,
                          int64_t count, int64_t term_budget);
/* Same with the generator read from a store segment already in HBM. */
int qx_expansion_multiply_segment(qx_expansion* e, qx_store* s, int32_t segment,
                                  int64_t term_budget);
int qx_expansion_size(qx_expansion* e, int64_t* terms);
int qx_expansion_max_abs_imag(qx_expansion* e, double* worst);
int qx_expansion_download(qx_expansion* e, uint64_t* keys, double* re, double* im,
                          int64_t cap_terms);
/* Unscaled real coefficient of each word (0 if absent): coeffs.get (measure.py:35-37). */
int qx_expansion_lookup(qx_expansion* e, const uint64_t* words, int64_t n_words, double* re);

/* ---- term hash-partition for multi-GPU rebalancing ----------
 * Reorders every segment so that terms owned by rank r = mix(key) % world are
 * contiguous, rank-major; send_counts[r * n_segments + s] = terms of segment s owned by r.
 * After the call the store is laid out [rank0: seg0..segS-1][rank1: ...]. */
int qx_store_partition_by_owner(qx_store* s, int32_t world, int64_t* send_counts);
/* Inverse side of the exchange: d_keys/d_lambdas (DEVICE pointers) hold what this rank
 * received, laid out [source 0: seg0..segS-1][source 1: ...] with
 * recv_counts[q * n_segments + s] terms each; the store becomes segment-major
 * (sources in rank order inside a segment), ready for qx_merge. */
int qx_store_assemble(qx_store* s, const uint64_t* d_keys, const double* d_lambdas, int32_t world,
                      const int64_t* recv_counts);

/* ---- instrumentation: per kernel-class CUDA-event timing -------------------- */
typedef enum {
  QX_K_CLIFFORD = 0,
  QX_K_SPLIT = 1,
  QX_K_EXPAND_COUNT = 2,
  QX_K_EXPAND_EMIT = 3,
  QX_K_SORT_HIST = 4,
  QX_K_SORT_PASS = 5,
  QX_K_REDUCE = 6,
  QX_K_SMALL_MERGE = 7,
  QX_K_READOUT_PRODUCT = 8,
  QX_K_READOUT_REDUCE = 9,
  QX_K_PARTITION = 10,
  QX_K_DENSE_PREP = 11,  /* grouped operator step: class words, source sort, group scan */
  QX_K_DENSE_EMIT = 12,  /* grouped operator step: one thread per output slot */
  QX_K_BUCKET_EMIT = 13, /* bucketed operator step: slots computed, ranked and written in final order */
  QX_K_CLASSES = 14
} qx_kernel_class;
int qx_profile_enable(int on);
int qx_profile_reset(void);
/* launches, summed device milliseconds and summed algorithmic bytes of one class
 * since the last reset (synchronises the device). */
int qx_profile_read(int kernel_class, int64_t* launches, double* total_ms, double* alg_bytes);
/* Total kernel launches issued by this library since load (never reset). */
int qx_launch_count(int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* QIMAX_B200_H */
