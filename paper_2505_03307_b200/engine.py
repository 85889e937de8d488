"""Simulation engine: the reference's ``engine.run`` on the B200 term store.

Same entry points and report as the reference (``engine.py:45-243``): ``run``,
``run_all_modes``, ``compare_reports``, ``Mode``, ``RunReport``.  Semantics per mode
are the reference's -- where terms branch, where they are merged, which
coefficients are dropped -- but the schedule is built for the GPU:

* every gate/operator that is an exact signed axis permutation (H, S, X, SX, CX,
  and any composed U_k block with entries 0/+-1) is a bijection on Pauli words and
  keeps |lambda|, so the merge the reference runs after it can only re-sort.  Those
  are queued and executed as ONE fused launch per run of such gates
  (``qx_apply_clifford``), and the sort is deferred to the next real merge;
* a gate/operator that branches (any rotation whose matrix is not a signed
  permutation -- including angles like pi/2 whose cosine is 6e-17, exactly as the
  reference treats them) flushes the queue, runs the branching kernel
  (``qx_apply_split`` in v1, ``qx_apply_operator`` in v2/v3) and merges with the
  reference's drop rule, at the same point of the circuit as the reference;
* terms stay in HBM from ``init_z`` to the final download.

The host walks the circuit; it never touches a term.
"""

from __future__ import annotations

import time
from operator import is_ as _is
from dataclasses import dataclass, field
from enum import Enum
from typing import Sequence

import numpy as np

from . import lut as _lut
from .circuit import Instruction, divide_instruction
from .errors import ConsistencyError, NumericalCollapseError, ResourceLimitError
from .stabilizer import (
    DEFAULT_EPS,
    DENSE_FLATTEN_BUDGET,
    GeneratorSet,
    SimpleGenerator,
    keys_to_indices,
    pad_dense,
    rank_stats,
    split_tables,
)
from .store import CircuitProgram, DeviceStore


class Mode(Enum):
    V1 = "v1"
    V2 = "v2"
    V3 = "v3"

    @classmethod
    def coerce(cls, value) -> "Mode":
        if isinstance(value, Mode):
            return value
        return cls(str(value).lower())


@dataclass
class RunReport:
    """Final state, rank trace, timings and counters (reference engine.py:57-78)."""

    mode: Mode
    n: int
    final: GeneratorSet
    rank_trace: list
    timings: dict
    counters: dict
    k: int
    k_prime: int
    order: list = field(default_factory=list)
    # additions (not in the reference): what the device did
    device: dict = field(default_factory=dict)

    @property
    def mean_rank(self) -> float:
        return rank_stats(self.final)[1]

    @property
    def max_rank(self) -> int:
        return max(max(step) for step in self.rank_trace)


@dataclass
class AgreementReport:
    index_sets_equal: bool
    max_lambda_deviation: float


_DEVICE_TIMERS = bool(__import__("os").environ.get("QX_DEVICE_TIMERS"))
_WIDE_COMPACT = not __import__("os").environ.get("QX_NO_WIDE_COMPACT")


class _Phase:
    """``with walker.phase(name):`` -- see _Walker.phase."""

    __slots__ = ("w", "name", "store", "first", "t0")

    def __init__(self, w, name):
        self.w, self.name = w, name

    def __enter__(self):
        store = self.w.store
        self.store = store if self.w.device_timers and getattr(store, "mark", None) is not None else None
        self.t0 = time.perf_counter()
        self.first = self.store.mark() if self.store is not None else -1
        return self

    def __exit__(self, exc_type, exc, tb):
        w = self.w
        dt = time.perf_counter() - self.t0
        w.host_timings[self.name] = w.host_timings.get(self.name, 0.0) + dt
        if self.store is None:
            w.timings[self.name] += dt
        elif exc_type is None:
            w.regions.append((self.name, self.store, self.first, self.store.mark()))
        return False


class _Walker:
    """Schedules the device work of one run.

    Sign-permutation ops are queued and flushed as one fused launch.  The merge of a
    branching op is *deferred* past the permutation ops that follow it: they are bijections
    on words that keep |lambda|, so merging before or after them sums the same duplicates in
    the same order and drops the same terms -- but afterwards the result is already in the
    final order, which saves the reference's second sort (its canonicalize after every V_k).
    The deferred merge runs before the next branching op or at the end; rank-trace entries
    and v1 update counts that fall in between are filled in then.
    """

    def __init__(self, store: DeviceStore, n: int, ids, eps: float, timings: dict,
                 before_merge=None, reduce_ranks=None):
        self.store, self.n, self.ids, self.eps = store, n, list(ids), eps
        self.timings = timings
        self.before_merge, self.reduce_ranks = before_merge, reduce_ranks
        self.eager = False             # merge after every step (eps could drop an input term)
        self.dry = False               # replaying bookkeeping against recorded ranks: op words are not needed
        self.queue: list = []
        self.queue_has_cx = False
        self.unsorted = False          # a permutation ran since the last merge
        self.pending = None            # (step, phase) of a branching op whose merge is deferred
        self.staged = None             # (counts, axes, weights) of a U_k not launched yet (v2/v3)
        self.open_slots: list = []     # trace rows waiting for the deferred merge
        self.pending_gates = 0         # v1 gates applied since the deferred branch
        self.clean_gates = 0           # v1 gates that saw the current (merged) ranks, not yet booked
        self.ranks = [1] * len(self.ids)
        self.launch_log = {"clifford_runs": 0, "branch_ops": 0, "merges": 0, "sorts": 0}
        self.updates = None            # v1 only: term-gate updates per generator
        self.partition_rows = []       # slot-partitioned finish: trace rows that hold this share's counts
        self.partition_step = None
        self.device_timers = _DEVICE_TIMERS
        self.regions = []              # (phase, store, first event, second event): resolved by collect_timings
        self.host_timings = {"sub_flatten": 0.0, "cx": 0.0}

    # -- timers --------------------------------------------------------------------
    def phase(self, name: str):
        """Times a device phase for RunReport.timings (reference engine.py:92).  One-launch runs
        report the kernel's own clock.  Step-by-step runs: with ``device_timers`` (run(...,
        device_timers=True) or QX_DEVICE_TIMERS=1) CUDA events on the store's stream around the
        calls, resolved once at the end of the run -- the launches are asynchronous, a host clock
        around them measures the submission; the default is that host clock (every merge ends in a
        read-back, so it differs only for Clifford runs), because two event records per phase cost
        more than the phases of the small configs (C1: 0.10 -> 0.13 ms).  The host clock is kept
        beside either in ``report.device['host_timings']``."""
        return _Phase(self, name)

    def collect_timings(self):
        """Device phases in seconds, from the recorded event pairs (waits for the last event)."""
        for name, store, a, b in self.regions:
            self.timings[name] += store.elapsed_ms(a, b) * 1e-3
        self.regions = []

    # -- queue ---------------------------------------------------------------------
    def push_perm(self, qubit: int, table: int):
        if table != _lut.IDENTITY_PERM:
            self.queue.append(_lut.perm_op(self.n, qubit, table))

    def push_cx(self, control: int, target: int):
        self.queue.append(_lut.cx_op(self.n, control, target))
        self.queue_has_cx = True

    def flush(self):
        if not self.queue:
            return
        with self.phase("cx" if self.queue_has_cx else "sub_flatten"):
            self.store.apply_clifford(np.array(self.queue, dtype=_lut.op_dtype(self.n)))
        self.queue, self.queue_has_cx = [], False
        self.unsorted = True
        self.launch_log["clifford_runs"] += 1

    # -- merges ----------------------------------------------------------------------
    def book_gates(self):
        """v1 update counts: gates counted since the ranks last changed see exactly these ranks.
        Called before every assignment to ``self.ranks`` (one array operation per merge instead of
        one per gate)."""
        if self.updates is not None and self.clean_gates:
            self.updates += np.asarray(self.ranks, dtype=np.int64) * self.clean_gates
        self.clean_gates = 0

    def _merge_now(self, step: int, phase: str, after_branch: bool):
        self.book_gates()
        with self.phase(phase):
            if after_branch and self.before_merge is not None:
                self.before_merge(self.store)      # term-partitioned runs: equal keys must meet first
            self.ranks = self.store.merge(self.eps)
            if self.reduce_ranks is not None:
                self.ranks = self.reduce_ranks(self.ranks)
        self.unsorted = False
        self.launch_log["merges"] += 1
        for local, r in enumerate(self.ranks):
            if r == 0:
                raise NumericalCollapseError(
                    f"all terms of generator {self.ids[local]} dropped at operator step {step}"
                )

    def stage_operator(self, counts, axes, weights):
        """v2/v3: hold a branching U_k back until the permutation ops behind it are known; they
        are folded into its expansion kernel (qx_apply_operator_run)."""
        self.staged = (counts, axes, weights)

    def _run_staged(self, step: int, phase: str):
        self.book_gates()
        counts, axes, weights = self.staged
        self.staged = None
        program = np.array(self.queue, dtype=np.uint32)
        self.queue, self.queue_has_cx = [], False
        with self.phase(phase):
            if self.before_merge is not None:
                # term-partitioned runs re-home terms between the expansion and the merge
                self.store.apply_operator(counts, axes, weights)
                self.store.apply_clifford(program)
                self.before_merge(self.store)
                self.ranks = self.store.merge(self.eps)
            else:
                raw, self.ranks = self.store.apply_operator_run(counts, axes, weights, program, self.eps)
                # raw branches of the step (slots where the grouped step ran: the raw list is never written)
                self.launch_log["raw_terms"] = self.launch_log.get("raw_terms", 0) + int(raw)
            if self.reduce_ranks is not None:
                self.ranks = self.reduce_ranks(self.ranks)
        self.unsorted = False
        self.launch_log["merges"] += 1
        if len(program):
            self.launch_log["clifford_runs"] += 1
            self.launch_log["fused_runs"] = self.launch_log.get("fused_runs", 0) + 1
        for local, r in enumerate(self.ranks):
            if r == 0:
                raise NumericalCollapseError(
                    f"all terms of generator {self.ids[local]} dropped at operator step {step}"
                )

    def resolve(self, trace):
        """Run the deferred merge (after the permutation ops queued behind it)."""
        if self.pending is None:
            return
        step, phase = self.pending
        if self.staged is not None:
            self._run_staged(step, phase)
        else:
            self.flush()
            self._merge_now(step, phase, after_branch=True)
        self.pending = None
        row = list(self.ranks)
        for slot in self.open_slots:
            trace[slot] = row.copy()
        self.open_slots = []
        if self.updates is not None and self.pending_gates:
            self.updates += np.asarray(self.ranks, dtype=np.int64) * self.pending_gates
        self.pending_gates = 0

    def branched(self, step: int, phase: str, trace):
        """A branching kernel just ran: its merge is now owed."""
        self.launch_log["branch_ops"] += 1
        self.pending = (step, phase)
        if self.eager:
            self.resolve(trace)

    def step_done(self, step: int, phase: str, trace):
        """End of a permutation-only step."""
        if self.eager:
            self.flush()
            self._merge_now(step, phase, after_branch=False)

    def snapshot(self, trace):
        if self.pending is None:
            trace.append(list(self.ranks))
        else:
            self.open_slots.append(len(trace))
            trace.append(None)

    def snapshots(self, trace, k: int):
        """k rank-trace rows at once (runs of permutation operators)."""
        if self.pending is None:
            row = list(self.ranks)
            trace.extend([row.copy() for _ in range(k)])
        else:
            self.open_slots.extend(range(len(trace), len(trace) + k))
            trace.extend([None] * k)

    def count_gate(self):
        """v1: one more gate sees the current terms."""
        if self.pending is None:
            self.clean_gates += 1
        else:
            self.pending_gates += 1

    def finish(self, trace):
        self.resolve(trace)
        self.book_gates()
        self.flush()
        if self.unsorted:
            # only permutations since the last merge: canonicalize can only re-sort
            with self.phase("cx"):
                self.store.sort()
            self.unsorted = False
            self.launch_log["sorts"] += 1


def run(instructions: Sequence[Instruction], n: int, mode, eps: float = DEFAULT_EPS, *,
        device=None, generators=None, capacity: int = 0, pinned: bool = False,
        download: bool = True, initial=None, before_merge=None, reduce_ranks=None,
        slot_part=None, slot_reduce=None, device_timers=None) -> RunReport:
    """Simulate a circuit; returns the canonical final generator set.

    Positional arguments and result are the reference's (engine.py:89).  Keyword
    extras: ``device`` (CUDA ordinal; default QX_DEVICE / LOCAL_RANK / 0),
    ``generators`` (evolve only these generator ids -- they are independent, this is
    the multi-GPU shard), ``capacity`` (initial terms of HBM to reserve), ``pinned``
    (download into page-locked memory), ``download=False`` (leave the result in HBM;
    ``report.final`` is then None and ``report.device['store']`` holds the live
    store), ``initial`` (list of (lambdas, keys) replacing init_z, for read-out
    back-propagation), ``before_merge(store)`` / ``reduce_ranks(ranks)`` (hooks of the
    term-partitioned multi-GPU mode, see dist.py: re-home terms before a merge that
    follows a branching step, and turn local ranks into global ones), ``slot_part=(part,
    parts)`` / ``slot_reduce(ranks)`` (slot-partitioned multi-GPU mode, dist.run_slot_partitioned:
    the last branching operator only produces this part's share of every generator;
    ``report.device['partitioned']`` says whether it did), ``device_timers`` (time the device
    phases of ``timings`` with CUDA events instead of the host clock, see _Walker.phase).
    """
    mode = Mode.coerce(mode)
    timings = {"partition": 0.0, "lut": 0.0, "sub_flatten": 0.0, "cx": 0.0}
    counters = {"gates": len(instructions), "sub_flatten_ops": 0, "cx_applications": 0}

    if n < 1:
        raise ValueError(f"qubit count must be positive, got {n}")
    t0 = time.perf_counter()
    if not isinstance(instructions, (list, tuple)):
        instructions = list(instructions)
    plan = _plan_for(instructions, n, mode)
    partition = plan.partition
    timings["partition"] = time.perf_counter() - t0

    if initial is not None:
        ids = list(range(len(initial)))
    else:
        ids = list(range(n)) if generators is None else [int(g) for g in generators]
        if any(g < 0 or g >= n for g in ids):
            raise ValueError(f"generator ids {ids} out of range for n={n}")

    store = DeviceStore(n, max(len(ids), 1), capacity, device)
    handed_over = False
    try:
        if initial is not None:
            store.upload(initial)
            walker_ranks = [len(l) for l, _ in initial]
            lams = [np.asarray(l, dtype=np.float64).ravel() for l, _ in initial if len(l)]
            min_abs = float(np.min(np.abs(np.concatenate(lams)))) if lams else 1.0   # one pass, not one per segment
        else:
            walker_ranks = [1] * len(ids)
            min_abs = 1.0
        w = _Walker(store, n, ids, eps, timings, before_merge, reduce_ranks)
        if device_timers is not None:
            w.device_timers = bool(device_timers)
        w.ranks = reduce_ranks(walker_ranks) if reduce_ranks is not None else walker_ranks
        # If eps could already drop an initial term, merge after every step like the
        # reference does; otherwise deferring the re-sort of permutation steps is exact.
        eager = eps > min_abs
        if initial is not None:
            # caller-supplied generators may hold duplicate or sub-eps terms: canonicalize first
            eager = eager or any(len(k) > 1 and len(np.unique(k)) != len(k) for _, k in initial)
        w.eager = eager
        trace = [list(w.ranks)]

        # One launch for the whole circuit while every generator stays small (csrc/program.cuh);
        # v2 only where its dense layout needs no term-dependent decision (stabilizer.py:264-286)
        programmed, program_segs, made, prefixed = False, None, initial is not None, 0
        if (not eager and n <= 32 and before_merge is None and reduce_ranks is None and slot_part is None
                and _PROGRAMS_ON and ids and max(walker_ranks, default=0) <= PROGRAM_MAX_TERMS
                and store._cx == _lut.STANDARD_CX
                and (mode is not Mode.V2 or (4 ** n <= DENSE_FLATTEN_BUDGET and eps > 0.0))):
            t0 = time.perf_counter()
            if mode is not Mode.V1:
                plan.lut()
            program = _program_for(plan, instructions, n, mode, store.device)
            timings["lut"] = time.perf_counter() - t0
            if program is not None and program.fit_steps != 0:
                # generators that start as Z words are made in the kernel (no upload); a run that
                # does not fit leaves the store as init_z would have.  fit_steps: what an earlier
                # run of this plan found -- None: every step fits (or nothing is known yet), K > 0:
                # some generator outgrows shared memory at step K, so only the first K steps are
                # the one launch and the walk goes on step by step behind them
                prefix = program.fit_steps or 0
                whole = prefix == 0
                t0 = time.perf_counter()
                fitted, rows, program_raw, program_segs = store.run_program(
                    program, eps, init_qubits=None if made else ids, to_host=download and whole, pinned=pinned,
                    max_steps=prefix)
                made = True
                phase_key = "sub_flatten" if program.rows else "cx"
                w.host_timings[phase_key] += time.perf_counter() - t0
                if fitted and whole:
                    timings[phase_key] += store.program_ms * 1e-3      # the kernel's own clock (%globaltimer)
                    programmed = True
                    # the bookkeeping is a pure function of the plan's events and the recorded ranks:
                    # a run that recorded the ranks of the plan's previous run (the usual case: same
                    # circuit again) takes that run's trace, counters and update counts as they are
                    memo_key = (mode, tuple(walker_ranks))
                    memo = plan._replays.get(memo_key)
                    if memo is not None and memo[0] == rows:
                        _, tail, counter_delta, log_after, updates, last_ranks = memo
                        trace.extend([r.copy() for r in tail])
                        for k, v in counter_delta.items():
                            counters[k] = counters.get(k, 0) + v
                        w.launch_log.update(log_after)
                        w.updates = None if updates is None else updates.copy()
                        w.ranks = list(last_ranks)
                    else:
                        n0, c0 = len(trace), dict(counters)
                        w.store, w.dry = _ReplayStore(rows, store.device), True
                        _walk_events(w, _program_events(plan, instructions, mode), mode, trace, counters)
                        w.store, w.dry = store, False
                        w.book_gates()
                        plan._replays[memo_key] = (
                            rows, [r.copy() for r in trace[n0:]],
                            {k: v - c0.get(k, 0) for k, v in counters.items() if v != c0.get(k, 0)},
                            dict(w.launch_log), None if w.updates is None else w.updates.copy(), list(w.ranks))
                    w.launch_log["program_steps"] = program.steps
                    w.launch_log["raw_terms"] = w.launch_log.get("raw_terms", 0) + int(program_raw)
                elif fitted:
                    timings[phase_key] += store.program_ms * 1e-3
                    prefixed = prefix
                    w.store = _PrefixStore(rows, prefix, store)
                    w.launch_log["program_steps"] = prefix
                    w.launch_log["raw_terms"] = w.launch_log.get("raw_terms", 0) + int(program_raw)
                else:
                    # a generator outgrew it at this step: from the next run on only the steps in
                    # front of it are the one launch (0: none fits, never tried again)
                    program.fit_steps = min(store.program_stopped, prefix) if prefix else store.program_stopped
        if not made:
            store.init_z(ids)
        if programmed:
            pass
        elif mode is Mode.V1:
            if eager:
                w.updates = np.zeros(len(w.ids), dtype=np.int64)
                _walk_v1_eager(instructions, partition, w, trace, counters)
            else:
                _replay_v1(plan.v1_events(instructions), w, trace, counters)
        else:
            t0 = time.perf_counter()
            lut, is_perm, tables = plan.lut()
            timings["lut"] = time.perf_counter() - t0
            if eager or n > 32:
                _walk_operators(partition, lut, is_perm, tables, w, trace, counters, mode, eager)
            else:
                _replay_operators(plan.operator_events(), w, trace, counters, mode)

        if prefixed:
            # the walk has passed the steps the launch did: they come first, and the step that did
            # not fit -- a branching operator -- is the earliest the tail below can still owe
            if w.store.seen != prefixed:
                raise ConsistencyError(f"one-launch prefix of {prefixed} steps, the walk consumed {w.store.seen}")
            w.store = store
        streamed = None
        partitioned = None
        if programmed:
            pass
        elif slot_part is not None and before_merge is None and reduce_ranks is None:
            partitioned = _finish_partitioned(w, trace, slot_part, slot_reduce)
        elif download and before_merge is None and reduce_ranks is None:
            streamed = _finish_streamed(w, trace, pinned)
        if streamed is None and not programmed:
            w.finish(trace)              # deferred merge, queued permutations, canonical order
        counters["operators"] = partition.k + partition.k_prime

        w.collect_timings()              # device phases: CUDA events (host clock beside them in info)
        info = {"device": store.device, **w.launch_log, "host_timings": dict(w.host_timings)}
        if partitioned is not None:
            info["partitioned"] = partitioned
            if w.partition_step is not None:
                info["partition_rows"] = w.partition_rows
                info["partition_step"] = w.partition_step
        if w.updates is not None:
            w.book_gates()
            info["updates_per_generator"] = w.updates.tolist()
        final = None
        if download:
            segs = streamed if streamed is not None else program_segs if program_segs is not None else store.segments(pinned)
            final_gens = [SimpleGenerator(n, lam, keys_to_indices(keys, n)) for lam, keys in segs]
            whole = len(final_gens) == n and not partitioned
            final = GeneratorSet(n, final_gens) if whole else _Shard(n, ids, final_gens)
        else:
            info["store"] = store
            handed_over = True
        return RunReport(mode=mode, n=n, final=final, rank_trace=trace, timings=timings,
                         counters=counters, k=partition.k, k_prime=partition.k_prime,
                         order=list(partition.order), device=info)
    finally:
        # the store leaves with the report only on success; an error frees its HBM right away
        # instead of leaving it to the garbage collector (a retry near the capacity limit)
        if not handed_over:
            store.close()



# ------------------------------------------------------------------------------------------
# circuit plans: everything about a run that depends on the gate list only
# ------------------------------------------------------------------------------------------
# Walking 5000 gates in Python (partition, composed blocks, op words, branch tables) costs more
# than the device needs for the whole of configs 1/2/3/5.  None of it depends on the terms, so
# it is done once per gate list and replayed: a plan is a short list of EVENTS (queue these op
# words / branch here with these tables / snapshot the ranks) -- C5 in v3 is 41 events instead
# of 1647 operator steps.  Plans are found again by IDENTITY of the (immutable) instructions:
# `all(a is b)` over 5000 gates is ~0.1 ms, hashing them would cost more than it saves.
_PLAN_SLOTS = 8
_PROGRAMS_ON = not __import__("os").environ.get("QX_NO_PROGRAM")
SMALL_RAW = 8192                  # raw terms per generator the one-launch operator step takes (QX_SMALL_MAX)
_plans: list = []


class _Plan:
    def __init__(self, instructions, n: int):
        self.instructions = tuple(instructions)
        self.n = n
        self.partition = divide_instruction(self.instructions, n)
        self._lut = None
        self._v1 = None
        self._ops = None
        self._programs = {}            # (mode, device) -> CircuitProgram | None (does not qualify / did not fit)
        self._replays = {}             # (mode, initial ranks) -> bookkeeping of the last one-launch run

    def matches(self, instructions, n: int) -> bool:
        mine = self.instructions
        return n == self.n and len(instructions) == len(mine) and all(map(_is, instructions, mine))

    def lut(self):
        if self._lut is None:
            self._lut = _lut.build_lut(self.partition)
        return self._lut

    def v1_events(self, instructions):
        if self._v1 is None:
            self._v1 = _compile_v1(self.instructions, self.partition, self.n)
        return self._v1

    def operator_events(self):
        if self._ops is None:
            self._ops = _compile_operators(self.partition, *self.lut(), self.n)
        return self._ops


# ------------------------------------------------------------------------------------------
# whole-circuit programs (csrc/program.cuh)
# ------------------------------------------------------------------------------------------
# What a plan's events make the walker do on the device does not depend on the terms (as long as
# every generator stays small, nothing is term-partitioned and eps cannot drop an input term):
# the walker is run ONCE against a store that only records the calls, the record becomes a
# device-resident step list, and from then on a run is one launch + one read-back; the walker is
# then replayed against the recorded ranks for the rank trace, the update counts and the
# collapse error -- the same code that books them in the step-by-step path.
PROGRAM_MAX_TERMS = 4096          # terms per generator the one-launch path holds (kPgSrcCap)


class _RecordingStore:
    """Stands in for a DeviceStore while a plan is compiled: records the device steps."""

    mark = None                       # no stream: phases are not timed

    def __init__(self, n: int, n_gen: int):
        self.n, self.n_gen = n, n_gen
        self.steps, self.order_next = [], False

    def apply_clifford(self, program):
        if len(program):
            self.steps.append(("clifford", [int(v) for v in program]))

    def order_for_operator(self, counts, by_key: bool = True):
        if not by_key:
            raise _NoProgram
        self.order_next = True

    def apply_operator_run(self, counts, axes, weights, program, eps, term_limit: int = 0):
        self.steps.append(("oprun", self.order_next, counts, axes, weights, [int(v) for v in program]))
        self.order_next = False
        return 0, [1] * self.n_gen

    def sort(self):
        self.steps.append(("sort",))

    def __getattr__(self, name):      # anything else (merge, apply_split, count_operator ...): no program
        raise _NoProgram


class _ReplayStore:
    """Stands in for the store after the program ran: hands the recorded ranks to the walker."""

    mark = None

    def __init__(self, rows, device):
        self.rows, self.next, self.device = rows, 0, device

    def apply_clifford(self, program):
        pass

    def order_for_operator(self, counts, by_key: bool = True):
        pass

    def sort(self):
        pass

    def apply_operator_run(self, counts, axes, weights, program, eps, term_limit: int = 0):
        row = self.rows[self.next]
        self.next += 1
        return 0, list(row)


class _PrefixStore:
    """The store of a run whose first ``done`` device steps were ONE launch (a circuit whose
    generators outgrow shared memory later): those steps hand out the recorded ranks, everything
    behind them goes to the real store.  Steps are counted exactly as _RecordingStore records them."""

    def __init__(self, rows, done: int, real):
        self.rows, self.done, self.real = rows, done, real
        self.seen = self.next = 0

    def apply_clifford(self, program):
        if not len(program):
            return
        if self.seen < self.done:
            self.seen += 1
        else:
            self.real.apply_clifford(program)

    def order_for_operator(self, counts, by_key: bool = True):
        if self.seen >= self.done:           # otherwise part of the recorded operator step
            self.real.order_for_operator(counts, by_key)

    def apply_operator_run(self, counts, axes, weights, program, eps, term_limit: int = 0):
        if self.seen < self.done:
            self.seen += 1
            row = self.rows[self.next]
            self.next += 1
            return 0, list(row)
        return self.real.apply_operator_run(counts, axes, weights, program, eps, term_limit)

    def sort(self):
        if self.seen < self.done:
            self.seen += 1
        else:
            self.real.sort()

    def __getattr__(self, name):
        return getattr(self.real, name)


class _NoProgram(Exception):
    pass


def _program_events(plan: "_Plan", instructions, mode):
    if mode is Mode.V1:
        return plan.v1_events(instructions)
    return plan.operator_events()


def _walk_events(w: _Walker, compiled, mode, trace, counters):
    if mode is Mode.V1:
        _replay_v1(compiled, w, trace, counters)
    else:
        _replay_operators(compiled, w, trace, counters, mode)
    w.finish(trace)


def _program_for(plan: "_Plan", instructions, n: int, mode, device: int):
    """The plan's device program for this mode, compiled on first use; None if it has none."""
    key = (mode, device)
    if key not in plan._programs:
        program = None
        try:
            rec = _RecordingStore(n, n)
            w = _Walker(rec, n, range(n), DEFAULT_EPS, {"partition": 0.0, "lut": 0.0, "sub_flatten": 0.0, "cx": 0.0})
            _walk_events(w, _program_events(plan, instructions, mode), mode, [list(w.ranks)],
                         {"sub_flatten_ops": 0, "cx_applications": 0})
            if rec.steps:
                program = CircuitProgram(n, rec.steps, device)
        except _NoProgram:
            program = None
        plan._programs[key] = program
    return plan._programs[key]


def _plan_for(instructions, n: int, mode) -> _Plan:
    for i, plan in enumerate(_plans):
        if plan.matches(instructions, n):
            if i:
                _plans.insert(0, _plans.pop(i))
            return plan
    plan = _Plan(instructions, n)
    _plans.insert(0, plan)
    del _plans[_PLAN_SLOTS:]
    return plan


def clear_plans():
    """Forget the cached circuit plans (tests; long-running services that stream distinct circuits)."""
    _plans.clear()


def _compile_v1(instructions, partition, n: int) -> tuple:
    """Events of the gate-by-gate walk (reference engine.py:155-180) for a store that merges only
    where terms branch: ('q', op words, has_cx, gates) | ('split', position, qubit, tables) |
    ('snap',) at operator boundaries."""
    sh1, sh2 = (32, 48) if n > 32 else (2, 8)
    pos_a = [(2 * (n - 1 - q)) << sh1 for q in range(n)]
    pos_b = [(2 * (n - 1 - q)) << sh2 for q in range(n)]
    fixed = {g: t << 16 for g, t in _lut.FIXED_PERMS.items()}
    fixed_get = fixed.get
    bounds = iter(np.cumsum(partition.operator_sizes()).tolist())
    nb = next(bounds, -1)
    events, ops, has_cx, cnt, n_cx = [], [], False, 0, 0

    def close():
        nonlocal ops, has_cx, cnt
        if ops or cnt:
            events.append(("q", ops, has_cx, cnt))
        ops, has_cx, cnt = [], False, 0

    for pos, inst in enumerate(instructions, start=1):
        wires = inst.wires
        if len(wires) == 2:
            ops.append(1 | pos_a[wires[0]] | pos_b[wires[1]])
            has_cx = True
            n_cx += 1
            cnt += 1
        else:
            op = fixed_get(inst.gate)
            if op is not None:
                ops.append(op | pos_a[wires[0]])
                cnt += 1
            else:
                block = _lut.gate_branch_block(inst.gate, inst.theta)
                table = _lut.perm_word(block)
                if table is not None:
                    if table != _lut.IDENTITY_PERM:
                        ops.append(_lut.perm_op(n, wires[0], table))
                    cnt += 1
                else:
                    close()
                    # the same gate as a one-qubit operator table: small stores take the fused
                    # expand + run + merge launch of the operator path (two contributions per
                    # word at most, so the sums are the reference's bit for bit)
                    full = np.tile(np.eye(3), (n, 1, 1))
                    full[wires[0]] = block
                    events.append(("split", pos, wires[0], split_tables(block),
                                   _lut.operator_tables(full) if n <= 32 else None))
        if pos == nb:
            close()
            events.append(("snap",))
            nb = next(bounds, -1)
    close()
    return events, n_cx, len(instructions) - n_cx


def _replay_v1(compiled, w: _Walker, trace, counters):
    events, n_cx, n_1q = compiled
    w.updates = np.zeros(len(w.ids), dtype=np.int64)
    snaps = 0                          # rows that only repeat the current ranks: appended in bulk
    for ev in events:
        kind = ev[0]
        if kind == "q":
            if w.dry:
                w.queue.extend(ev[1][:1])      # only whether there are ops matters to the bookkeeping
            else:
                w.queue.extend(ev[1])
            w.queue_has_cx = w.queue_has_cx or ev[2]
            if w.pending is None:
                w.clean_gates += ev[3]
            else:
                w.pending_gates += ev[3]
        elif kind == "snap":
            snaps += 1
        else:
            _, pos, qubit, tables, as_operator = ev
            if snaps:
                w.snapshots(trace, snaps)
                snaps = 0
            w.resolve(trace)                   # this gate must see merged terms
            w.count_gate()
            w.flush()
            if as_operator is not None and w.before_merge is None and 2 * max(w.ranks, default=0) <= SMALL_RAW:
                w.stage_operator(*as_operator)     # split + the run behind it + merge: one launch
            else:
                with w.phase("sub_flatten"):
                    w.store.apply_split(qubit, *tables)
            w.branched(pos - 1, "sub_flatten", trace)
    if snaps:
        w.snapshots(trace, snaps)
    counters["cx_applications"] += n_cx
    if n_1q:
        counters["v1_gate_applications"] = counters.get("v1_gate_applications", 0) + n_1q


def _compile_operators(partition, lut, is_perm, tables, n: int) -> tuple:
    """Events of the operator chain (reference engine.py:110-132), n <= 32, deferred merges:
    ('q', op words, has_cx, snapshots) for runs of permutation operators and CX groups,
    ('b', step, counts, axes, weights) for a U_k that branches (followed by its own snapshot)."""
    events, ops, has_cx, snaps = [], [], False, 0
    n_cx = 0
    ui = vi = 0
    if partition.k:
        all_perm = is_perm.all(axis=1).tolist()
        shifts = (2 * (n - 1 - np.arange(n, dtype=np.uint64)))[None, :]
        ops_all = (tables.astype(np.uint64) << np.uint64(16)) | (shifts << np.uint64(2))
        live = tables != _lut.IDENTITY_PERM
        perm_ops = ops_all[live].tolist()
        perm_off = np.concatenate(([0], np.cumsum(live.sum(axis=1)))).tolist()

    def close():
        nonlocal ops, has_cx, snaps
        if ops or snaps:
            events.append(("q", ops, has_cx, snaps))
        ops, has_cx, snaps = [], False, 0

    for step, bit in enumerate(partition.order):
        if bit == 0:
            if all_perm[ui]:
                ops.extend(perm_ops[perm_off[ui]:perm_off[ui + 1]])
            else:
                close()
                events.append(("b", step, *_lut.operator_tables(lut[ui])))
            ui += 1
        else:
            for inst in partition.v_groups[vi]:
                ops.append(_lut.cx_op(n, *inst.wires))
            has_cx = has_cx or bool(partition.v_groups[vi])
            n_cx += len(partition.v_groups[vi])
            vi += 1
        snaps += 1
    close()
    return events, partition.k, n_cx


def _replay_operators(compiled, w: _Walker, trace, counters, mode):
    events, n_u, n_cx = compiled
    n = w.n
    for ev in events:
        if ev[0] == "q":
            if w.dry:
                w.queue.extend(ev[1][:1])      # only whether there are ops matters to the bookkeeping
            else:
                w.queue.extend(ev[1])
            w.queue_has_cx = w.queue_has_cx or ev[2]
            w.snapshots(trace, ev[3])
            continue
        _, step, counts, axes, weights = ev
        w.resolve(trace)               # expand merged terms only
        w.flush()
        ph = w.phase("sub_flatten").__enter__()
        if mode is Mode.V2 and 4 ** n > DENSE_FLATTEN_BUDGET:
            # dense layout: a branching substitution needs a 4**n scatter buffer
            # (reference stabilizer.py:264-276); one-hot rows take the fast path
            raw = w.store.count_operator(counts)
            over = any(r > have for r, have in zip(raw, w.store.ranks()))
            if w.reduce_ranks is not None:
                # term-partitioned runs: a rank that holds no branching term of a generator
                # must raise too, or it would wait for the others in the next collective
                over = w.reduce_ranks([int(over)])[0] > 0
            if over:
                raise ResourceLimitError(
                    f"dense flatten needs a 4**{n}-element buffer (> {DENSE_FLATTEN_BUDGET}); "
                    "use the ragged layout for circuits of this size"
                )
        if mode is Mode.V3:
            # the reference's ragged flatten walks the strings grouped by their branch-count
            # pattern (stabilizer.py:294-296); same order here, so that sums of three or more
            # contributions round the same way (the store may also sit in a permuted order:
            # the re-sort after the last Clifford run is deferred)
            w.store.order_for_operator(counts)
        dense_gens = []
        if mode is Mode.V2 and w.eps == 0.0 and 4 ** n <= DENSE_FLATTEN_BUDGET and w.before_merge is None:
            # dense layout, eps = 0: a generator with a branching row comes back from the
            # reference's 4**n buffer with every word, zeros included (stabilizer.py:277-286)
            raw = w.store.count_operator(counts)
            dense_gens = [g for g, (r, have) in enumerate(zip(raw, w.store.ranks())) if r > have]
        if dense_gens:
            w.store.apply_operator(counts, axes, weights)
            pad_dense(w.store, n, dense_gens)
        else:
            w.stage_operator(counts, axes, weights)
        ph.__exit__(None, None, None)
        w.branched(step, "sub_flatten", trace)
    counters["sub_flatten_ops"] += n_u
    counters["cx_applications"] += n_cx


_STREAM_DEBUG = bool(__import__("os").environ.get("QX_STREAM_DEBUG"))
_NARROW_DOWNLOAD = not __import__("os").environ.get("QX_NO_NARROW_DOWNLOAD")
_NARROW_FORM = int(__import__("os").environ.get("QX_NARROW_FORM", "2"))   # 1: 32-bit keys, 2: packed allowed
STREAM_MIN_RAW = 1 << 23          # below this a single download is not worth splitting
STREAM_SHARDS = 4


def _finish_streamed(w: _Walker, trace, pinned: bool):
    """Last branching operator of a run whose result goes to the host: evolve contiguous
    generator ranges one after the other, each on a store (and CUDA stream) of its own, and
    start every range's download as soon as its merge is done, so that the PCIe copy of one
    range overlaps the kernels of the next.  Generators are independent (reference
    engine.py:113-116), so the result is the same.  Returns the per-generator (lambdas, keys)
    list, or None when the plain finish applies (no staged operator, small result)."""
    if w.pending is None or w.staged is None or len(w.ids) < 2:
        return None
    counts, axes, weights = w.staged
    raw = w.store.count_operator(counts)
    # a generator never holds more than 4**n terms, however many raw branches feed it
    if sum(min(r, 4 ** w.n) for r in raw) < STREAM_MIN_RAW:
        return None
    step, phase = w.pending
    # contiguous ranges of about equal raw size, smallest first: its copy starts early and the
    # heavier ranges compute underneath it
    target = sum(raw) / STREAM_SHARDS
    bounds, acc = [0], 0
    for g, r in enumerate(raw):
        acc += r
        if acc >= target and g + 1 < len(raw):
            bounds.append(g + 1)
            acc = 0
    bounds.append(len(raw))
    ranges = sorted(zip(bounds[:-1], bounds[1:]), key=lambda ab: sum(raw[ab[0]:ab[1]]))
    program = np.array(w.queue, dtype=np.uint32)
    w.queue, w.queue_has_cx, w.staged, w.pending = [], False, None, None
    w.book_gates()
    ph = w.phase(phase).__enter__()
    t0 = time.perf_counter()
    parts, children = {}, []
    ranks = [0] * len(w.ids)
    try:
        for lo, hi in ranges:
            # no capacity hint: the operator step reserves what it needs (slots, not raw branches)
            child = w.store.slice(lo, hi, 0)
            children.append(child)
            if pinned and w.n <= 16 and _NARROW_DOWNLOAD:
                child.set_keep_narrow(_NARROW_FORM)   # only downloaded next: 16- or 32-bit keys over PCIe
            _, r = child.apply_operator_run(counts, axes, weights, program, w.eps)
            ranks[lo:hi] = r
            for local, v in enumerate(r):
                if v == 0:
                    raise NumericalCollapseError(
                        f"all terms of generator {w.ids[lo + local]} dropped at operator step {step}"
                    )
            parts[lo] = (hi, child.download_async(pinned))
            if _STREAM_DEBUG:
                print(f"  range [{lo},{hi}) issued at {1e3 * (time.perf_counter() - t0):.2f} ms, {sum(r)} terms")
        for child in children:
            child.synchronize()
            if _STREAM_DEBUG:
                print(f"  synchronized at {1e3 * (time.perf_counter() - t0):.2f} ms")
    finally:
        for child in children:
            child.close()
    ph.__exit__(None, None, None)
    w.ranks = ranks
    w.launch_log["merges"] += 1
    w.launch_log["branch_ops"] += 0
    w.launch_log["streamed_ranges"] = len(ranges)
    w.launch_log["d2h_bytes"] = sum(getattr(c, "d2h_bytes", 0) for c in children)
    for slot in w.open_slots:
        trace[slot] = list(ranks)
    w.open_slots = []
    if w.updates is not None and w.pending_gates:
        w.updates += np.asarray(ranks, dtype=np.int64) * w.pending_gates
    w.pending_gates = 0
    w.unsorted = False
    out = []
    for lo in sorted(parts):
        hi, (off, keys, lam) = parts[lo]
        out.extend((lam[off[i]:off[i + 1]], keys[off[i]:off[i + 1]]) for i in range(hi - lo))
    return out


def _finish_partitioned(w: _Walker, trace, slot_part, slot_reduce):
    """Slot-partitioned multi-GPU finish: every device holds the same terms in front of the last
    branching operator and works off its own range of output slots (qx_apply_operator_run_part).
    Returns True if the store now holds only this part's share, False if the operator did not take
    the grouped path (the result is then complete and identical on every device), None if there
    is no staged operator (the plain finish applies)."""
    if w.pending is None or w.staged is None:
        return None
    part, parts = slot_part
    counts, axes, weights = w.staged
    step, phase = w.pending
    program = np.array(w.queue, dtype=np.uint32)
    w.queue, w.queue_has_cx, w.staged, w.pending = [], False, None, None
    w.book_gates()
    ph = w.phase(phase).__enter__()
    ranks, partitioned = w.store.apply_operator_run_part(counts, axes, weights, program, w.eps, part, parts)
    if partitioned and slot_reduce is not None:
        ranks = slot_reduce(ranks)              # global ranks: sum of the shares
    ph.__exit__(None, None, None)
    w.ranks = list(ranks)
    w.unsorted = False
    w.launch_log["merges"] += 1
    if partitioned is False or slot_reduce is not None or parts == 1:
        for local, r in enumerate(w.ranks):
            if r == 0:
                raise NumericalCollapseError(
                    f"all terms of generator {w.ids[local]} dropped at operator step {step}"
                )
    for slot in w.open_slots:
        trace[slot] = list(w.ranks)
    if partitioned and slot_reduce is None and parts > 1:
        # the caller sums the shares' counts itself (dist.run_slot_partitioned): these rows and the
        # rows appended from now on hold this share's counts
        w.partition_rows = list(w.open_slots)
        w.partition_step = step
    w.open_slots = []
    if w.updates is not None and w.pending_gates:
        w.updates += np.asarray(w.ranks, dtype=np.int64) * w.pending_gates
    w.pending_gates = 0
    return partitioned


@dataclass
class _Shard:
    """A subset of the generators (multi-GPU shard or read-out words): same fields as
    GeneratorSet without the exactly-n check, plus the global ids."""

    n: int
    ids: list
    generators: list


def _walk_v1_eager(instructions, partition, w: _Walker, trace, counters):
    """The same walk with a merge after every gate (eps could drop an input term)."""
    boundaries = set(np.cumsum(partition.operator_sizes()).tolist())
    n = w.n
    fixed = _lut.FIXED_PERMS
    n_cx = n_1q = 0
    for pos, inst in enumerate(instructions, start=1):
        wires = inst.wires
        if len(wires) == 2:
            w.count_gate()
            w.queue.append(_lut.cx_op(n, wires[0], wires[1]))
            w.queue_has_cx = True
            n_cx += 1
            w.step_done(pos - 1, "cx", trace)
        else:
            q = wires[0]
            table = fixed.get(inst.gate)
            block = None
            if table is None:
                block = _lut.gate_branch_block(inst.gate, inst.theta)
                table = _lut.perm_word(block)
            if table is not None:
                w.count_gate()
                if table != _lut.IDENTITY_PERM:
                    w.queue.append(_lut.perm_op(n, q, table))
                w.step_done(pos - 1, "sub_flatten", trace)
            else:
                w.resolve(trace)               # this gate must see merged terms
                w.count_gate()
                w.flush()
                with w.phase("sub_flatten"):
                    w.store.apply_split(q, *split_tables(block))
                w.branched(pos - 1, "sub_flatten", trace)
            n_1q += 1
        if pos in boundaries:
            w.snapshot(trace)
    counters["cx_applications"] += n_cx
    if n_1q:
        counters["v1_gate_applications"] = counters.get("v1_gate_applications", 0) + n_1q


# raw terms a multi-word operator walk may pile up before duplicates are summed (eps = 0)
WIDE_RAW_BUDGET = 1 << 16


def _operator_on_support(w: _Walker, block, step: int, mode) -> bool:
    """A branching U_k on a multi-word store whose terms live on at most 32 qubits: pack them into
    one-word keys over their support (csrc/wide.cu qx_store_compact), run the one-word operator
    step there -- the reference's sub + flatten + canonicalize (stabilizer.py:189-337), with its
    string order in v3 (stabilizer.py:294-296) -- and spread the result back.  Identity digits
    neither branch nor change a coefficient, so this is what the reference computes with big-int
    indices (stabilizer.py:40-59).  Generators without a digit on a qubit the operator touches are
    left alone (every such term maps to itself with weight exactly 1).  Returns False (nothing
    touched but the queue flushed) when the support of the others is wider than a word or the
    run is term-partitioned."""
    if w.before_merge is not None or w.reduce_ranks is not None or w.store.words <= 1 or not _WIDE_COMPACT:
        return False
    w.flush()                          # queued permutations move the support
    counts, axes, weights = _lut.operator_tables(block)
    # qubits the operator touches at all (any cell that is not "this axis, weight +1")
    ident_axes = np.arange(1, 4)
    touched = 0
    for q in range(w.n):
        if not (np.all(counts[q] == 1) and np.all(axes[q][:, 0] == ident_axes) and np.all(weights[q][:, 0] == 1.0)):
            touched |= 1 << q
    masks = w.store.support()
    take = [bool(m & touched) for m in masks]
    union = 0
    for m, t in zip(masks, take):
        if t:
            union |= m
    sel = [q for q in range(w.n) if (union >> q) & 1]
    if not any(take):
        return True                    # no generator has a digit the operator touches: nothing changes
    if len(sel) > 32:
        return False
    c, a, wt = counts[sel], axes[sel], weights[sel]
    w.book_gates()
    narrow = w.store.compact(sel, take)
    try:
        if mode is Mode.V3:
            narrow.order_for_operator(c)
        _, nranks = narrow.apply_operator_run(c, a, wt, np.zeros(0, dtype=np.uint32), w.eps)
        w.store.expand_from(narrow, sel, take)
    finally:
        narrow.close()
    ranks = [nr if t else old for nr, old, t in zip(nranks, w.ranks, take)]
    w.ranks = list(ranks)
    # the generators that went through the operator step are canonical now; the others sit as the
    # last permutation run left them
    w.unsorted = w.unsorted and not all(take)
    w.launch_log["branch_ops"] += 1
    w.launch_log["merges"] += 1
    w.launch_log["compacted_operators"] = w.launch_log.get("compacted_operators", 0) + 1
    for local, r in enumerate(w.ranks):
        if r == 0:
            raise NumericalCollapseError(f"all terms of generator {w.ids[local]} dropped at operator step {step}")
    return True


def _walk_operators(partition, lut, is_perm, tables, w: _Walker, trace, counters, mode, eager):
    """Operator chain (reference engine.py:110-132): U_k = substitute + flatten, V_k = CX run."""
    n = w.n
    ui = vi = 0
    if partition.k:
        # op words of every permutation cell of the circuit in one go (lut.perm_op, vectorised):
        # the walk below only slices a Python list per operator
        all_perm = is_perm.all(axis=1).tolist()
        shifts = (2 * (n - 1 - np.arange(n, dtype=np.uint64)))[None, :]
        wide = tables.astype(np.uint64) << np.uint64(16)
        ops_all = (wide | (shifts << np.uint64(32))) if n > 32 else (wide | (shifts << np.uint64(2)))
        live = tables != _lut.IDENTITY_PERM
        perm_ops = ops_all[live].tolist()
        perm_off = np.concatenate(([0], np.cumsum(live.sum(axis=1)))).tolist()
    for step, bit in enumerate(partition.order):
        if bit == 0:
            if all_perm[ui]:
                w.queue.extend(perm_ops[perm_off[ui]:perm_off[ui + 1]])
                w.step_done(step, "sub_flatten", trace)
            elif n > 32:
                # Multi-word keys: the operator is applied gate by gate, wire by wire, with the
                # v1 kernels and merged ONCE, where the reference merges its flattened expansion
                # (stabilizer.py:240-256).  The raw terms are the same Cartesian product (a path
                # per non-zero product of gate entries instead of a branch per non-zero block
                # entry: paths to the same word are summed by the merge, to rounding what the
                # reference's 3x3 products sum), so term sets after the drop rule agree.
                # Every split doubles the raw list (multi-word splits write both branches of every
                # term), so a long operator is summed in between with eps = 0: nothing is dropped
                # before the operator's own merge, only duplicates meet earlier.
                w.resolve(trace)               # expand merged terms only
                bucket = partition.u_groups[ui]
                ph = w.phase("sub_flatten").__enter__()
                if mode is Mode.V2:
                    # dense layout: a row of the substituted block that is not one-hot needs the
                    # 4**n scatter buffer (reference stabilizer.py:264-276).  Nothing has ever
                    # branched when this is reached, so the generators are a handful of terms.
                    counts, _, _ = _lut.operator_tables(lut[ui])
                    wires_ = np.flatnonzero(counts.max(axis=1) > 1).tolist()
                    w.flush()
                    for _, words in w.store.segments():
                        for word in words:
                            for q in wires_:
                                d = (int(word) >> (2 * (n - 1 - q))) & 3
                                if d and counts[q, d - 1] > 1:
                                    raise ResourceLimitError(
                                        f"dense flatten needs a 4**{n}-element buffer (> {DENSE_FLATTEN_BUDGET}); "
                                        "use the ragged layout for circuits of this size"
                                    )
                if _operator_on_support(w, lut[ui], step, mode):
                    # the store's support fits one word: the grouped one-word operator step ran on
                    # the compacted terms (sub + flatten + merge, exactly where the reference merges)
                    ph.__exit__(None, None, None)
                else:
                    raw = sum(w.ranks)
                    for wire in sorted(bucket):
                        for inst in bucket[wire]:
                            table = _lut.FIXED_PERMS.get(inst.gate)
                            block = None
                            if table is None:
                                block = _lut.gate_branch_block(inst.gate, inst.theta)
                                table = _lut.perm_word(block)
                            if table is not None:
                                w.push_perm(wire, table)
                            else:
                                w.flush()
                                w.store.apply_split(wire, *split_tables(block))
                                raw *= 2
                                if raw > WIDE_RAW_BUDGET:
                                    raw = sum(w.store.merge(0.0))
                                    w.unsorted = False
                    ph.__exit__(None, None, None)
                    w.branched(step, "sub_flatten", trace)
            else:
                w.resolve(trace)               # expand merged terms only
                w.flush()
                counts, axes, weights = _lut.operator_tables(lut[ui])
                ph = w.phase("sub_flatten").__enter__()
                if mode is Mode.V2 and 4 ** n > DENSE_FLATTEN_BUDGET:
                    # dense layout: a branching substitution needs a 4**n scatter buffer
                    # (reference stabilizer.py:264-276); one-hot rows take the fast path
                    raw = w.store.count_operator(counts)
                    over = any(r > have for r, have in zip(raw, w.store.ranks()))
                    if w.reduce_ranks is not None:
                        # term-partitioned runs: a rank that holds no branching term of a generator
                        # must raise too, or it would wait for the others in the next collective
                        over = w.reduce_ranks([int(over)])[0] > 0
                    if over:
                        raise ResourceLimitError(
                            f"dense flatten needs a 4**{n}-element buffer (> {DENSE_FLATTEN_BUDGET}); "
                            "use the ragged layout for circuits of this size"
                        )
                if mode is Mode.V3:
                    # the reference's ragged flatten walks the strings grouped by their branch-count
                    # pattern (stabilizer.py:294-296); same order here, so that sums of three or more
                    # contributions round the same way (the store may also sit in a permuted order:
                    # the re-sort after the last Clifford run is deferred)
                    w.store.order_for_operator(counts)
                dense_gens = []
                if mode is Mode.V2 and w.eps == 0.0 and 4 ** n <= DENSE_FLATTEN_BUDGET and w.before_merge is None:
                    # dense layout, eps = 0: a generator with a branching row comes back from the
                    # reference's 4**n buffer with every word, zeros included (stabilizer.py:277-286)
                    raw = w.store.count_operator(counts)
                    dense_gens = [g for g, (r, have) in enumerate(zip(raw, w.store.ranks())) if r > have]
                if dense_gens:
                    w.store.apply_operator(counts, axes, weights)
                    pad_dense(w.store, n, dense_gens)
                else:
                    w.stage_operator(counts, axes, weights)
                ph.__exit__(None, None, None)
                w.branched(step, "sub_flatten", trace)
            counters["sub_flatten_ops"] += 1
            ui += 1
        else:
            for inst in partition.v_groups[vi]:
                w.push_cx(*inst.wires)
                counters["cx_applications"] += 1
            w.step_done(step, "cx", trace)
            vi += 1
        w.snapshot(trace)


def run_all_modes(instructions: Sequence[Instruction], n: int, eps: float = DEFAULT_EPS, **kw):
    """Every mode on the same circuit + pairwise comparison (reference engine.py:221-226)."""
    reports = {mode: run(instructions, n, mode, eps, **kw) for mode in Mode}
    return reports, compare_reports(list(reports.values()))


def compare_reports(reports: Sequence[RunReport]) -> AgreementReport:
    """Index-set equality and max coefficient deviation (reference engine.py:229-243)."""
    equal, worst = True, 0.0
    for i, a in enumerate(reports):
        for b in reports[i + 1:]:
            for ga, gb in zip(a.final.generators, b.final.generators):
                if ga.rank != gb.rank or list(ga.indices) != list(gb.indices):
                    equal = False
                elif ga.rank:
                    worst = max(worst, float(np.max(np.abs(ga.lambdas - gb.lambdas))))
    return AgreementReport(equal, worst if equal else float("inf"))
