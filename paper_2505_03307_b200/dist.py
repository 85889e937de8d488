"""Multi-GPU plumbing: one process per GPU, ``torch.distributed`` (NCCL over NVLink).

Nothing here exists in the reference (it is single-process, engine.py:12-13); this is
the B200-native scale-out of SURVEY.md sections 5.9 / 8e.

* ``run_sharded`` -- the default.  The n generators evolve independently
  (reference engine.py:113-116), so each rank takes a subset (longest-processing-time
  on predicted rank) and runs the whole circuit on its own HBM with NO data-path
  collective.  Afterwards the rank traces are all-gathered (a few integers) and, if
  asked, the final generators are gathered as padded tensors.
* ``run_term_partitioned`` -- when there are fewer generators than GPUs or one
  generator dominates.  Every rank holds the terms it owns (owner = mix64(key) % world).
  Clifford runs and the branching kernels are local; only immediately before a merge
  that follows a branching step are terms re-homed with one all-to-all-v
  (``exchange_terms``), because that is the only point where equal keys must meet.
  Scalars (ranks for the trace / collapse check) are all-reduced.

* ``run_slot_partitioned`` -- one circuit, every rank takes a range of the output slots of the
  last branching operator (csrc/dense.cu): even split whatever the skew, no collective.
* ``expectation_sharded`` / ``prob_z_sharded`` -- read-out, observable-parallel:
  the words are independent back-propagations (``measure.expectation_heisenberg``), each rank
  takes every world-th word, and ONE all-reduce of the result vector hands every rank all
  scalars (each scalar is owned by one rank, the others add +0.0: the sum is exact).

The functions take an injected ``runner`` / tensors so the host logic (sharding,
split sizes, gather/assemble) is testable with the gloo backend on CPU; the compute
always goes through the CUDA library.
"""

from __future__ import annotations

import numpy as np

from .stabilizer import GeneratorSet, SimpleGenerator, keys_to_indices

MIX_A = np.uint64(0x9E3779B97F4A7C15)
MIX_B = np.uint64(0xBF58476D1CE4E5B9)
MIX_C = np.uint64(0x94D049BB133111EB)


def owner_of(keys: np.ndarray, world: int) -> np.ndarray:
    """Host mirror of the device hash in csrc/partition.cu (splitmix64 finaliser % world)."""
    with np.errstate(over="ignore"):
        z = keys.astype(np.uint64) + MIX_A
        z = (z ^ (z >> np.uint64(30))) * MIX_B
        z = (z ^ (z >> np.uint64(27))) * MIX_C
        z = z ^ (z >> np.uint64(31))
    return (z % np.uint64(world)).astype(np.int64)


def lpt_shards(weights, world: int) -> list:
    """Longest-processing-time assignment of generator ids to ranks.

    Generator ranks are skewed by orders of magnitude on the ansatz circuits
    (SURVEY.md 5.9), so ``j % world`` would leave most GPUs idle.
    """
    loads = [0.0] * world
    shards = [[] for _ in range(world)]
    for g in sorted(range(len(weights)), key=lambda i: (-float(weights[i]), i)):
        r = min(range(world), key=lambda i: (loads[i], i))
        shards[r].append(g)
        loads[r] += float(weights[g])
    return [sorted(s) for s in shards]


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised (launch with torchrun)")
    return dist


def _comm_device(group=None):
    import torch

    dist = _dist()
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if "nccl" in str(backend) else torch.device("cpu")


class RemoteRankError(RuntimeError):
    """Another rank of the job failed; raised on the ranks that did not, so that nobody is left
    waiting in a collective."""


def agree_on_errors(exc, group=None):
    """Every rank calls this with its own exception (or None) BEFORE the next collective.  If any
    rank failed, all of them raise: the failing ranks their own exception, the others a
    ``RemoteRankError`` naming the first failing rank and its message.  One small all-gather."""
    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = None if exc is None else (type(exc).__name__, str(exc))
    if world == 1:
        everyone = [mine]
    else:
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
    failed = [(r, e) for r, e in enumerate(everyone) if e is not None]
    if not failed:
        return
    if exc is not None:
        raise exc
    r, (kind, msg) = failed[0]
    raise RemoteRankError(f"rank {r} failed with {kind}: {msg} (this is rank {rank})")


def run_sharded(instructions, n: int, mode, eps: float = 1e-12, *, weights=None, gather: bool = True,
                group=None, runner=None, **run_kw):
    """Generator-sharded run.  Returns (report, shards).

    ``report`` is this rank's RunReport, except that ``rank_trace`` covers all n
    generators (all-gathered) and, with ``gather=True``, ``final`` is the full
    GeneratorSet on every rank.  ``weights`` are predicted per-generator costs for the
    LPT split (default: uniform).  ``runner`` defaults to ``engine.run``.
    """
    import torch

    dist = _dist()
    if runner is None:
        from .engine import run as runner
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    shards = lpt_shards(weights if weights is not None else [1.0] * n, world)
    mine = shards[rank]
    report, failure = None, None
    try:
        report = runner(instructions, n, mode, eps, generators=mine, **run_kw) if mine else None
    except Exception as exc:          # a shard's collapse / resource error: the others must not wait for it
        failure = exc
    agree_on_errors(failure, group)

    dev = _comm_device(group)
    # ---- rank trace: every rank contributes its columns (a few integers per step)
    steps = len(report.rank_trace) if report is not None else 0
    t = torch.tensor([steps], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    steps = int(t.item())
    cols = torch.zeros((steps, n), dtype=torch.int64, device=dev)
    if report is not None:
        local = torch.tensor(report.rank_trace, dtype=torch.int64, device=dev)
        cols[:, torch.tensor(mine, dtype=torch.int64, device=dev)] = local
    dist.all_reduce(cols, op=dist.ReduceOp.SUM, group=group)
    full_trace = cols.cpu().tolist()

    final = None
    if gather:
        final = _gather_generators(report, mine, shards, n, dev, group)
    if report is None:
        from .engine import Mode, RunReport

        report = RunReport(Mode.coerce(mode), n, None, [], {}, {}, 0, 0, [])
    report.rank_trace = full_trace
    if gather:
        report.final = final
    return report, shards


def run_slot_partitioned(instructions, n: int, mode, eps: float = 1e-12, *, group=None, runner=None, **run_kw):
    """One circuit, every rank evolves all generators up to the LAST branching operator (cheap:
    the rank grows geometrically, so the last operator is nearly all of the work) and then works
    off its own contiguous range of that operator's output slots -- no data-path collective, and
    the split is even however skewed the generators are (xyz_chain(16,2): generator 0 alone holds
    a third of the terms, which caps generator sharding at 3x).

    Returns this rank's RunReport: ``rank_trace`` is global (the shares' counts are all-reduced),
    ``final.generators[j]`` is this rank's share of generator j in canonical order (shares of
    different ranks are disjoint; their union is the generator) unless
    ``report.device['partitioned']`` is False (the operator did not qualify for the grouped path;
    every rank then holds the complete result).
    """
    import torch

    from .errors import NumericalCollapseError

    dist = _dist()
    if runner is None:
        from .engine import run as runner
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = _comm_device(group)
    # No collective inside the run: a rank that fails (out of memory, ...) would otherwise leave
    # the others waiting in it.  The shares' counts are summed afterwards, behind an agreement
    # on errors, and the trace rows the share filled in are patched with the global ranks.
    report, failure = None, None
    try:
        report = runner(instructions, n, mode, eps, slot_part=(rank, world), slot_reduce=None, **run_kw)
    except Exception as exc:
        failure = exc
    agree_on_errors(failure, group)
    rows = report.device.get("partition_rows") or []
    if report.device.get("partitioned") and rows:
        t = torch.tensor(report.rank_trace[rows[0]], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        total = t.cpu().tolist()
        for row in rows:
            report.rank_trace[row] = list(total)
        for g, r in enumerate(total):
            if r == 0:
                raise NumericalCollapseError(
                    f"all terms of generator {g} dropped at operator step {report.device.get('partition_step')}"
                )
    return report


def _gather_generators(report, mine, shards, n, dev, group):
    """All-gather of ragged (keys, lambdas) per generator as padded flat tensors."""
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    gens = report.final.generators if report is not None else []
    sizes = torch.zeros(n, dtype=torch.int64, device=dev)
    for gi, g in zip(mine, gens):
        sizes[gi] = g.rank
    dist.all_reduce(sizes, op=dist.ReduceOp.SUM, group=group)
    sizes_h = sizes.cpu().tolist()
    per_rank = [sum(sizes_h[g] for g in s) for s in shards]
    width = max(per_rank + [1])
    keys = torch.zeros(width, dtype=torch.int64, device=dev)
    lam = torch.zeros(width, dtype=torch.float64, device=dev)
    at = 0
    for g in gens:
        k = torch.from_numpy(g.keys().view(np.int64).copy())
        keys[at:at + g.rank] = k.to(dev)
        lam[at:at + g.rank] = torch.from_numpy(np.ascontiguousarray(g.lambdas)).to(dev)
        at += g.rank
    all_keys = [torch.empty_like(keys) for _ in range(world)]
    all_lam = [torch.empty_like(lam) for _ in range(world)]
    dist.all_gather(all_keys, keys, group=group)
    dist.all_gather(all_lam, lam, group=group)
    out = [None] * n
    for r, shard in enumerate(shards):
        kk = all_keys[r].cpu().numpy().view(np.uint64)
        ll = all_lam[r].cpu().numpy()
        at = 0
        for g in shard:
            m = sizes_h[g]
            out[g] = SimpleGenerator(n, ll[at:at + m].copy(), keys_to_indices(kk[at:at + m].copy(), n))
            at += m
    return GeneratorSet(n, out)


# --------------------------------------------------------------------------------------
# term hash-partition: the all-to-all-v
# --------------------------------------------------------------------------------------
def exchange_partitioned(keys, lam, send_counts, group=None):
    """All-to-all-v of terms already grouped [destination rank][segment].

    keys (int64 view of the uint64 words) and lam (float64) are flat tensors on the
    communication device; ``send_counts[r, s]`` = terms of segment s going to rank r.
    Returns (recv_keys, recv_lam, recv_counts) with the received terms grouped
    [source rank][segment] -- the layout ``qx_store_assemble`` consumes.
    """
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    dev = keys.device
    sc = torch.as_tensor(np.ascontiguousarray(send_counts), dtype=torch.int64).to(dev)
    assert sc.shape[0] == world
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)              # row q of rc = what rank q sends me
    in_split = sc.sum(dim=1).cpu().tolist()
    out_split = rc.sum(dim=1).cpu().tolist()
    recv_keys = torch.empty(int(sum(out_split)), dtype=keys.dtype, device=dev)
    recv_lam = torch.empty(int(sum(out_split)), dtype=lam.dtype, device=dev)
    total = int(sum(in_split))
    dist.all_to_all_single(recv_keys, keys[:total], out_split, in_split, group=group)
    dist.all_to_all_single(recv_lam, lam[:total], out_split, in_split, group=group)
    return recv_keys, recv_lam, rc.cpu().numpy()


class _DeviceArray:
    """Zero-copy torch view of a raw device pointer (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": typestr, "data": (int(ptr), False), "version": 2, "strides": None,
        }


def exchange_terms(store, group=None):
    """Re-home the store's terms by owner: device partition -> all-to-all-v over NCCL -> assemble.

    After this call every key lives on exactly one rank, so a local ``merge`` is a global
    merge.  No host copy of any term is made.
    """
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    counts = store.partition_by_owner(world)
    total = int(counts.sum())
    d_keys, d_lam, _ = store.device_view()
    dev = torch.device("cuda", store.device)
    if total:
        keys = torch.as_tensor(_DeviceArray(d_keys, total, "<i8"), device=dev)
        lam = torch.as_tensor(_DeviceArray(d_lam, total, "<f8"), device=dev)
    else:
        keys = torch.empty(0, dtype=torch.int64, device=dev)
        lam = torch.empty(0, dtype=torch.float64, device=dev)
    if _comm_device(group).type == "cpu":
        # gloo (tests: several ranks sharing one GPU): the collective runs on host copies
        rk, rl, recv_counts = exchange_partitioned(keys.cpu(), lam.cpu(), counts, group)
        recv_keys, recv_lam = rk.to(dev), rl.to(dev)
    else:
        recv_keys, recv_lam, recv_counts = exchange_partitioned(keys, lam, counts, group)
    torch.cuda.current_stream(dev).synchronize()
    store.assemble(recv_keys.data_ptr(), recv_lam.data_ptr(), recv_counts)
    return recv_counts


def run_term_partitioned(instructions, n: int, mode, eps: float = 1e-12, *, group=None, device=None,
                         gather: bool = True):
    """Whole circuit with every generator's terms hash-partitioned over the ranks."""
    import torch

    from .engine import run

    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)

    def before_merge(store):
        exchange_terms(store, group)

    def global_ranks(local_ranks):
        dev = _comm_device(group)
        t = torch.tensor(local_ranks, dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.cpu().tolist()

    # rank 0 starts with all Z_j, the others start empty: the first exchange spreads them
    initial = None
    if rank != 0:
        initial = [(np.zeros(0), np.zeros(0, dtype=np.uint64)) for _ in range(n)]
    report = run(instructions, n, mode, eps, device=device, initial=initial,
                 before_merge=before_merge, reduce_ranks=global_ranks, download=True)
    if gather:
        report.final = _gather_partitioned(report.final, n, group)
    return report


def _gather_partitioned(final, n, group):
    """Union of the per-rank sorted parts of every generator, re-sorted by key on the host."""
    dist = _dist()
    world = dist.get_world_size(group)
    parts = [None] * world
    payload = [(g.lambdas, g.keys()) for g in final.generators]
    dist.all_gather_object(parts, payload, group=group)
    out = []
    for g in range(n):
        lam = np.concatenate([parts[r][g][0] for r in range(world)])
        keys = np.concatenate([parts[r][g][1] for r in range(world)])
        order = np.argsort(keys, kind="stable")
        out.append(SimpleGenerator(n, lam[order], keys_to_indices(keys[order], n)))
    return GeneratorSet(n, out)


# ------------------------------------------------------------------------------------
# read-out, observable-parallel
# ------------------------------------------------------------------------------------
def expectation_sharded(instructions, n: int, words, mode="v1", eps: float = 1e-12, *, group=None,
                        evaluator=None, **kw) -> np.ndarray:
    """<psi|W|psi> for every word of ``words`` on every rank; rank r evaluates words r, r + world, ...

    The words never interact (each is pushed back through the inverse circuit on its own,
    ``measure.expectation_heisenberg``), so the only collective is the final all-reduce of
    len(words) float64 scalars -- the read-out reduction BASELINE.json's north star names.
    ``evaluator(instructions, n, words, mode, eps)`` defaults to ``expectation_heisenberg``.
    """
    import torch

    dist = _dist()
    if evaluator is None:
        from .measure import expectation_heisenberg as evaluator
    words = [int(w) for w in words]
    for w in words:
        if not 0 <= w < 4 ** n:
            raise ValueError(f"word index {w} out of range [0, 4**{n})")
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = list(range(rank, len(words), world))
    out = np.zeros(len(words), dtype=np.float64)
    if mine:
        out[mine] = np.asarray(evaluator(instructions, n, [words[i] for i in mine], mode, eps, **kw),
                               dtype=np.float64)
    if len(words):
        t = torch.from_numpy(out).to(_comm_device(group))
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        out = t.cpu().numpy()
    return out


def prob_z_sharded(instructions, n: int, mode="v1", eps: float = 1e-12, *, group=None, evaluator=None,
                   **kw) -> np.ndarray:
    """(n, 2) array of (p0, p1) for every qubit: p0 = (1 + <Z_k>) / 2, the same number the
    reference reads from the expansion (measure.py:94-111: p0 = 1/2 + 2^(n-1) coeff(Z_k), and
    <Z_k> = 2^n coeff(Z_k)), with its consistency check and clamp."""
    from .errors import ConsistencyError

    z = expectation_sharded(instructions, n, [3 * 4 ** (n - 1 - k) for k in range(n)], mode, eps,
                            group=group, evaluator=evaluator, **kw)
    p0 = 0.5 + 0.5 * z
    for k, p in enumerate(p0):
        if not -1e-10 <= p <= 1.0 + 1e-10:
            raise ConsistencyError(f"probability {p} for qubit {k} outside [0, 1]")
    p0 = np.clip(p0, 0.0, 1.0)
    return np.stack([p0, 1.0 - p0], axis=1)
