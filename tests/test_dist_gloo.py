"""Host-side multi-GPU logic on CPU: world_size 2, gloo backend.

The compute kernels need a GPU, so the per-rank ``runner`` is replaced by a fake that answers
from the CPU oracle (test infrastructure); what is under test is the plumbing that has no GPU
in it: LPT sharding, gathering rank traces and ragged generators, and the all-to-all-v of
hash-partitioned terms with its [source][segment] layout contract."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_runner(instructions, n, mode, eps=1e-12, *, generators=None, **kw):
    """engine.run look-alike backed by the oracle (only for exercising dist.py on CPU)."""
    import stabsim_port as port

    from paper_2505_03307_b200.engine import Mode, RunReport, _Shard
    from paper_2505_03307_b200.stabilizer import SimpleGenerator, keys_to_indices

    res = port.run(instructions, n, mode, eps, generators=generators)
    gens = [SimpleGenerator(n, lam, keys_to_indices(idx, n)) for lam, idx in res["final"]]
    return RunReport(Mode.coerce(mode), n, _Shard(n, list(generators), gens), res["rank_trace"], {},
                     res["counters"], res["k"], res["k_prime"], res["order"])


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import stabsim_port as oracle

        from paper_2505_03307_b200 import dist as qd
        from paper_2505_03307_b200 import workloads

        # ---- generator-sharded run, LPT on skewed weights
        n, gates = 8, workloads.gen_xyz_chain(8, 2, 1, 4)
        weights = [4 ** (n - g) for g in range(n)]
        report, shards = qd.run_sharded(gates, n, "v3", weights=weights, runner=_fake_runner)
        assert sorted(g for s in shards for g in s) == list(range(n))
        want = oracle.run(gates, n, "v3")
        assert report.rank_trace == want["rank_trace"]
        for g, (lam, idx) in zip(report.final.generators, want["final"]):
            assert np.array_equal(g.keys(), idx) and np.array_equal(g.lambdas, lam)

        # ---- more ranks than generators with work: an empty shard must not deadlock
        report, shards = qd.run_sharded(workloads.gen_ghz(1) if False else [], 1, "v1", runner=_fake_runner)
        assert report.rank_trace == [[1]] and int(report.final.generators[0].indices[0]) == 3

        # ---- slot-partitioned run: the runner gets (rank, world) and does NO collective; the fake
        # answers with an index-range share of the oracle's result (what the device's bucket
        # ranges amount to) and names the trace rows that hold its share's counts; the driver sums
        # them over the ranks behind an agreement on errors
        def _slot_runner(instructions, n, mode, eps=1e-12, *, slot_part=None, slot_reduce=None, **kw):
            from paper_2505_03307_b200.engine import Mode, RunReport, _Shard
            from paper_2505_03307_b200.stabilizer import SimpleGenerator, keys_to_indices

            assert slot_reduce is None
            part, parts = slot_part
            res = oracle.run(instructions, n, mode, eps)
            gens, local = [], []
            for lam, idx in res["final"]:
                sel = np.arange(len(idx)) % parts == part
                gens.append(SimpleGenerator(n, lam[sel], keys_to_indices(idx[sel], n)))
                local.append(int(sel.sum()))
            trace = res["rank_trace"][:-1] + [local]
            return RunReport(Mode.coerce(mode), n, _Shard(n, list(range(n)), gens), trace, {}, res["counters"],
                             res["k"], res["k_prime"], res["order"],
                             {"partitioned": True, "partition_rows": [len(trace) - 1], "partition_step": len(trace) - 2})

        rep = qd.run_slot_partitioned(gates, n, "v3", runner=_slot_runner)
        assert rep.rank_trace == want["rank_trace"] and rep.device["partitioned"] is True
        mine = sum(g.rank for g in rep.final.generators)
        t = torch.tensor([mine], dtype=torch.int64)
        dist.all_reduce(t)
        assert int(t.item()) == sum(want["rank_trace"][-1])

        # ---- a failure on ONE rank reaches every rank instead of leaving the others in a collective
        def _failing_runner(instructions, n, mode, eps=1e-12, **kw):
            if rank == 1:
                raise ResourceLimitError("out of memory on this rank only")
            return _slot_runner(instructions, n, mode, eps, **kw)

        from paper_2505_03307_b200.errors import ResourceLimitError

        with pytest.raises((ResourceLimitError, qd.RemoteRankError)) as caught:
            qd.run_slot_partitioned(gates, n, "v3", runner=_failing_runner)
        assert (caught.type is ResourceLimitError) == (rank == 1)
        assert rank == 1 or "rank 1 failed with ResourceLimitError" in str(caught.value)

        def _failing_shard(instructions, n, mode, eps=1e-12, *, generators=None, **kw):
            if 0 in generators:
                raise ResourceLimitError("this shard ran out of memory")
            return _fake_runner(instructions, n, mode, eps, generators=generators, **kw)

        with pytest.raises((ResourceLimitError, qd.RemoteRankError)):
            qd.run_sharded(gates, n, "v3", weights=weights, runner=_failing_shard)

        # ---- observable-parallel read-out: words dealt round-robin, one all-reduce of the scalars
        n5, circ = 5, workloads.gen_random(5, 40, 11)
        words = [0, 3, 4 ** 5 - 1] + [int(v) for v in np.random.default_rng(5).integers(0, 4 ** 5, size=14)]
        seen = []

        def _evaluator(instructions, n, ws, mode, eps):
            seen.extend(ws)
            return oracle.expectation_heisenberg(instructions, n, ws, mode, eps)

        got = qd.expectation_sharded(circ, n5, words, "v1", evaluator=_evaluator)
        assert seen == words[rank::world]                       # this rank evaluated only its share
        assert np.array_equal(got, oracle.expectation_heisenberg(circ, n5, words, "v1"))
        assert len(qd.expectation_sharded(circ, n5, [], evaluator=_evaluator)) == 0
        pz = qd.prob_z_sharded(circ, n5, evaluator=_evaluator)
        final = oracle.run(circ, n5, "v3")["final"]
        ex = oracle.density_expansion(final, n5)
        for k in range(n5):
            assert abs(pz[k, 0] - oracle.prob_z(final, n5, k, ex)[0]) < 1e-10 and pz[k, 0] + pz[k, 1] == 1.0
        with pytest.raises(ValueError):
            qd.expectation_sharded(circ, n5, [4 ** 5], evaluator=_evaluator)

        # ---- all-to-all-v of hash-partitioned terms
        rng = np.random.default_rng(100 + rank)
        n_seg = 3
        segs = [rng.integers(0, 4 ** 10, size=s, dtype=np.uint64) for s in (50 + 7 * rank, 0, 400)]
        lams = [rng.uniform(-1, 1, size=len(k)) for k in segs]
        counts = np.zeros((world, n_seg), dtype=np.int64)
        send_k, send_l = [], []
        for r in range(world):                      # what the device partition kernel produces
            for s in range(n_seg):
                sel = qd.owner_of(segs[s], world) == r
                counts[r, s] = int(sel.sum())
                send_k.append(segs[s][sel])
                send_l.append(lams[s][sel])
        keys = torch.from_numpy(np.concatenate(send_k).view(np.int64))
        lam = torch.from_numpy(np.concatenate(send_l))
        rk, rl, rc = qd.exchange_partitioned(keys, lam, counts)
        assert rc.shape == (world, n_seg) and int(rc.sum()) == len(rk) == len(rl)
        got = rk.numpy().view(np.uint64)
        assert np.all(qd.owner_of(got, world) == rank)          # I only hold what I own
        np.save(os.path.join(out_dir, f"sent_{rank}.npy"), np.concatenate(segs))
        np.save(os.path.join(out_dir, f"recv_{rank}.npy"), got)
        np.save(os.path.join(out_dir, f"rc_{rank}.npy"), rc)
        np.save(os.path.join(out_dir, f"sc_{rank}.npy"), counts)
    finally:
        dist.destroy_process_group()


def test_world2_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    sent = np.concatenate([np.load(tmp_path / f"sent_{r}.npy") for r in range(world)])
    recv = np.concatenate([np.load(tmp_path / f"recv_{r}.npy") for r in range(world)])
    assert sorted(sent.tolist()) == sorted(recv.tolist())        # nothing lost, nothing duplicated
    for r in range(world):                                        # recv_counts[q] on r == send_counts[r] on q
        rc = np.load(tmp_path / f"rc_{r}.npy")
        for q in range(world):
            assert np.array_equal(rc[q], np.load(tmp_path / f"sc_{q}.npy")[r])


def test_lpt_shards_balance():
    from paper_2505_03307_b200.dist import lpt_shards, owner_of

    ranks = [41737064, 55284529, 18866855, 6353359, 2125649, 708223, 236205, 78732, 26253, 8757, 2925, 981,
             333, 117, 45, 12]                                    # xyz_chain(16, 2) final ranks
    for world in (1, 2, 4, 8):
        shards = lpt_shards(ranks, world)
        assert sorted(g for s in shards for g in s) == list(range(16))
        loads = [sum(ranks[g] for g in s) for s in shards]
        assert max(loads) <= max(max(ranks), sum(ranks) / world * 1.34)
    assert lpt_shards([1, 1, 1], 5)[3:] == [[], []]
    keys = np.arange(100000, dtype=np.uint64) * np.uint64(2654435761)
    share = np.bincount(owner_of(keys, 8), minlength=8) / len(keys)
    assert np.all(np.abs(share - 0.125) < 0.01)
