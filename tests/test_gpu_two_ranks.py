"""The multi-GPU drivers with TWO REAL RANKS and the real CUDA library.  This pool gives one GPU
per call, so both ranks share cuda:0 and the collectives run over gloo (NCCL refuses two ranks on
one device); everything else is the production path: generator shards by LPT, the hash partition
+ all-to-all-v + assemble of the term-partitioned run, bucket ranges of the slot-partitioned run,
the observable-parallel read-out.  Each rank compares what it gets with the plain single-store
run of the same circuit: term sets always identical; coefficients bit for bit, except where terms
of one key arrive from different ranks (term partition: the sum runs over the sources in rank
order, equal to rounding)."""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, os.path.join(HERE, ".."))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2505_03307_b200 as qx
        from paper_2505_03307_b200 import _native
        from paper_2505_03307_b200 import dist as qd
        from paper_2505_03307_b200 import workloads

        def same(a, b, tol=0.0):
            assert a.rank_trace == b.rank_trace, name
            for ga, gb in zip(a.final.generators, b.final.generators):
                assert np.array_equal(ga.keys(), gb.keys())
                if tol:
                    assert np.max(np.abs(ga.lambdas - gb.lambdas), initial=0.0) < tol
                else:
                    assert np.array_equal(ga.lambdas, gb.lambdas), (name, mode)

        log = []
        for name, mode in (("c2_10q_near_clifford", "v1"), ("c2_10q_near_clifford", "v3"), ("c4_xyz_8_4", "v3"),
                           ("c5_32q_clifford_t", "v3")):
            n, gates = workloads.build(name)
            plain = qx.run(gates, n, mode, device=0)
            # ---- generators sharded (LPT on the final ranks), gathered on every rank
            sharded, shards = qd.run_sharded(gates, n, mode, weights=[g.rank for g in plain.final.generators],
                                             device=0)
            assert sorted(g for s in shards for g in s) == list(range(n)) and all(len(s) for s in shards)
            # a shard's operator step may take another summation path than the full store's (raw
            # expansion / grouped / factored sums are chosen from the sizes of the whole store):
            # equal to rounding on the deep ansatz, bit for bit elsewhere
            same(sharded, plain, tol=1e-12 if name == "c4_xyz_8_4" else 0.0)
            # ---- terms hash-partitioned: all-to-all-v before every merge that follows a branching step
            if name != "c5_32q_clifford_t":
                part = qd.run_term_partitioned(gates, n, mode, device=0)
                same(part, plain, tol=1e-12)
            log.append(name + ":" + mode)
        # ---- one circuit, the last operator's buckets split over the ranks, no data-path collective
        for name in ("c4_xyz_12_2", "c4_xyz_10_3"):
            n, gates = workloads.build(name)
            plain = qx.run(gates, n, "v3", device=0)
            rep = qd.run_slot_partitioned(gates, n, "v3", device=0)
            assert rep.device["partitioned"] is True and rep.rank_trace == plain.rank_trace
            np.savez(os.path.join(out_dir, f"share_{name}_{rank}.npz"),
                     **{f"k{j}": g.keys() for j, g in enumerate(rep.final.generators)},
                     **{f"l{j}": g.lambdas for j, g in enumerate(rep.final.generators)})
            if rank == 0:
                np.savez(os.path.join(out_dir, f"plain_{name}.npz"),
                         **{f"k{j}": g.keys() for j, g in enumerate(plain.final.generators)},
                         **{f"l{j}": g.lambdas for j, g in enumerate(plain.final.generators)})
            log.append(name + f":bucketed={_native.bucket_last()['cap'] > 0}")
        # ---- read-out, observable-parallel: every rank ends with all scalars
        n, gates = workloads.build("c1_4q_clifford_t")
        final = qx.run(gates, n, "v3", device=0).final
        ex = qx.density_expansion(final, device=0)
        got = qd.expectation_sharded(gates, n, range(4 ** n), device=0)
        want = np.array([qx.expectation(final, w, ex) for w in range(4 ** n)])
        assert np.max(np.abs(got - want)) < 1e-10
        with open(os.path.join(out_dir, f"ok_{rank}.txt"), "w") as fh:
            fh.write("\n".join(log))
    finally:
        dist.destroy_process_group()


def test_two_real_ranks_share_one_gpu(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"ok_{r}.txt").exists()
    # the shares of the slot-partitioned run: disjoint key ranges whose union is the plain result
    for name, n in (("c4_xyz_12_2", 12), ("c4_xyz_10_3", 10)):
        plain = np.load(tmp_path / f"plain_{name}.npz")
        shares = [np.load(tmp_path / f"share_{name}_{r}.npz") for r in range(world)]
        for j in range(n):
            keys = np.concatenate([s[f"k{j}"] for s in shares])
            lam = np.concatenate([s[f"l{j}"] for s in shares])
            order = np.argsort(keys, kind="stable")
            assert np.array_equal(keys[order], plain[f"k{j}"]) and np.array_equal(lam[order], plain[f"l{j}"])
