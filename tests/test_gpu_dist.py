"""Multi-GPU code paths exercised on ONE GPU: world_size = 1 over NCCL (the only size this
environment can run).  Checks that the sharded and the term-partitioned drivers reproduce the
plain single-store run bit for bit, including the device-pointer all-to-all-v."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import qx  # noqa: E402

from paper_2505_03307_b200 import dist as qd  # noqa: E402
from paper_2505_03307_b200 import workloads  # noqa: E402


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def _same(a, b, tol=0.0):
    for ga, gb in zip(a.final.generators, b.final.generators):
        assert np.array_equal(ga.indices, gb.indices)
        if tol:
            assert np.max(np.abs(ga.lambdas - gb.lambdas)) < tol
        else:
            assert np.array_equal(ga.lambdas, gb.lambdas)
    assert a.rank_trace == b.rank_trace


@pytest.mark.parametrize("name,mode", [("c2_10q_near_clifford", "v1"), ("c2_10q_near_clifford", "v3"),
                                       ("c4_xyz_8_4", "v3")])
def test_sharded_and_partitioned_equal_plain(nccl_world1, name, mode):
    n, gates = workloads.build(name)
    plain = qx.run(gates, n, mode)
    sharded, shards = qd.run_sharded(gates, n, mode, weights=[g.rank for g in plain.final.generators])
    assert shards == [list(range(n))]
    _same(sharded, plain)
    part = qd.run_term_partitioned(gates, n, mode)
    # the partitioned run merges raw branch lists; the plain run sums groups with many sources in
    # factored form (dense.cu): same terms, coefficients equal to rounding
    _same(part, plain, tol=1e-12 if name.startswith("c4_") else 0.0)


def test_exchange_terms_loopback(nccl_world1):
    from paper_2505_03307_b200.store import DeviceStore

    rng = np.random.default_rng(9)
    n = 12
    gens = []
    for size in (3000, 0, 50_000):
        keys = rng.integers(0, 4 ** n, size=size, dtype=np.uint64)
        gens.append((rng.uniform(-1, 1, size=size), keys))
    with DeviceStore(n, 3, 0) as st:
        st.upload(gens)
        counts = qd.exchange_terms(st)
        assert counts.shape == (1, 3) and counts[0].tolist() == [3000, 0, 50_000]
        for (lam, keys), (gl, gk) in zip(gens, st.segments()):
            assert np.array_equal(gk, keys) and np.array_equal(gl, lam)     # world = 1: order kept


@pytest.mark.parametrize("name,parts", [("c4_xyz_12_2", 3), ("c4_xyz_10_3", 2)])
def test_slot_partition_shares_union_to_the_full_result(name, parts):
    """run(..., slot_part=(p, parts)): the shares of the parts are disjoint, canonical, and their
    union is the plain result -- checked here part by part on one GPU (what run_slot_partitioned
    does on `parts` GPUs, where only the share counts are all-reduced)."""
    n, gates = workloads.build(name)
    plain = qx.run(gates, n, "v3")
    shares = [qx.run(gates, n, "v3", slot_part=(p, parts)) for p in range(parts)]
    assert all(s.device["partitioned"] is True for s in shares)
    for j, g in enumerate(plain.final.generators):
        keys = np.concatenate([s.final.generators[j].keys() for s in shares])
        lam = np.concatenate([s.final.generators[j].lambdas for s in shares])
        for s in shares:
            k = s.final.generators[j].keys()
            assert np.all(k[1:] > k[:-1])                       # every share is canonical
        order = np.argsort(keys, kind="stable")
        assert np.array_equal(keys[order], g.keys()) and np.array_equal(lam[order], g.lambdas)
    assert [sum(col) for col in zip(*[s.rank_trace[-1] for s in shares])] == plain.rank_trace[-1]


def test_run_slot_partitioned_world1(nccl_world1):
    n, gates = workloads.build("c4_xyz_12_2")
    plain = qx.run(gates, n, "v3")
    rep = qd.run_slot_partitioned(gates, n, "v3")
    assert rep.rank_trace == plain.rank_trace
    for ga, gb in zip(rep.final.generators, plain.final.generators):
        assert np.array_equal(ga.keys(), gb.keys()) and np.array_equal(ga.lambdas, gb.lambdas)


def test_sharded_readout_equals_the_expansion_route(nccl_world1):
    """dist.expectation_sharded / prob_z_sharded (Heisenberg back-propagation per word, scalars
    all-reduced over NCCL) against the reference's route, the density expansion, on config 1:
    all 256 words and every qubit's probabilities."""
    n, gates = workloads.build("c1_4q_clifford_t")
    final = qx.run(gates, n, "v3").final
    ex = qx.density_expansion(final)
    got = qd.expectation_sharded(gates, n, range(4 ** n))
    want = np.array([qx.expectation(final, w, ex) for w in range(4 ** n)])
    assert np.max(np.abs(got - want)) < 1e-10
    pz = qd.prob_z_sharded(gates, n)
    for k in range(n):
        assert abs(pz[k, 0] - qx.prob_z(final, k, ex)[0]) < 1e-10
