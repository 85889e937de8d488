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
