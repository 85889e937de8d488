"""CPU-side checks of the class decomposition behind the grouped operator step (csrc/dense.cu),
through the host-only entry point qx_operator_classes, against the oracle's raw expansion:
terms with different class words never produce the same output word, and the raw outputs of a
group lie inside its box of prod_j radix_j slots."""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
import stabsim_port as oracle  # noqa: E402

import paper_2505_03307_b200 as qx  # noqa: E402
from paper_2505_03307_b200 import _native as nat, lut  # noqa: E402


def classes(n, block):
    counts, axes, weights = lut.operator_tables(block)
    counts = np.ascontiguousarray(counts, dtype=np.int32).reshape(-1)
    axes = np.ascontiguousarray(axes, dtype=np.int32).reshape(-1)
    weights = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
    cid = np.zeros(n * 3, dtype=np.int32)
    rad = np.zeros(n * 3, dtype=np.int32)
    cax = np.zeros(n * 9, dtype=np.int32)
    cwt = np.zeros(n * 9, dtype=np.float64)
    nat.check(nat.lib().qx_operator_classes(n, nat.ptr(counts), nat.ptr(axes), nat.ptr(weights), nat.ptr(cid),
                                            nat.ptr(rad), nat.ptr(cax), nat.ptr(cwt)))
    return cid.reshape(n, 3), rad.reshape(n, 3), cax.reshape(n, 3, 3), cwt.reshape(n, 3, 3)


def test_known_blocks():
    n = 4
    gates = [qx.Instruction("RZ", (0,), 0.4), qx.Instruction("H", (1,)), qx.Instruction("RX", (2,), 1.1),
             qx.Instruction("RX", (3,), 0.3), qx.Instruction("RY", (3,), 0.9), qx.Instruction("RZ", (3,), 2.0)]
    block = oracle.lut_blocks(oracle.partition(gates, n), n)[0]
    cid, rad, cax, cwt = classes(n, block)
    assert cid[0].tolist() == [1, 1, 3] and rad[0].tolist() == [2, 2, 1]       # RZ: {X,Y} mix, Z alone
    assert cid[1].tolist() == [1, 2, 3] and rad[1].tolist() == [1, 1, 1]       # H: a permutation
    assert cax[1, 0, 0] == 3 and cwt[1, 0, 0] == 1.0                            # X -> Z
    assert cid[2].tolist() == [1, 2, 2] and rad[2].tolist() == [1, 2, 2]       # RX: X alone, {Y,Z} mix
    assert cid[3].tolist() == [1, 1, 1] and rad[3].tolist() == [3, 3, 3]       # generic rotation
    # weights: row of the block restricted to the class's axes
    for a in range(3):
        assert np.array_equal(cwt[3, a], block[3, a])


@pytest.mark.parametrize("seed", range(6))
def test_groups_partition_the_collisions(seed):
    rng = np.random.default_rng(seed)
    n = 5
    names = ["RX", "RY", "RZ", "H", "S"]
    gates = []
    for q in range(n):
        for _ in range(int(rng.integers(0, 3))):
            g = str(rng.choice(names))
            gates.append(qx.Instruction(g, (q,), float(rng.uniform(0, 6.28)) if g.startswith("R") else 0.0))
    gates = gates or [qx.Instruction("RY", (0,), 0.5)]
    block = oracle.lut_blocks(oracle.partition(gates, n), n)[0]
    cid, rad, cax, _ = classes(n, block)
    keys = np.unique(rng.integers(0, 4 ** n, size=120, dtype=np.uint64))
    owner = {}          # output word -> class word of the terms that reach it
    for k in keys:
        digs = [int(oracle.digit(np.array([k], dtype=np.uint64), n, j)[0]) for j in range(n)]
        cw = tuple(0 if d == 0 else int(cid[j, d - 1]) for j, d in enumerate(digs))
        slots = 1
        allowed = []
        for j, d in enumerate(digs):
            if d:
                slots *= int(rad[j, d - 1])
                allowed.append(set(cax[j, d - 1, : rad[j, d - 1]].tolist()))
            else:
                allowed.append({0})
        _, raw = oracle.expand_operator(np.ones(1), np.array([k], dtype=np.uint64), n, block)
        assert len(set(raw.tolist())) == len(raw) <= slots
        for out in raw:
            od = [int(oracle.digit(np.array([out], dtype=np.uint64), n, j)[0]) for j in range(n)]
            assert all(o in allowed[j] for j, o in enumerate(od))            # inside the group's box
            assert owner.setdefault(int(out), cw) == cw                        # only its own group reaches it
