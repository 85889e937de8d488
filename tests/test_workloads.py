"""workloads.py draws the same circuits as the reference's generators (same seeds)."""

import numpy as np
import pytest

from paper_2505_03307_b200 import circuit as ir
from paper_2505_03307_b200 import workloads as wl


def _same(mine, rows):
    assert len(mine) == len(rows)
    for g, (name, wires, theta) in zip(mine, rows):
        assert g.gate == name and list(g.wires) == wires
        assert g.theta == float.fromhex(theta)          # bit-exact angles


def test_reference_generators_reproduced(golden):
    ref = golden.load_json("circuits.json")["_reference_generators"]
    _same(wl.gen_ghz(5), ref["ghz_5"]["gates"])
    _same(wl.gen_graph(6, wl.ring_edges(6)), ref["graph_ring_6"]["gates"])
    _same(wl.gen_xyz_chain(4, 4, 2, 1), ref["xyz_4_4_2_seed1"]["gates"])
    _same(wl.gen_xyz_chain(16, 2, 1, 4), ref["xyz_16_2_1_seed4"]["gates"])
    _same(wl.gen_random(5, 40, 9), ref["random_5_40_seed9"]["gates"])
    _same(wl.gen_random(16, 984, np.random.default_rng(3), wl.CLIFFORD_POOL),
          ref["random_clifford_16_984_seed3"]["gates"])


@pytest.mark.parametrize("name,n,m,t", [
    ("c1_4q_clifford_t", 4, 11, 2), ("c2_10q_near_clifford", 10, 200, 10),
    ("c3_16q_clifford", 16, 1000, 0), ("c5_32q_clifford_t", 32, 5000, 20),
])
def test_baseline_config_shapes(golden, name, n, m, t):
    nq, gates = wl.build(name)
    assert nq == n and len(gates) == m
    assert sum(g.gate == "RZ" for g in gates) == t
    _same(gates, golden.load_json("circuits.json")[name]["gates"])


def test_xyz_gate_count():
    for n, layers, reps in ((4, 3, 5), (16, 2, 1)):
        assert len(wl.gen_xyz_chain(n, layers, reps, 0)) == layers * (3 * n * reps + n - 1)


def test_partition_alternates_and_replays():
    n, gates = wl.build("c2_10q_near_clifford")
    part = ir.divide_instruction(gates, n)
    assert part.order == ir.create_chain(part.k, part.k_prime, part.order[0] == 0)
    assert sum(part.operator_sizes()) == len(gates)
    assert (part.k, part.k_prime) == (34, 34)
    assert sorted(map(repr, part.replay())) == sorted(map(repr, gates))


def test_instruction_validation():
    with pytest.raises(ValueError):
        ir.Instruction("T", (0,))                             # reference tests/test_circuit.py:26-28
    with pytest.raises(ValueError):
        ir.Instruction("CX", (1, 1))
    with pytest.raises(ValueError):
        ir.Instruction("H", (0,), 0.5)
    with pytest.raises(ValueError):
        ir.Instruction("RX", (-1,), 0.5)
    with pytest.raises(ValueError):
        ir.divide_instruction([ir.h(3)], 3)
    with pytest.raises(ValueError):
        ir.create_chain(3, 1, True)
    assert ir.create_chain(2, 1, True) == [0, 1, 0]
