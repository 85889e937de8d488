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


def test_circuit_text_and_json_round_trip():
    """The reference's circuit file formats (circuit.py:281-352): lossless text round trip,
    comments and blank lines, the JSON array form, and line numbers in parse errors; checked
    against the reference's own parser/serializer on the circuits it dumped (golden)."""
    import json

    import pytest

    import paper_2505_03307_b200 as qx
    from paper_2505_03307_b200 import workloads

    for name in ("c1_4q_clifford_t", "c2_10q_near_clifford", "c4_xyz_8_4"):
        _, gates = workloads.build(name)
        text = qx.serialize_circuit(gates)
        assert qx.parse_circuit(text) == gates                   # angles survive bit for bit (repr)
        as_json = json.dumps([{"gate": g.gate, "wires": list(g.wires), "theta": g.theta} for g in gates])
        assert qx.parse_circuit("  " + as_json) == gates
    assert qx.serialize_circuit([]) == ""
    assert qx.serialize_circuit([qx.Instruction("CX", (0, 1)), qx.Instruction("RZ", (1,), 0.25)]) == "cx 0 1\nrz 1 0.25\n"
    parsed = qx.parse_circuit("# ghz\nH 0\n\ncx 0 1   # entangle\nrz 1 0.5\n")
    assert [g.gate for g in parsed] == ["H", "CX", "RZ"] and parsed[2].theta == 0.5
    for bad, line in (("h 0\nfoo 1\n", 2), ("cx 0\n", 1), ("rz 0\n", 1), ("h 0 0.3\n", 1), ("cx 1 1\n", 1),
                      ("rz a 0.1\n", 1), ("rx 0 abc\n", 1)):
        with pytest.raises(qx.CircuitParseError) as err:
            qx.parse_circuit(bad)
        assert err.value.line_no == line and str(err.value).startswith(f"line {line}: ")
    with pytest.raises(qx.CircuitParseError):
        qx.parse_circuit('[{"gate": "h"}]')
    with pytest.raises(qx.CircuitParseError):
        qx.parse_circuit("[1, 2")


def test_formats_match_the_reference_when_it_is_importable():
    """In the build container the reference itself is available: byte-identical serialization
    and identical parse results.  Skipped where /root/reference does not exist (GPU box)."""
    import os
    import sys

    import pytest

    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference tree not present")
    sys.path.insert(0, ref)
    try:
        from stabsim import circuit as rc
    finally:
        sys.path.remove(ref)
    import paper_2505_03307_b200 as qx
    from paper_2505_03307_b200 import workloads

    for name in ("c1_4q_clifford_t", "c4_xyz_8_4", "c5_32q_clifford_t"):
        _, gates = workloads.build(name)
        theirs = [rc.Instruction(g.gate, g.wires, g.theta) for g in gates]
        text = rc.serialize_circuit(theirs)
        assert qx.serialize_circuit(gates) == text
        assert [(g.gate, g.wires, g.theta) for g in qx.parse_circuit(text)] == \
               [(g.gate, g.wires, g.theta) for g in rc.parse_circuit(text)]
