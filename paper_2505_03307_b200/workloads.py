"""Synthetic circuit families and the BASELINE.json workload table.

These are *input generators*, not part of the accelerated path (SURVEY.md
section 2, "OUT OF SCOPE (keep as-is)").  They draw from numpy's PCG64 in the
same call order as the reference's ``circuit.py:206-278`` so that a seed names
the same circuit on both sides; ``tests/test_workloads.py`` pins that against
circuits dumped from the reference (``tests/golden/circuits.json``).

``WORKLOADS`` names the five BASELINE.json configs the way SURVEY.md section 8d
resolves them (T == RZ(pi/4); config 4 as the (n, layers) ladder because
n=20, L=4 is infeasible for any exact method).
"""

from __future__ import annotations

import math
from typing import Iterable, Sequence

import numpy as np

from . import circuit as ir

TWO_PI = 2.0 * math.pi
CLIFFORD_POOL = ("H", "S", "X", "SX", "CX")


def _generator(rng):
    return rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)


def gen_ghz(n: int) -> list:
    """H(0) then CX(i, i+1): the GHZ preparation (reference circuit.py:206-210)."""
    if n < 1:
        raise ValueError(f"need at least one qubit, got {n}")
    return [ir.h(0), *(ir.cx(i, i + 1) for i in range(n - 1))]


def ring_edges(n: int) -> list:
    """Edges of the n-cycle (reference circuit.py:223-230)."""
    edges = [(i, i + 1) for i in range(max(n - 1, 0))] if n >= 2 else []
    if n > 2:
        edges.append((n - 1, 0))
    return edges


def gen_graph(n: int, edges: Iterable) -> list:
    """Graph state, CZ lowered to H-CX-H (reference circuit.py:213-220)."""
    out = [ir.h(q) for q in range(n)]
    for a, b in edges:
        if a == b or min(a, b) < 0 or max(a, b) >= n:
            raise ValueError(f"bad edge ({a}, {b}) for n={n}")
        out.extend((ir.h(b), ir.cx(a, b), ir.h(b)))
    return out


def gen_xyz_chain(n: int, layers: int, repeats: int, rng=None) -> list:
    """QNN-style ansatz: RX/RY/RZ columns then a CX ladder per layer.

    Angle draw order is (layer, repeat, axis, qubit) exactly as the reference
    (circuit.py:233-256), one ``uniform(0, 2*pi)`` per rotation.
    """
    if n < 2:
        raise ValueError(f"chain needs at least 2 qubits, got {n}")
    gen = _generator(rng)
    out = []
    for _layer in range(layers):
        for _rep in range(repeats):
            for make in (ir.rx, ir.ry, ir.rz):
                out.extend(make(q, gen.uniform(0.0, TWO_PI)) for q in range(n))
        out.extend(ir.cx(j, j + 1) for j in range(n - 1))
    return out


def gen_random(n: int, m: int, rng=None, gates: Sequence[str] = ir.ALL_GATES) -> list:
    """m gates drawn uniformly from ``gates`` (reference circuit.py:259-278).

    Draw order per gate: gate id; then for CX a 2-subset via ``choice``; for a
    rotation the wire and then the angle; otherwise the wire.
    """
    gen = _generator(rng)
    pool = [g for g in gates if not (g == "CX" and n < 2)]
    out = []
    for _ in range(m):
        name = pool[int(gen.integers(len(pool)))]
        if name == "CX":
            pair = gen.choice(n, size=2, replace=False)
            out.append(ir.cx(int(pair[0]), int(pair[1])))
            continue
        wire = int(gen.integers(n))
        theta = gen.uniform(0.0, TWO_PI) if name in ir.ROTATIONS else 0.0
        out.append(ir.Instruction(name, (wire,), theta))
    return out


def near_clifford(n: int, m: int, t: int, seed: int) -> list:
    """m-gate circuit with exactly t T gates, T lowered to RZ(pi/4) (SURVEY.md 8d helper)."""
    rng = np.random.default_rng(seed)
    base = gen_random(n, m - t, rng, gates=CLIFFORD_POOL)
    where = np.sort(rng.integers(0, len(base) + 1, size=t))
    wires = rng.integers(0, n, size=t)
    for k in reversed(range(t)):
        base.insert(int(where[k]), ir.rz(int(wires[k]), math.pi / 4))
    return base


def config1() -> tuple:
    """C1: 4-qubit Clifford+T, 11 gates."""
    t = math.pi / 4
    gates = [
        ir.h(0), ir.cx(0, 1), ir.rz(1, t), ir.s(2), ir.h(2), ir.cx(1, 2),
        ir.cx(2, 3), ir.rz(3, t), ir.h(3), ir.s(0), ir.cx(3, 0),
    ]
    return 4, gates


def config2() -> tuple:
    """C2: 10-qubit near-Clifford, 200 gates with 10 T."""
    return 10, near_clifford(10, 200, 10, seed=2)


def config3() -> tuple:
    """C3: 16-qubit pure Clifford, GHZ prefix + 984 random Clifford gates = 1000."""
    n = 16
    return n, gen_ghz(n) + gen_random(n, 984, np.random.default_rng(3), CLIFFORD_POOL)


def config4(n: int = 16, layers: int = 2, seed: int = 4) -> tuple:
    """C4 ladder point: xyz_chain(n, layers, repeats=1, rng=4). (16, 2) is the largest-rank config.
    ``seed`` other than 4 draws another instance of the same ansatz (multi-GPU weak scaling)."""
    return n, gen_xyz_chain(n, layers, 1, rng=seed)


def config5() -> tuple:
    """C5: 32-qubit Clifford+T, 5000 gates with 20 T."""
    return 32, near_clifford(32, 5000, 20, seed=5)


WORKLOADS = {
    "c1_4q_clifford_t": config1,
    "c2_10q_near_clifford": config2,
    "c3_16q_clifford": config3,
    "c4_xyz_8_4": lambda: config4(8, 4),
    "c4_xyz_10_3": lambda: config4(10, 3),
    "c4_xyz_12_2": lambda: config4(12, 2),
    "c4_xyz_14_2": lambda: config4(14, 2),
    "c4_xyz_16_2": lambda: config4(16, 2),
    "c4_xyz_18_2": lambda: config4(18, 2),
    "c4_xyz_20_2": lambda: config4(20, 2),      # ~1.0e10 terms, ~330 GB: beyond one GPU
    "c4_xyz_20_4": lambda: config4(20, 4),      # BASELINE config 4 as written: infeasible
    "c5_32q_clifford_t": config5,
}


def build(name: str, instance: int = 0) -> tuple:
    """(n, instructions) of a named workload.  ``instance`` > 0 draws another circuit of the same
    family and shape (config-4 ladder only: other rotation angles, same gates and wires)."""
    if instance and name.startswith("c4_xyz_"):
        n, layers = (int(v) for v in name.split("_")[2:4])
        return config4(n, layers, seed=4 + 1000 * instance)
    try:
        return WORKLOADS[name]()
    except KeyError:
        raise ValueError(f"unknown workload {name!r}; have {sorted(WORKLOADS)}") from None
