"""Generate tests/golden/wide.json: circuits on MORE than 32 qubits run by the UNMODIFIED reference
(Python big-int indices, stabilizer.py:40-59) in this container.

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_wide.py

The numpy oracle port keeps uint64 keys (n <= 32), so parity of the multi-word device path
(csrc/wide.cu) is pinned directly on what the reference computes: Clifford circuits (rank 1 per
generator at any width), near-Clifford circuits in v1 and v3 (a few T gates), Clifford circuits through the
operator pipeline (v3, every U_k a signed permutation), and the apply_cx big-int unit case of the
reference's own tests (tests/test_stabilizer.py:262-267).
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

from stabsim import circuit as rc                # noqa: E402  (the reference)
from stabsim import engine as reng               # noqa: E402
from stabsim import stabilizer as rstab          # noqa: E402

from paper_2505_03307_b200 import workloads      # noqa: E402  (only to name the same circuits)

CLIFFORD = ("H", "S", "X", "SX", "CX")


def near_clifford(n, m, t, seed):
    rng = np.random.default_rng(seed)
    base = workloads.gen_random(n, m - t, rng, gates=CLIFFORD)
    where = np.sort(rng.integers(0, len(base) + 1, size=t))
    wires = rng.integers(0, n, size=t)
    for k in reversed(range(t)):
        base.insert(int(where[k]), workloads.ir.rz(int(wires[k]), math.pi / 4))
    return base


def case(name, n, gates, mode):
    rep = reng.run([rc.Instruction(g.gate, tuple(g.wires), g.theta) for g in gates], n, mode)
    return {
        "name": name, "n": n, "mode": mode,
        "gates": [[g.gate, list(g.wires), float(g.theta).hex()] for g in gates],
        "rank_trace_last": [int(v) for v in rep.rank_trace[-1]],
        "max_rank": int(rep.max_rank),
        "final": [{"lam": [float(v).hex() for v in g.lambdas], "idx": [str(int(v)) for v in g.indices]}
                  for g in rep.final.generators],
    }


def main():
    cases = []
    for n in (33, 40, 64, 100):
        cases.append(case(f"ghz_{n}", n, workloads.gen_ghz(n), "v1"))
    cases.append(case("ghz_64_v3", 64, workloads.gen_ghz(64), "v3"))
    cases.append(case("ring_48", 48, workloads.gen_graph(48, workloads.ring_edges(48)), "v1"))
    for n, m, seed in ((40, 400, 11), (64, 600, 12), (130, 500, 13)):
        gates = workloads.gen_random(n, m, np.random.default_rng(seed), gates=CLIFFORD)
        cases.append(case(f"clifford_{n}_v1", n, gates, "v1"))
        cases.append(case(f"clifford_{n}_v3", n, gates, "v3"))
    for n, m, t, seed in ((34, 300, 6, 21), (40, 500, 8, 22), (64, 400, 7, 23)):
        cases.append(case(f"near_clifford_{n}_t{t}", n, near_clifford(n, m, t, seed), "v1"))
    # the same kind of circuit through the operator pipeline: branching U_k on big-int indices
    for n, m, t, seed in ((34, 300, 6, 21), (40, 500, 8, 22), (70, 300, 9, 24)):
        cases.append(case(f"near_clifford_{n}_t{t}_v3", n, near_clifford(n, m, t, seed), "v3"))
    # unit: CX on a 40-qubit word (reference tests/test_stabilizer.py:262-267 style)
    n = 40
    g = rstab.SimpleGenerator(n, np.array([1.0, -0.5]), [4 ** 39 + 3, 2 * 4 ** 39 + 4 ** 20])
    out = rstab.apply_cx(g, 0, 39)
    unit = {"n": n, "c": 0, "t": 39, "in": {"lam": [1.0, -0.5], "idx": [str(4 ** 39 + 3), str(2 * 4 ** 39 + 4 ** 20)]},
            "out": {"lam": [float(v) for v in out.lambdas], "idx": [str(int(v)) for v in out.indices]}}
    path = os.path.join(ROOT, "tests", "golden", "wide.json")
    with open(path, "w") as fh:
        json.dump({"_meta": {"reference": "stabsim 0.1.0"}, "data": {"cases": cases, "apply_cx": unit}}, fh)
    print("wrote", path, os.path.getsize(path), "bytes;", len(cases), "cases; max ranks",
          {c["name"]: c["max_rank"] for c in cases})


if __name__ == "__main__":
    main()
