"""Host side of the whole-circuit programs (engine._RecordingStore / _ReplayStore): the step list a
plan compiles to and the bookkeeping replay, without a GPU.  The reference chain it mirrors:
engine.py:110-132 (operators), :155-180 (gate by gate)."""

import numpy as np

import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import engine


def _steps(gates, n, mode):
    mode = engine.Mode.coerce(mode)
    plan = engine._Plan(gates, n)
    rec = engine._RecordingStore(n, n)
    w = engine._Walker(rec, n, range(n), 1e-12, {"partition": 0.0, "lut": 0.0, "sub_flatten": 0.0, "cx": 0.0})
    engine._walk_events(w, engine._program_events(plan, gates, mode), mode, [list(w.ranks)],
                        {"sub_flatten_ops": 0, "cx_applications": 0})
    return plan, rec.steps


def test_worked_circuit_compiles_to_one_branching_step():
    # SX(0), RZ(pi/3, 0), CX(0,1): reference tests/test_engine.py:38-68
    gates = [qx.Instruction("SX", (0,)), qx.Instruction("RZ", (0,), np.pi / 3), qx.Instruction("CX", (0, 1))]
    for mode in ("v1", "v3"):
        _, steps = _steps(gates, 3, mode)
        kinds = [s[0] for s in steps]
        assert kinds.count("oprun") == 1
        assert kinds[-1] == "oprun"                    # the CX run is folded into the operator step
        oprun = steps[kinds.index("oprun")]
        assert oprun[1] == (mode == "v3")              # the reference's string order only in v3
        assert len(oprun[5]) >= 1                      # ... the CX op word rides along


def test_clifford_circuit_compiles_to_run_and_sort():
    gates = qx.gen_ghz(5)
    for mode in ("v1", "v3"):
        _, steps = _steps(gates, 5, mode)
        assert [s[0] for s in steps] == ["clifford", "sort"]


def test_replay_books_the_recorded_ranks():
    gates = [qx.Instruction("H", (0,)), qx.Instruction("RZ", (0,), 0.3), qx.Instruction("CX", (0, 1)),
             qx.Instruction("RX", (1,), 0.7)]
    n = 2
    plan, steps = _steps(gates, n, "v3")
    rows = [[2, 1], [3, 2]][: sum(1 for s in steps if s[0] == "oprun")]
    w = engine._Walker(engine._ReplayStore(rows, 0), n, range(n), 1e-12,
                       {"partition": 0.0, "lut": 0.0, "sub_flatten": 0.0, "cx": 0.0})
    trace = [list(w.ranks)]
    engine._walk_events(w, engine._program_events(plan, gates, engine.Mode.V3), engine.Mode.V3, trace,
                        {"sub_flatten_ops": 0, "cx_applications": 0})
    assert trace[0] == [1, 1] and trace[-1] == rows[-1]
    assert len(trace) == plan.partition.k + plan.partition.k_prime + 1     # reference tests/test_engine.py:77
    assert all(row is not None for row in trace)


class _FakeStore:
    """Counts what reaches the 'real' store behind a one-launch prefix."""

    mark = None

    def __init__(self, n_gen):
        self.n_gen, self.calls = n_gen, []

    def apply_clifford(self, program):
        self.calls.append(("clifford", len(program)))

    def order_for_operator(self, counts, by_key=True):
        self.calls.append(("order",))

    def apply_operator_run(self, counts, axes, weights, program, eps, term_limit=0):
        self.calls.append(("oprun", len(program)))
        return 7, [5] * self.n_gen

    def sort(self):
        self.calls.append(("sort",))


def test_prefix_store_hands_out_recorded_ranks_then_forwards():
    # three branching operators; the first two were one launch, the third goes to the real store
    gates = [qx.Instruction("H", (0,)), qx.Instruction("RZ", (0,), 0.3), qx.Instruction("CX", (0, 1)),
             qx.Instruction("RX", (1,), 0.7), qx.Instruction("CX", (1, 0)), qx.Instruction("RY", (0,), 1.1),
             qx.Instruction("CX", (0, 1))]
    n = 2
    plan, steps = _steps(gates, n, "v3")
    kinds = [s[0] for s in steps]
    assert kinds.count("oprun") == 3
    done = kinds.index("oprun", kinds.index("oprun") + 1) + 1          # everything up to the second operator step
    rows = [[2, 1], [3, 2]]
    fake = _FakeStore(n)
    store = engine._PrefixStore(rows, done, fake)
    w = engine._Walker(store, n, range(n), 1e-12, {"partition": 0.0, "lut": 0.0, "sub_flatten": 0.0, "cx": 0.0})
    trace = [list(w.ranks)]
    engine._walk_events(w, engine._program_events(plan, gates, engine.Mode.V3), engine.Mode.V3, trace,
                        {"sub_flatten_ops": 0, "cx_applications": 0})
    assert store.seen == done and store.next == 2
    # only the third operator (with its source order) reached the real store
    assert [c[0] for c in fake.calls] == ["order", "oprun"]
    assert trace[-1] == [5, 5] and [2, 1] in trace and [3, 2] in trace
    assert w.launch_log["raw_terms"] == 7
