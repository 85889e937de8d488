"""Whole-circuit programs (csrc/program.cuh, qx_store_run_program): one launch per
run for circuits whose generators stay small, against the step-by-step replay of the same plan --
final generators bit for bit (keys and coefficients), rank trace, counters, v1 update counts, the
collapse error (reference engine.py:148-152: generator and step) -- and against the oracle.  Covers
every step kind (Clifford run, branching operator with and without the v3 source order, final
re-sort), the three modes, caller-supplied initial generators (read-out back-propagation), the
"did not fit" fallback and the BASELINE configs 1, 2, 3, 5."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from gpu_util import oracle, qx, report_gens  # noqa: E402

from paper_2505_03307_b200 import _native, engine, workloads  # noqa: E402
from paper_2505_03307_b200.errors import NumericalCollapseError  # noqa: E402


def _both(gates, n, mode, **kw):
    """(programmed run, step-by-step run) of the same circuit; asserts the first took one launch."""
    engine.clear_plans()
    engine._PROGRAMS_ON = True
    try:
        qx.run(gates, n, mode, **kw)                     # compiles the plan and its program
        before = _native.launch_count()
        a = qx.run(gates, n, mode, **kw)
        launches = _native.launch_count() - before
    finally:
        engine._PROGRAMS_ON = False
    try:
        engine.clear_plans()
        b = qx.run(gates, n, mode, **kw)
    finally:
        engine._PROGRAMS_ON = True
    return a, b, launches


def _same(a, b):
    assert a.rank_trace == b.rank_trace
    assert a.counters == b.counters
    assert a.device.get("updates_per_generator") == b.device.get("updates_per_generator")
    for (la, ka), (lb, kb) in zip(report_gens(a), report_gens(b)):
        assert np.array_equal(ka, kb)
        assert np.array_equal(la, lb)                    # bit for bit


@pytest.mark.parametrize("mode", ["v1", "v2", "v3"])
def test_random_circuits_one_launch_equals_step_by_step(mode):
    for case in range(40):
        rng = np.random.default_rng([77, case])
        n = int(rng.integers(2, 9))
        gates = qx.gen_random(n, int(rng.integers(1, 60)), rng)
        a, b, launches = _both(gates, n, mode)
        _same(a, b)
        assert "program_steps" in a.device and "program_steps" not in b.device
        assert launches <= 3, launches                   # the circuit kernel + the read-back kernel(s)
        want = oracle.run(gates, n, mode)
        assert a.rank_trace == want["rank_trace"]
        for (lam, keys), (wl, wk) in zip(report_gens(a), want["final"]):
            assert np.array_equal(keys, wk) and np.max(np.abs(lam - wl), initial=0.0) < 1e-10


@pytest.mark.parametrize("name", ["c1_4q_clifford_t", "c2_10q_near_clifford", "c3_16q_clifford", "c5_32q_clifford_t"])
@pytest.mark.parametrize("mode", ["v1", "v3"])
def test_baseline_configs_one_launch(name, mode):
    n, gates = workloads.build(name)
    a, b, launches = _both(gates, n, mode)
    _same(a, b)
    assert "program_steps" in a.device
    assert launches <= 3, launches


def test_v1_and_v3_bitwise_the_oracles_through_programs():
    for case in range(30):
        rng = np.random.default_rng([78, case])
        n = int(rng.integers(3, 8))
        gates = qx.gen_random(n, 40, rng)
        for mode in ("v1", "v3"):
            got = qx.run(gates, n, mode)
            assert "program_steps" in got.device
            want = oracle.run(gates, n, mode)
            for (lam, keys), (wl, wk) in zip(report_gens(got), want["final"]):
                assert np.array_equal(keys, wk) and np.array_equal(lam, wl)


def test_collapse_message_matches_step_by_step():
    # eps below the initial coefficient (no eager schedule) but above cos(pi/4): both branches of
    # the first rotation drop
    n = 3
    gates = [qx.Instruction("H", (0,)), qx.Instruction("CX", (0, 1)), qx.Instruction("RZ", (1,), np.pi / 4),
             qx.Instruction("H", (2,))]
    msgs = []
    for on in (True, False):
        engine.clear_plans()
        engine._PROGRAMS_ON = on
        try:
            for mode in ("v1", "v3"):
                with pytest.raises(NumericalCollapseError) as err:
                    qx.run(gates, n, mode, eps=0.8)
                msgs.append((on, mode, str(err.value)))
        finally:
            engine._PROGRAMS_ON = True
    assert [m for on, _, m in msgs if on] == [m for on, _, m in msgs if not on]
    want = None
    try:
        oracle.run(gates, n, "v3", eps=0.8)
    except Exception as exc:                              # the port raises the reference's message
        want = str(exc)
    assert want is not None and msgs[1][2] == want


@pytest.mark.parametrize("mode", ["v1", "v3"])
def test_a_circuit_that_outgrows_shared_memory_starts_with_one_launch(mode):
    """xyz_chain(8,2): the first operator steps fit one launch, a later one does not.  The first run
    finds that out (and replays everything step by step); from the second run on the steps in
    front are ONE launch and the walk goes on step by step behind them.  All three runs and the
    run without programs agree bit for bit."""
    n, gates = 8, qx.gen_xyz_chain(8, 2, 1, rng=4)
    engine.clear_plans()
    first = qx.run(gates, n, mode)
    assert "program_steps" not in first.device
    plan = engine._plan_for(gates, n, engine.Mode.coerce(mode))
    program = plan._programs[(engine.Mode.coerce(mode), first.device["device"])]
    assert program is not None and 0 < program.fit_steps < program.steps
    before = _native.launch_count()
    second = qx.run(gates, n, mode)
    launches_prefixed = _native.launch_count() - before
    assert second.device["program_steps"] == program.fit_steps
    third = qx.run(gates, n, mode)
    engine._PROGRAMS_ON = False
    try:
        engine.clear_plans()
        before = _native.launch_count()
        plain = qx.run(gates, n, mode)
        launches_plain = _native.launch_count() - before
    finally:
        engine._PROGRAMS_ON = True
    assert launches_prefixed < launches_plain
    for rep in (first, second, third):
        _same(rep, plain)
    want = oracle.run(gates, n, mode)
    assert second.rank_trace == want["rank_trace"]
    for (lam, keys), (wl, wk) in zip(report_gens(second), want["final"]):
        assert np.array_equal(keys, wk) and np.max(np.abs(lam - wl)) < 1e-10


def test_initial_generators_and_shards_go_through_programs():
    n, gates = workloads.build("c2_10q_near_clifford")
    full = qx.run(gates, n, "v3")
    part = qx.run(gates, n, "v3", generators=[7, 2, 9])
    assert "program_steps" in part.device
    for g, (lam, keys) in zip([7, 2, 9], report_gens(part)):
        assert np.array_equal(keys, full.final.generators[g].keys())
        assert np.array_equal(lam, full.final.generators[g].lambdas)
    rng = np.random.default_rng(5)
    init = [(rng.uniform(0.5, 1.0, size=4), np.sort(rng.choice(4 ** n, size=4, replace=False)).astype(np.uint64))
            for _ in range(5)]
    a, b, _ = _both(gates, n, "v3", initial=init)
    _same(a, b)
    assert "program_steps" in a.device


def test_phase_timers_are_measured_on_the_device():
    """RunReport.timings keeps the reference's four keys (engine.py:92); the device phases come from
    the circuit kernel's own clock (one-launch runs) or CUDA events (device_timers=True)."""
    n, gates = workloads.build("c2_10q_near_clifford")
    engine.clear_plans()
    qx.run(gates, n, "v3")
    rep = qx.run(gates, n, "v3")
    assert set(rep.timings) == {"partition", "lut", "sub_flatten", "cx"}
    assert "program_steps" in rep.device
    host = rep.device["host_timings"]["sub_flatten"]
    assert 0.0 < rep.timings["sub_flatten"] <= host           # kernel time inside the host's launch + wait
    engine._PROGRAMS_ON = False
    try:
        engine.clear_plans()
        by_events = qx.run(gates, n, "v3", device_timers=True)
        by_clock = qx.run(gates, n, "v3")
    finally:
        engine._PROGRAMS_ON = True
    assert by_events.timings["sub_flatten"] > 0.0 and by_clock.timings["sub_flatten"] > 0.0
    assert by_events.rank_trace == by_clock.rank_trace == rep.rank_trace
