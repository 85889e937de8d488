"""bench.py -- the driver's measurement contract for the extended-stabilizer hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4_xyz_16_2] [--mode v3]

One "step" = one whole circuit: init_z -> every gate/operator -> final canonical generators
(the paper's timing window).  The metric is BASELINE.json's: term-gate updates/s,
where the update count of a circuit is sum over gates of the ranks before the gate in the
reference's v1 semantics -- a property of the circuit, the same numerator for
every mode and for the CPU arm.  Default workload: BASELINE's largest-rank config, the
xyz_chain(16, 2) point of config 4 (1.25e8 final terms; the n=20, L=4 point is infeasible for
any exact method).

  value     updates/s, K steps bracketed by barrier + synchronize, CUDA events on the launch
            stream, max over ranks; terms never leave HBM inside the timed region
  e2e       the same through the public API run(instructions, n, mode) with host buffers: gate
            tables go host->device and the final generators come back into pinned host memory
  roofline  the dominant kernel (one onesweep radix pass, 32 B of algorithmic traffic per term)
            timed per launch with CUDA events in a second, instrumented set of steps
  cpu_baseline  the numpy oracle port on the host cores over a bounded sample (a subset of the
            same circuit's generators -- they evolve independently), same unit

N > 1 (torchrun), default --scaling strong: ONE circuit; every rank evolves it up to the last
branching operator (a negligible share of the work) and then works off its own contiguous range
of that operator's buckets, i.e. of (generator, key) order (dist.run_slot_partitioned: even split
however skewed the generators are; generator sharding caps at ~3x here because generator 0 holds
a third of the terms).  --scaling weak (replicas, only on request): every rank evolves one whole
circuit instance of the workload (same ansatz and shape, its own rotation angles), so per-GPU work
is fixed and value is the sum of the ranks' update counts over the slowest rank's time.  Either
way there is no data-path collective; the only NCCL traffic is the barrier, the agreement on
errors and the max/sum of scalars (the shares' counts in strong mode).
--impl reference runs the CPU arm.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2505_03307_b200 import workloads  # noqa: E402

DEFAULT_WORKLOAD = "c4_xyz_16_2"
# generator subset used as the bounded CPU sample of each workload (None = whole circuit)
CPU_SAMPLE = {"c4_xyz_16_2": list(range(2, 16)), "c4_xyz_18_2": list(range(4, 18)),
              "c4_xyz_14_2": list(range(0, 14))}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        try:
            with open(path) as fh:
                v = float(json.load(fh)["hbm_gbs"])
            if v > 0:
                return v, "measured (MEASURED_PEAKS.json)"
        except (OSError, ValueError, KeyError, TypeError):
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc, self.nvml_thread = device, [], None, None

    def _nvml_start(self):
        """NVML in a thread, one reading every 4 ms: the device-timed region is ~30 ms long, which
        nvidia-smi's own loop (>= 100 ms per reading) samples once at best."""
        import pynvml as nv
        nv.nvmlInit()
        ids = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        index = self.device
        if ids and all(tok.strip().isdigit() for tok in ids.split(",")) and self.device < len(ids.split(",")):
            index = int(ids.split(",")[self.device])
        h = nv.nvmlDeviceGetHandleByIndex(index)
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        bits = ((nv.nvmlClocksEventReasonHwSlowdown, 3), (nv.nvmlClocksEventReasonHwThermalSlowdown, 4),
                (nv.nvmlClocksEventReasonSwThermalSlowdown, 5), (nv.nvmlClocksEventReasonSwPowerCap, 6))
        nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)            # fail here, not in the thread
        nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.stop = threading.Event()

        def poll():
            while not self.stop.is_set():
                try:
                    row = [str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), str(mx), "", "", "", "", ""]
                    mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for bit, col in bits:
                        row[col] = "Active" if mask & bit else "Not Active"
                    self.rows.append(row)
                except Exception:
                    return
                self.stop.wait(0.004)

        self.nvml_thread = threading.Thread(target=poll, daemon=True)
        self.nvml_thread.start()

    def __enter__(self):
        self.nvml_thread = None
        try:
            self._nvml_start()
            return self
        except Exception:
            self.nvml_thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.nvml_thread is not None:
            self.stop.set()
            self.nvml_thread.join(timeout=2)
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
            except (ValueError, IndexError):
                continue
            for name, flag in zip(names, r[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml, 4 ms period" if self.nvml_thread is not None else "nvidia-smi -lms 100"}


def job_config(name, mode, n, n_gates, total_updates, final_terms, world, strong):
    """The `config` object of BOTH arms (ours and --impl reference): what the job is, nothing
    about how an arm runs it (the CPU arm's bounded sample is described in its cpu_baseline)."""
    return {"workload": name, "mode": mode, "qubits": n, "gates": n_gates,
            "term_gate_updates": float(total_updates), "final_terms": int(final_terms),
            "parallelism": (f"one circuit, buckets of the last operator split over {world} GPUs" if strong else
                            f"{world} circuit instance(s), one per GPU, all generators of an instance on its GPU"),
            "l2": "inputs larger than L2: every pass streams 2-5 GB per GPU, L2 is 126 MB"}


def lpt_shards(weights, world):
    """Longest-processing-time assignment of generators to ranks."""
    loads, shards = [0.0] * world, [[] for _ in range(world)]
    for g in sorted(range(len(weights)), key=lambda i: -weights[i]):
        r = loads.index(min(loads))
        shards[r].append(g)
        loads[r] += weights[g]
    return [sorted(s) for s in shards]


# ------------------------------------------------------------------------------------------
# CPU arm (numpy oracle port): also the cpu_baseline leg of the GPU arm
# ------------------------------------------------------------------------------------------
def host_cpu() -> str:
    """Model name and logical core count of the host (state them beside the CPU arm)."""
    model = "unknown CPU"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.lower().startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return f"{model}, {os.cpu_count() or 1} logical cores"


def _cpu_worker(args):
    name, mode, gens = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import stabsim_port as port

    n, gates = workloads.build(name)
    t0 = time.perf_counter()
    res = port.run(gates, n, mode, generators=gens)
    return time.perf_counter() - t0, [len(l) for l, _ in res["final"]]


def cpu_step(name, mode, gens, procs):
    """One pass of the oracle over `gens`, split over `procs` processes; returns wall seconds."""
    import multiprocessing as mp

    if procs <= 1:
        return _cpu_worker((name, mode, gens))[0]
    # rank grows towards low generator ids on the ladder: deal them round-robin from the heavy end
    parts = [gens[i::procs] for i in range(procs)]
    parts = [p for p in parts if p]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(len(parts)) as pool:
        pool.map(_cpu_worker, [(name, mode, p) for p in parts])
    return time.perf_counter() - t0


def cpu_full_circuit(name, mode, weights):
    """The WHOLE circuit on the host: one process per generator, the heaviest first (the pool
    hands the next generator to whichever core is free).  Returns wall seconds."""
    import multiprocessing as mp

    n, _ = workloads.build(name)
    order = sorted(range(n), key=lambda g: -weights[g])
    procs = max(1, min(os.cpu_count() or 1, n))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        list(pool.imap_unordered(_cpu_worker, [(name, mode, [g]) for g in order], chunksize=1))
    return time.perf_counter() - t0, procs


def final_terms_of(name, mode):
    """Final term count of a workload from the reference-made digests (no GPU on this arm)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "digests.json")) as fh:
            return int(sum(json.load(fh)["data"][f"{name}/{mode}"]["trace_last"]))
    except (OSError, KeyError, ValueError):
        return 0


def run_reference(args, updates_per_gen):
    """--impl reference: the reference algorithm (oracle port) on the host cores.  `config` is the
    GPU arm's (same job); every step is a bounded sample of it -- a subset of the circuit's
    generators, which evolve independently -- described in `cpu_baseline.sample`.  --ref-full
    also runs the whole circuit once (all generators, one process each, heavy first: minutes and
    tens of GB at the default workload) and reports it as `cpu_baseline.full_circuit`."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    n, gates = workloads.build(args.workload)
    gens = CPU_SAMPLE.get(args.workload) or list(range(n))
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, len(gens)))
    upd = float(sum(updates_per_gen[g] for g in gens))
    for _ in range(args.warmup):
        cpu_step(args.workload, args.mode, gens[-2:], 1)          # warm imports/pages, tiny
    t = [cpu_step(args.workload, args.mode, gens, procs) for _ in range(args.steps)]
    sec = sum(t) / len(t)
    value = upd / sec
    sample = (f"generators {gens[0]}..{gens[-1]} of {args.workload} ({len(gens)} of {n}; generators evolve "
              f"independently), {args.mode}, numpy port of the reference (oracle/stabsim_port.py), "
              f"{procs} processes; value = the sample's updates / the sample's time")
    cpu = {"value": value, "unit": "updates/s", "cores": procs, "kind": "port", "sample": sample, "host": host_cpu()}
    if args.ref_full:
        full_s, full_procs = cpu_full_circuit(args.workload, args.mode, updates_per_gen)
        cpu["full_circuit"] = {"value": float(sum(updates_per_gen)) / full_s, "unit": "updates/s", "seconds": full_s,
                               "cores": full_procs, "generators": n}
    strong = world > 1 and args.scaling == "strong"
    line = {
        "impl": "reference", "metric": "term_gate_updates_per_s", "value": value, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": job_config(args.workload, args.mode, n, len(gates), float(sum(updates_per_gen)),
                             final_terms_of(args.workload, args.mode), world, strong),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------
def gate_kernel_rooflines(device, peak, terms=60_000_000, n=16):
    """GB/s by algorithmic bytes of the v1 kernels on one generator of `terms` distinct
    random terms: {class: {"ms", "launches", "gbs", "frac"}} from CUDA events around every launch."""
    from paper_2505_03307_b200 import _native as nat, lut
    from paper_2505_03307_b200.stabilizer import split_tables
    from paper_2505_03307_b200.store import DeviceStore

    # distinct pseudo-random words: an odd multiplier is a bijection on 32-bit words
    keys = (np.arange(terms, dtype=np.uint64) * np.uint64(2654435761)) & np.uint64(4 ** n - 1)
    lam = np.random.default_rng(3).uniform(-1, 1, size=terms)
    prog = [lut.cx_op(n, q, q + 1) for q in range(n - 1)] + [lut.perm_op(n, q, lut.FIXED_PERMS["H"]) for q in range(0, n, 3)]
    prog = np.array(prog, dtype=lut.op_dtype(n))
    tabs = split_tables(lut.gate_branch_block("RZ", 0.7))
    for rep in range(3):
        with DeviceStore(n, 1, 2 * terms + 16, device) as st:
            st.upload([(lam, keys)])
            st.synchronize()
            if rep == 1:
                nat.profile_enable(True)
                nat.profile_reset()
            st.apply_clifford(prog)
            st.sort()
            st.apply_split(n // 2, *tabs)
            st.merge(1e-12)
            st.synchronize()
    prof = nat.profile_read()
    nat.profile_enable(False)
    out = {"terms": terms, "qubits": n}
    for k, v in prof.items():
        if v["launches"]:
            gbs = v["alg_bytes"] / max(v["ms"], 1e-9) / 1e6
            out[k] = {"ms": round(v["ms"] / v["launches"], 4), "launches": v["launches"], "gbs": round(gbs, 1),
                      "frac": round(gbs / peak, 3)}
    return out



def count_updates_gpu(name, device, instance=0):
    """v1-defined update count per generator, measured with the GPU's own v1 mode (untimed)."""
    import paper_2505_03307_b200 as qx

    n, gates = workloads.build(name, instance)
    rep = qx.run(gates, n, "v1", device=device, download=False)
    rep.device["store"].close()
    return rep.device["updates_per_generator"], rep.rank_trace[-1]


def table_bytes(n, gates):
    """Host->device bytes of one run: packed gate words + per-operator branch tables."""
    from paper_2505_03307_b200 import circuit as ir

    part = ir.divide_instruction(gates, n)
    return 4 * len(gates) + part.k * n * 3 * (4 + 3 * 4 + 3 * 8)


def run_ours(args):
    import torch

    import paper_2505_03307_b200 as qx
    from paper_2505_03307_b200 import _native as nat

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    # QX_BENCH_BACKEND=gloo + QX_BENCH_SHARE_GPU=1: several ranks on ONE GPU with CPU collectives --
    # only to exercise the multi-rank code path on a one-GPU box (tools/bench_two_ranks.sh)
    backend = os.environ.get("QX_BENCH_BACKEND", "nccl")
    share = os.environ.get("QX_BENCH_SHARE_GPU", "") == "1"
    device = local % torch.cuda.device_count() if share else local
    red_dev = "cuda" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(device)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(device)
    weak = args.scaling == "weak" and world > 1
    instance = rank if weak else 0
    n, gates = workloads.build(args.workload, instance)

    # untimed: update counts (v1 semantics) and final ranks for LPT sharding
    updates_per_gen, final_ranks = count_updates_gpu(args.workload, device, instance)
    total_updates = float(sum(updates_per_gen))
    if weak:
        mine = list(range(n))                      # my own circuit instance, all of its generators
        t = torch.tensor([total_updates], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_updates = float(t.item())
    else:
        mine = list(range(n))                      # strong: all generators, my range of the output slots
    strong = world > 1 and not weak
    my_cap = int(sum(final_ranks[g] for g in mine) * 2.6 / (world if strong else 1)) + 1024
    if strong:
        from paper_2505_03307_b200 import dist as qd

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def step_resident():
        if strong:
            rep = qd.run_slot_partitioned(gates, n, args.mode, device=device, capacity=my_cap, download=False)
        else:
            rep = qx.run(gates, n, args.mode, device=device, generators=mine, capacity=my_cap, download=False)
        rep.device["store"].close()
        return rep

    def step_e2e():
        if strong:
            return qd.run_slot_partitioned(gates, n, args.mode, device=device, capacity=my_cap, pinned=True)
        return qx.run(gates, n, args.mode, device=device, generators=mine, capacity=my_cap, pinned=True)

    for _ in range(max(args.warmup, 3)):
        step_resident()

    # ---- value: K steps, device-timed on the launch stream, max over ranks
    barrier()
    l0 = nat.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clocks:
        ev0.record()
        for _ in range(args.steps):
            step_resident()
        ev1.record()
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = nat.launch_count() - l0
    t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    value = total_updates / (ms_per_step * 1e-3)

    # ---- e2e: public API with host buffers (tables H2D, final generators D2H into pinned memory)
    step_e2e()
    barrier()
    t0 = time.perf_counter()
    last = None
    e2e_each = []
    for _ in range(args.steps):
        last = None                      # drop the previous result first: its pinned block is reused
        t1 = time.perf_counter()
        last = step_e2e()
        e2e_each.append(time.perf_counter() - t1)
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    t = torch.tensor([e2e_s], device=red_dev, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    final_terms = sum(g.rank for g in last.final.generators)
    # bytes that crossed PCIe: the run reports them when it shipped 32-bit keys (n <= 16, widened on the host)
    d2h = last.device.get("d2h_bytes", 16 * final_terms) + 8 * (len(mine) + 1)
    del last

    # ---- roofline of the dominant kernel: instrumented steps (CUDA events around every launch)
    nat.profile_enable(True)
    nat.profile_reset()
    for _ in range(max(1, min(args.steps, 3))):
        step_resident()
    prof = nat.profile_read()
    nat.profile_enable(False)
    peak, peak_src = peaks()
    busy = {k: v for k, v in prof.items() if v["launches"]}
    dom = max(busy, key=lambda k: busy[k]["ms"]) if busy else None
    roof = None
    if dom:
        d = busy[dom]
        achieved = d["alg_bytes"] / (d["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                "launches_per_step": d["launches"] / max(1, min(args.steps, 3)),
                "avg_launch_ms": d["ms"] / d["launches"],
                "alg_bytes_per_launch": d["alg_bytes"] / d["launches"],
                "classes": {k: {"ms": round(v["ms"], 4), "launches": v["launches"],
                                "gbs": round(v["alg_bytes"] / max(v["ms"], 1e-9) / 1e6, 1)}
                            for k, v in busy.items()}}
        # the whole step by SURVEY.md 8d's UNFUSED measure (B_term = 16): every step where ranks change
        # counted as operator-apply 16 B x (N_in + N_raw) + merge 16 B x (N_raw + N_out), N_raw = what
        # the step reports (output slots where the grouped step ran) -- the traffic separate
        # expand / sort / reduce passes would need at the very least, over the measured step time
        rep = step_resident()
        trace = [sum(r) for r in rep.rank_trace]
        n_in = sum(a for a, b in zip(trace, trace[1:]) if a != b)
        n_out = sum(b for a, b in zip(trace, trace[1:]) if a != b)
        raw = int(rep.device.get("raw_terms", 0))
        step_bytes = 16.0 * (n_in + raw) + 16.0 * (raw + n_out)
        step_gbs = step_bytes / (ms_per_step * 1e-3) / 1e9
        roof["step"] = {"alg_bytes": step_bytes, "achieved": step_gbs, "frac": step_gbs / peak, "unit": "GB/s",
                        "measure": "SURVEY 8d unfused: 16 B x (N_in + N_raw) + 16 B x (N_raw + N_out) per rank-changing "
                                   "step, over ms_per_step", "raw_terms": raw}
        traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(traffic_file):
            with open(traffic_file) as fh:
                roof["traffic"] = json.load(fh).get(dom)

    # ---- the gate-by-gate (v1) kernels of north-star subsystems (2) and (3) at scale, measured live:
    # one generator of 6e7 random terms through a 21-op Clifford run (bit-sliced kernel), a re-sort
    # (radix passes), an RZ split and the merge behind it (passes + segmented reduce)
    if roof is not None and world == 1 and not args.no_gate_kernels:
        roof["gate_kernels"] = gate_kernel_rooflines(device, peak)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- cpu_baseline (rank 0, N = 1 only): oracle port on a bounded sample, one core
    cpu = None
    if world == 1 and not args.no_cpu:
        gens = CPU_SAMPLE.get(args.workload) or list(range(n))
        sec = cpu_step(args.workload, args.mode, gens, 1)
        cpu = {"value": float(sum(updates_per_gen[g] for g in gens)) / sec, "unit": "updates/s", "cores": 1,
               "kind": "port", "host": host_cpu(),
               "sample": f"generators {gens[0]}..{gens[-1]} of {args.workload} ({len(gens)} of {n}), {args.mode}, "
                         f"numpy port of the reference (oracle/stabsim_port.py), {sec:.1f} s on 1 core"}

    line = {
        "metric": "term_gate_updates_per_s", "value": value, "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak" if (weak or world == 1) else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": job_config(args.workload, args.mode, n, len(gates), total_updates, int(sum(final_ranks)), world,
                             strong),
        "e2e": {"value": total_updates / e2e_s, "unit": "updates/s", "ms_per_step": e2e_s * 1e3,
                "ms_per_step_min": min(e2e_each) * 1e3, "ms_per_step_median": statistics.median(e2e_each) * 1e3,
                "h2d_bytes_per_step": table_bytes(n, gates), "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "ranks": {"world": world, "backend": backend if world > 1 else None},
        "clocks": clocks.summary(),
        "roofline": roof,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--mode", default="v3")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-gate-kernels", action="store_true", help="skip the live roofline of the v1 gate kernels")
    ap.add_argument("--ref-full", action="store_true",
                    help="--impl reference: also run the WHOLE circuit once on the host (all generators)")
    ap.add_argument("--scaling", default="strong", choices=("weak", "strong"),
                    help="N > 1: ONE circuit, the buckets of its last operator split over the GPUs (strong, the "
                         "north star's sharding; default) or replicas, one circuit instance per GPU (weak)")
    args = ap.parse_args()
    if args.impl == "reference":
        # update counts of the sample come from the fixture table (no GPU on this arm)
        with open(os.path.join(ROOT, "tests", "golden", "updates.json")) as fh:
            table = json.load(fh)["data"]
        if args.workload not in table:
            print(json.dumps({"impl": "reference", "unavailable": f"no update table for {args.workload}"}))
            return
        run_reference(args, table[args.workload])
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
