"""Experiment: does evolving generator ranges of the last operator CONCURRENTLY (one host thread and
one CUDA stream per range) beat the single-store step?  The issue-bound slot kernel of one range
could share the SMs with the bandwidth-bound sort passes of another.  Prints both wall times."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import engine, workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c4_xyz_16_2"
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n, gates = workloads.build(name)
stats = {}

def finish_threaded(w, trace, pinned):
    if w.pending is None or w.staged is None:
        return None
    counts, axes, weights = w.staged
    raw = w.store.count_operator(counts)
    target = sum(raw) / shards
    bounds, acc = [0], 0
    for g, r in enumerate(raw):
        acc += r
        if acc >= target and g + 1 < len(raw) and len(bounds) < shards:
            bounds.append(g + 1); acc = 0
    bounds.append(len(raw))
    ranges = list(zip(bounds[:-1], bounds[1:]))
    program = np.array(w.queue, dtype=np.uint32)
    w.queue, w.queue_has_cx, w.staged, w.pending = [], False, None, None
    ranks = [0] * len(w.ids)
    children = [w.store.slice(lo, hi, 0) for lo, hi in ranges]
    def work(child, lo, hi):
        _, r = child.apply_operator_run(counts, axes, weights, program, w.eps)
        ranks[lo:hi] = r
        child.synchronize()
    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(c, lo, hi)) for c, (lo, hi) in zip(children, ranges)]
    for t in ths: t.start()
    for t in ths: t.join()
    stats["last_op_ms"] = 1e3 * (time.perf_counter() - t0)
    stats["ranges"] = ranges
    for c in children: c.close()
    w.ranks = ranks
    for slot in w.open_slots: trace[slot] = list(ranks)
    w.open_slots = []
    w.unsorted = False
    return [(np.zeros(0), np.zeros(0, dtype=np.uint64))] * len(w.ids)      # nothing downloaded

def plain():
    t0 = time.perf_counter()
    rep = qx.run(gates, n, "v3", download=False)
    rep.device["store"].synchronize()
    t = time.perf_counter() - t0
    rep.device["store"].close()
    return 1e3 * t, sum(rep.rank_trace[-1])

for _ in range(3): plain()
print("plain   :", sorted(plain()[0] for _ in range(8))[:4], plain()[1])
orig = engine._finish_streamed
engine._finish_streamed = finish_threaded
def threaded():
    t0 = time.perf_counter()
    rep = qx.run(gates, n, "v3", download=True)
    return 1e3 * (time.perf_counter() - t0), sum(rep.rank_trace[-1])
for _ in range(3): threaded()
res = [threaded() for _ in range(8)]
print(f"threaded x{shards}:", sorted(r[0] for r in res)[:4], res[0][1], stats)
