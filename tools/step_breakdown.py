"""Host-side wall-clock breakdown of one circuit run: every DeviceStore call timed with a
synchronize after it, plus store creation/destruction.  Diagnoses overhead outside the kernels."""

import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import store as store_mod
from paper_2505_03307_b200 import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4_xyz_16_2")
ap.add_argument("--mode", default="v3")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--capacity", type=int, default=0)
args = ap.parse_args()

acc = collections.defaultdict(float)
cnt = collections.Counter()


def wrap(cls, name):
    orig = getattr(cls, name)

    def timed(self, *a, **k):
        t0 = time.perf_counter()
        out = orig(self, *a, **k)
        if name not in ("close", "__init__"):
            self.synchronize()
        acc[name] += time.perf_counter() - t0
        cnt[name] += 1
        return out

    setattr(cls, name, timed)


for m in ("__init__", "init_z", "apply_clifford", "apply_split", "apply_operator", "merge", "sort", "close",
          "download"):
    wrap(store_mod.DeviceStore, m)

n, gates = workloads.build(args.workload)
for step in range(args.steps + 1):
    acc.clear()
    cnt.clear()
    t0 = time.perf_counter()
    rep = qx.run(gates, n, args.mode, download=False, capacity=args.capacity)
    rep.device["store"].close()
    total = time.perf_counter() - t0
    print(f"step {step}: total {total * 1e3:.2f} ms  host timings {{{', '.join(f'{k}: {v * 1e3:.2f}' for k, v in rep.timings.items())}}}")
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
        print(f"    {k:16s} x{cnt[k]:<3d} {v * 1e3:9.3f} ms")
    print(f"    {'(python/other)':16s}      {(total - sum(acc.values())) * 1e3:9.3f} ms", flush=True)
