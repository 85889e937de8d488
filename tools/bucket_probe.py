"""Bucketed operator step (csrc/bucket.cuh) on ansatz circuits: did it run, bucket geometry, wall time,
digest of the result (compare with QX_NO_BUCKET=1: the grouped step + sort)."""
import ctypes as C
import hashlib
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import _native


def last():
    out = (C.c_int64 * 8)()
    _native.lib().qx_bucket_last(out)
    return dict(zip(("groups", "tiles", "buckets", "max_bucket", "slots", "ell", "cap", "ctas_per_sm"), list(out)))


def digest(rep):
    h = hashlib.sha256()
    for g in rep.final.generators:
        h.update(np.ascontiguousarray(g.keys()).tobytes())
        h.update(np.ascontiguousarray(g.lambdas).tobytes())
    return h.hexdigest()[:16]


for arg in sys.argv[1:] or ["10,2", "12,2", "14,2"]:
    n, layers = (int(v) for v in arg.split(","))
    circ = qx.gen_xyz_chain(n, layers, 1, rng=4)
    qx.run(circ, n, "v3", device=0)
    t0 = time.perf_counter()
    rep = qx.run(circ, n, "v3", device=0)
    dt = time.perf_counter() - t0
    norms = [float(np.sum(g.lambdas ** 2)) for g in rep.final.generators]
    ok_sorted = all(np.all(np.diff(g.keys().astype(np.uint64)) > 0) for g in rep.final.generators if g.rank > 1)
    print(arg, "terms", sum(rep.rank_trace[-1]), "sha", digest(rep), "sorted", ok_sorted,
          "max|norm-1|", max(abs(v - 1) for v in norms), f"{dt*1e3:.1f} ms", last(), flush=True)
