"""D2H rate of this box: pinned download of a resident store, whole and per array."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_03307_b200.store import DeviceStore
n_terms = 100_000_000
rng = np.random.default_rng(0)
keys = rng.integers(0, 4 ** 16, size=n_terms, dtype=np.uint64)
lam = rng.uniform(-1, 1, size=n_terms)
with DeviceStore(16, 1, n_terms + 16) as st:
    st.upload([(lam, keys)])
    for rep in range(4):
        t0 = time.perf_counter()
        off, k, l = st.download(pinned=True)
        dt = time.perf_counter() - t0
        print(f"download {16 * n_terms / 1e9:.2f} GB pinned: {1e3 * dt:.2f} ms = {16 * n_terms / dt / 1e9:.1f} GB/s")
        del off, k, l
