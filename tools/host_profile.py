"""cProfile of the host side of run() on one workload (terms stay in HBM)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else "c4_xyz_16_2"
mode = sys.argv[2] if len(sys.argv) > 2 else "v3"
n, gates = workloads.build(name)
def step():
    rep = qx.run(gates, n, mode, download=False)
    rep.device["store"].close()
for _ in range(3):
    step()
cProfile.run("for _ in range(20): step()", "/tmp/host.prof")
pstats.Stats("/tmp/host.prof").sort_stats("tottime").print_stats(18)
