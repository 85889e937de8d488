import cProfile, pstats, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else "c5_32q_clifford_t"
mode = sys.argv[2] if len(sys.argv) > 2 else "v3"
n, gates = workloads.build(name)
for _ in range(3): qx.run(gates, n, mode)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): qx.run(gates, n, mode)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
