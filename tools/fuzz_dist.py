"""Fuzz the multi-GPU drivers on ONE GPU: generator shards (run(generators=...)), slot partitions
(run(slot_part=(p, parts))) and, over NCCL at world size 1, run_sharded / run_term_partitioned /
run_slot_partitioned, against the plain run on random ansatz and random circuits.  Not a test:
    python tools/fuzz_dist.py [seconds] [seed]"""
import os, socket, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch, torch.distributed as dist
import paper_2505_03307_b200 as qx
from paper_2505_03307_b200 import dist as qd, workloads

with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t_end = time.time() + budget
case = fails = last_bit = 0

def same(a, b, tol=0.0):
    ok = a.rank_trace == b.rank_trace
    for ga, gb in zip(a.final.generators, b.final.generators):
        ok = ok and np.array_equal(ga.keys(), gb.keys())
        ok = ok and (np.array_equal(ga.lambdas, gb.lambdas) if tol == 0.0 else
                     float(np.max(np.abs(ga.lambdas - gb.lambdas), initial=0.0)) < tol)
    return ok

while time.time() < t_end:
    rng = np.random.default_rng([seed, case]); case += 1
    if rng.integers(0, 2):
        n = int(rng.integers(6, 13))
        gates = workloads.gen_xyz_chain(n, int(rng.integers(1, 4 if n <= 9 else 3)), 1, int(rng.integers(0, 1 << 30)))
        if rng.integers(0, 2):
            gates = gates + workloads.gen_random(n, int(rng.integers(1, 20)), rng, gates=("H", "S", "X", "SX", "CX"))
    else:
        n = int(rng.integers(2, 10))
        gates = workloads.gen_random(n, int(rng.integers(1, 60)), rng)
    mode = str(rng.choice(["v1", "v3"]))
    plain = qx.run(gates, n, mode)
    bad = []
    # generator shards: any split of the generators evolves them exactly as the full run does
    cut = int(rng.integers(0, n + 1))
    ids = [int(v) for v in rng.permutation(n)]
    for part in (sorted(ids[:cut]), sorted(ids[cut:])):
        if part:
            rep = qx.run(gates, n, mode, generators=part)
            for local, g in enumerate(part):
                a, b = rep.final.generators[local], plain.final.generators[g]
                # the operator step picks raw expansion or grouped (factored) sums from the sizes of the
                # whole store, so a shard may round the last bit differently from the full run
                if not (np.array_equal(a.keys(), b.keys()) and float(np.max(np.abs(a.lambdas - b.lambdas), initial=0.0)) < 1e-12):
                    bad.append(("shard", g))
                elif not np.array_equal(a.lambdas, b.lambdas):
                    last_bit += 1
    if not same(qd.run_sharded(gates, n, mode)[0], plain):
        bad.append("run_sharded")
    if not same(qd.run_term_partitioned(gates, n, mode), plain, 1e-12):
        bad.append("run_term_partitioned")
    if mode == "v3":
        if not same(qd.run_slot_partitioned(gates, n, "v3"), plain):
            bad.append("run_slot_partitioned")
        parts = int(rng.integers(2, 6))
        shares = [qx.run(gates, n, "v3", slot_part=(p, parts)) for p in range(parts)]
        if all(s.device.get("partitioned") for s in shares):
            for j, g in enumerate(plain.final.generators):
                keys = np.concatenate([s.final.generators[j].keys() for s in shares])
                lam = np.concatenate([s.final.generators[j].lambdas for s in shares])
                order = np.argsort(keys, kind="stable")
                if not (np.array_equal(keys[order], g.keys()) and np.array_equal(lam[order], g.lambdas)):
                    bad.append(("slot union", j, parts))
        else:
            for s in shares:                       # not partitioned: every part holds the full result
                if not same(s, plain):
                    bad.append("slot fallback")
    if bad:
        fails += 1
        print("MISMATCH", case - 1, n, len(gates), mode, bad[:4], flush=True)
print(f"{case} circuits, {fails} mismatches; {last_bit} shard generators equal to rounding only")
dist.destroy_process_group()
