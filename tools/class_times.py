"""Run bench.py's GPU arm quietly and print ms/step plus selected kernel-class times."""
import json, os, subprocess, sys
tag = sys.argv[1] if len(sys.argv) > 1 else ""
out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu"] + sys.argv[2:],
                     capture_output=True, text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
try:
    d = json.loads(out.stdout.strip().splitlines()[-1])
    c = d["roofline"]["classes"]
    print(tag, "ms/step", round(d["ms_per_step"], 3), {k: round(v["ms"] / 3, 3) for k, v in c.items() if v["ms"] > 0.05}, flush=True)
except Exception as e:
    print(tag, "FAILED", e, out.stderr[-500:])
