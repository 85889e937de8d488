#!/bin/bash
# bucket tests + the bench step and kernel time (one line)
python -m pytest tests/test_gpu_bucket.py tests/test_gpu_eps_boundary.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do
python bench.py --steps 20 --warmup 3 --no-gate-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms_per_step', round(d['ms_per_step'],4), 'bucket_emit ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],4))"
done
