#!/bin/bash
# A/B of environment switches on the bench step: tools/ab_env.sh "QX_BUCKET_ROWS=0" "QX_BUCKET_ROWS=1" ...
here=$(cd "$(dirname "$0")/.." && pwd)
for rep in 1 2; do
for v in "$@"; do
  env $v python $here/bench.py --no-cpu --no-gate-kernels --steps 10 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['roofline']['classes']
print('$v', 'ms/step', round(d['ms_per_step'],3), 'emit', round(c['bucket_emit']['ms']/c['bucket_emit']['launches'],3), 'prep', round(c['dense_prep']['ms']/3,3), 'e2e', round(d['e2e']['ms_per_step'],2))"
done
done
