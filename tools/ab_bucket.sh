#!/bin/bash
# A/B of library builds on the bench step (bucketed path): tools/ab_bucket.sh base b3 ...
here=$(cd "$(dirname "$0")/.." && pwd)
for rep in 1 2; do
for v in "$@"; do
  lib=$here/paper_2505_03307_b200/lib/libqimax_b200_$v.so
  [ "$v" = base ] && lib=$here/paper_2505_03307_b200/lib/libqimax_b200.so
  QX_LIB=$lib python $here/bench.py --no-cpu --no-gate-kernels --steps 10 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['roofline']['classes']
print('$v', 'ms/step', round(d['ms_per_step'],3), 'emit', round(c['bucket_emit']['ms']/c['bucket_emit']['launches'],3), 'prep', round(c['dense_prep']['ms']/3,3), 'e2e', round(d['e2e']['ms_per_step'],2))"
done
done
