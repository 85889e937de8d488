#!/bin/bash
# A/B of library builds on the bench step: tools/ab_libs.sh base hw va ...  ("base" = the shipped library)
here=$(cd "$(dirname "$0")/.." && pwd)
for rep in 1 2; do
for v in "$@"; do
  lib=$here/paper_2505_03307_b200/lib/libqimax_b200_$v.so
  [ "$v" = base ] && lib=$here/paper_2505_03307_b200/lib/libqimax_b200.so
  QX_LIB=$lib python $here/bench.py --no-cpu --steps 10 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['roofline']['classes']
print('$v', 'ms/step', round(d['ms_per_step'],3), 'pass ms', round(c['sort_pass']['ms']/c['sort_pass']['launches'],4), 'frac', round(d['roofline']['frac'],4), 'emit', round(c['dense_emit']['ms']/c['dense_emit']['launches'],3), 'e2e', round(d['e2e']['ms_per_step'],2))"
done
done
