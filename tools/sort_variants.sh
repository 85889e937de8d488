for v in ${VARIANTS:-0 5 6}; do
  QX_SORT_VARIANT=$v python bench.py --no-cpu --steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['roofline']['classes']
print('variant $v', 'ms/step', round(d['ms_per_step'],3), 'pass ms', round(c['sort_pass']['ms']/c['sort_pass']['launches'],4), 'emit', round(c['dense_emit']['ms']/c['dense_emit']['launches'],3))"
done
for pf in 0 148 592; do
  QX_SORT_PREFETCH=$pf python bench.py --no-cpu --steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['roofline']['classes']
print('prefetch $pf', 'ms/step', round(d['ms_per_step'],3), 'pass ms', round(c['sort_pass']['ms']/c['sort_pass']['launches'],4))"
done
