#!/bin/bash
# A/B of library builds on one box: CONFIG=c4 tools/ab_variants.sh variants/*.so  -> one short line per build
for lib in "$@"; do
  PB200_LIB=$lib timeout 300 python bench.py --config ${CONFIG:-c2} --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys, json
d = json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r = d['roofline']; p = d['phase_ms_per_step']
print('$lib', 'step_ms=%.3f select=%.3f adapt=%.3f expmv=%.3f taylor_frac=%.3f launch_us=%.1f iso_us=%.1f' % (d['ms_per_step'], p['select_ms'], p['grow_ms'], p['expmv_ms'], r['frac'], 1e3*r['avg_launch_ms'], 1e3*r['isolated_l2_flushed']['ms']))"
done
