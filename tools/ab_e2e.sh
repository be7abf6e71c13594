#!/bin/bash
# e2e A/B of an environment switch on one box: tools/ab_e2e.sh PB200_NO_PDL  -> value / e2e / e2e_miss with the switch set and unset, twice
sw=${1:?environment switch}
for v in 1 0 1 0; do
  if [ $v = 1 ]; then export $sw=1; else unset $sw; fi
  python bench.py --config ${CONFIG:-c2} --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$sw=$v', 'value=%.1f e2e=%.1f e2e_miss=%.1f' % (d['value'], d['e2e']['value'], d['e2e_miss']['value']))"
done
