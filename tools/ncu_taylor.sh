#!/bin/bash
# ncu --set full of the Taylor tile kernels inside the timed steps of bench.py: tools/ncu_taylor.sh <config> <tag>
cfg=${1:-c2}; tag=${2:-r2_taylor_$cfg}
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:taylor_ -c 7 \
    -o gpurun_out/$tag -f python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/$tag.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.raw.csv 2>/dev/null
python tools/ncu_pick.py gpurun_out/$tag.raw.csv
[ -n "$KEEP_REP" ] || rm -f gpurun_out/$tag.ncu-rep   # the reports are tens of MB: gpurun brings back at most 64 MiB
