#!/bin/bash
# ncu --set full of the adapt-phase kernels (selection + incremental adapt) of ONE timed step: tools/ncu_adapt.sh <config> <tag>
cfg=${1:-c2}; tag=${2:-r2_adapt_$cfg}
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k "regex:inc_|select_|weights_|segment_|place_|scan_" -c 60 \
    -o gpurun_out/$tag -f python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/$tag.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.raw.csv 2>/dev/null
python tools/ncu_pick.py gpurun_out/$tag.raw.csv > gpurun_out/${tag}_summary.txt
grep -c "Kernel Name" gpurun_out/${tag}_summary.txt
[ -n "$KEEP_REP" ] || rm -f gpurun_out/$tag.ncu-rep
