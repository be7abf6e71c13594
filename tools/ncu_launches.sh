#!/bin/bash
# ncu launch list (durations only) of the timed steps of bench.py: tools/ncu_launches.sh <config> <steps> <tag>
cfg=${1:-c2}; steps=${2:-3}; tag=${3:-r2_launches_$cfg}
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 2000 --csv \
    --log-file gpurun_out/$tag.csv python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/$tag.csv $steps | tee gpurun_out/${tag}_summary.txt
