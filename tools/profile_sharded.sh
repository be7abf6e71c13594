#!/bin/bash
# Round-2 evidence for the sharded path on ONE GPU (a one-rank NCCL communicator: every collective call site runs as a
# self-exchange): bench lines for C2 / C4, a 2-rank function check over the host-staged test transport, the ncu launch
# list and an ncu --set full capture of the sharded tile kernels.  tools/profile_sharded.sh <tag>
tag=${1:-r2_sharded_final}
python bench.py --sharded --steps 10 --warmup 3 > gpurun_out/${tag}_c2.json 2> gpurun_out/${tag}_c2.err
python bench.py --sharded --config c4 --steps 5 --warmup 3 > gpurun_out/${tag}_c4.json 2> gpurun_out/${tag}_c4.err
PB200_BENCH_SAME_DEVICE=1 python bench.py --gpus 2 --transport gloo --q-nom 100000 --steps 3 --warmup 3 \
    > gpurun_out/${tag}_two_ranks_gloo.json 2> gpurun_out/${tag}_two_ranks_gloo.err
PB200_PROF_SHARDED=1 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 3000 --csv \
    --log-file gpurun_out/${tag}_launches.csv python tools/prof_steps.py 1e6 9 2 c2 > gpurun_out/${tag}_launches.log 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_launches.csv 2 > gpurun_out/${tag}_launches_summary.txt
PB200_PROF_SHARDED=1 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:taylor_tile -c 6 \
    -o gpurun_out/${tag}_taylor -f python tools/prof_steps.py 1e6 9 1 c2 > gpurun_out/${tag}_taylor.log 2>&1
ncu -i gpurun_out/${tag}_taylor.ncu-rep --page raw --csv > gpurun_out/${tag}_taylor.raw.csv 2>/dev/null
python tools/ncu_pick.py gpurun_out/${tag}_taylor.raw.csv > gpurun_out/${tag}_taylor_summary.txt
rm -f gpurun_out/${tag}_taylor.ncu-rep
for f in c2 c4 two_ranks_gloo; do python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/${tag}_$f.json").read().strip().splitlines()[-1])
    print("$f", d["value"], d["ms_per_step"], d.get("phase_ms_per_step"), d.get("state", {}).get("q_true"))
except Exception as e:
    print("$f", "FAILED", e)
PY
done
cat gpurun_out/${tag}_launches_summary.txt | head -40
