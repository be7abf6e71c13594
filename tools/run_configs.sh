#!/bin/bash
# BASELINE configs 3, 4, the config-5 sweep and the two paper-regime points on one B200 -> gpurun_out/r2_cfg_*.json
out=gpurun_out
run() { name=$1; shift; timeout 1500 python bench.py "$@" > $out/r2_cfg_$name.json 2> $out/r2_cfg_$name.err || echo "$name: rc=$?"; tail -c 200 $out/r2_cfg_$name.err; }
run c3 --config c3 --steps 20 --warmup 3 --cpu-baseline-steps 1
run c4 --config c4 --steps 20 --warmup 3 --cpu-baseline-steps 1
run c5_1e5 --config c5:1e5 --steps 20 --warmup 3 --no-cpu-baseline
run c5_1e7 --config c5:1e7 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e
run c5_3e7 --config c5:3e7 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
run c5_1e8 --config c5:1e8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
run paper3d --config paper3d --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
run paper1d --config paper1d --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
