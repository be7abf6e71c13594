#!/bin/bash
# compute-sanitizer over the sharded path: (1) one rank over the library's NCCL transport, (2) two ranks sharing the GPU
# over the host-staged test transport (rows with halo columns, routed keys, look-up requests really cross ranks).
tag=${1:-r2_sharded}
PB200_SANITIZE_SHARDED=1 timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_small.py \
    > gpurun_out/${tag}_memcheck_one_rank_nccl.log 2>&1
tail -4 gpurun_out/${tag}_memcheck_one_rank_nccl.log
for tool in memcheck racecheck; do
    timeout 1500 compute-sanitizer --tool $tool --target-processes all python -m torch.distributed.run --nnodes=1 \
        --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29655 tests/dist_worker.py \
        cfg1_holstein_L4_d8,ties_holstein_L5_d6,cube_2x2x2_d16 8 > gpurun_out/${tag}_${tool}_two_ranks.log 2>&1
    grep -E "SHARDED_OK|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/${tag}_${tool}_two_ranks.log | cut -c1-200
done
