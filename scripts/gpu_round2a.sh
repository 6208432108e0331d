#!/bin/bash
# round-2 GPU batch: drop-in acceptance through the GPU, bench, trip logs, shard balance
set -x
mkdir -p gpurun_out/r2a
python -m pytest tests/test_gpu_dropin.py -q -s > gpurun_out/r2a/dropin.txt 2>&1
python bench.py --steps 3 --warmup 3 > gpurun_out/r2a/bench.txt 2>&1
PP200_KERNEL_TIMING=1 PP200_TRIP_LOG=gpurun_out/r2a/trips_c10dd.txt PATHS=262144 OFFSET=2384256 python scripts/profile_run.py > gpurun_out/r2a/prof_c10dd.txt 2>&1
PP200_KERNEL_TIMING=1 PP200_TRIP_LOG=gpurun_out/r2a/trips_k12qd.txt PATHS=4096 OFFSET=0 PREC=qd SYSTEM=katsura12.sys MAX_NEWTON=4 python scripts/profile_run.py > gpurun_out/r2a/prof_k12qd.txt 2>&1
python scripts/shard_balance.py --prec d > gpurun_out/r2a/shard_balance_d.json 2> gpurun_out/r2a/shard_balance_d.err
python scripts/shard_balance.py --prec dd > gpurun_out/r2a/shard_balance_dd.json 2> gpurun_out/r2a/shard_balance_dd.err
tail -3 gpurun_out/r2a/*.txt
