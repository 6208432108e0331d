#!/bin/bash
PREC=d PATHS=262144 OFFSET=1500000 SKIP=10 bash scripts/gpu_round.sh r02d prof:lsq_trip_reg prof:ctrl_eval_trip
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02d/bench_default.json 2> gpurun_out/r02d/bench.err
tail -c 300 gpurun_out/r02d/bench_default.json
