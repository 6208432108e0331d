#!/bin/bash
# Refresh every piece of committed GPU evidence with the current build (one gpurun call):
#   bash scripts/final_round.sh TAG   ->  gpurun_out/TAG/{pytest_gpu.log, smoke.log, bench.json,
#   launches.csv, prof_*_{raw,details}.csv, prof_*_source.csv.gz, configs.jsonl}
TAG=${1:-final}
PATHS=131072 SKIP=10 bash scripts/gpu_round.sh $TAG tests smoke bench launches prof:lsq_trip prof:ctrl_eval_trip
timeout 2400 python scripts/measure_configs.py > gpurun_out/$TAG/configs.jsonl 2> gpurun_out/$TAG/configs.err
