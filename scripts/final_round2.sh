#!/bin/bash
# Refresh the committed GPU evidence with the current build (one gpurun call):
#   bash scripts/final_round2.sh TAG  ->  gpurun_out/TAG/{pytest_gpu.log, smoke.log, bench.json, launches.csv,
#   prof_*_{raw,details}.csv, prof_*_source.csv.gz, configs.jsonl, acceptance_b200.txt, gpu_criteria.txt}
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
POLYPATH_B200_TRACE=1 timeout 600 oracle/_ref/acceptance_b200 > $OUT/acceptance_b200.txt 2>&1; echo "rc $?" >> $OUT/acceptance_b200.txt
timeout 600 oracle/_ref/gpu_criteria > $OUT/gpu_criteria.txt 2>&1; echo "rc $?" >> $OUT/gpu_criteria.txt
PATHS=131072 SKIP=10 bash scripts/gpu_round.sh $TAG tests smoke bench launches prof:lsq_trip prof:ctrl_eval_trip
PREC=qd SYSTEM=katsura12.sys MAX_NEWTON=4 PATHS=4096 OFFSET=0 SKIP=20 bash scripts/gpu_round.sh $TAG prof:lsq_coop
timeout 3000 python scripts/measure_configs.py > $OUT/configs.jsonl 2> $OUT/configs.err
ls -la $OUT
