#!/bin/bash
# L2 persistence A/B (graph mode, alternated) and one instrumented run with it on
OUT=gpurun_out/${1:-l2}
mkdir -p $OUT
for p in 0 1 0 1; do
  echo "== persist $p" >> $OUT/l2.log
  PP200_L2_PERSIST=$p PATHS=262144 timeout 300 python scripts/profile_run.py >> $OUT/l2.log 2>&1
done
printf "512 128 main 128 PP200_L2_PERSIST=1\n512 128 main 128\n" | PATHS=131072 bash scripts/exp_trips.sh ${1:-l2}
