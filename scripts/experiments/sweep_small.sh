#!/bin/bash
# small-run engine choice: warp per path from the start vs thread per path with narrow blocks
OUT=gpurun_out/${1:-small}
mkdir -p $OUT
for cfg in "default" "PP200_TAIL_SLOTS=0 PP200_TRIP_BLOCK=32" "PP200_TAIL_SLOTS=0 PP200_TRIP_BLOCK=64" "PP200_TRIP_BLOCK=32 PP200_TAIL_SLOTS=592"; do
  E=$cfg; [ "$cfg" = "default" ] && E=""
  echo "== $cfg" >> $OUT/small.log
  env $E timeout 600 python scripts/measure_configs.py --only katsura12_qd cyclic5_dd cyclic5_qd --cpu-budget 0 >> $OUT/small.log 2>&1
done
