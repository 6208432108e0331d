#!/bin/bash
# Throughput sweep of launch geometry / register budgets (developer experiment, GPU box).
# Each line: SLOTS_PER_SM TRIP_BLOCK LIB
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
shift
while read -r SPS TB LIB; do
  [ -z "$SPS" ] && continue
  L=paper_1505_00383_b200/libpp200.so; [ "$LIB" != "main" ] && L=paper_1505_00383_b200/exp/libpp200_$LIB.so
  echo "== slots/SM $SPS block $TB lib $LIB" >> $OUT/sweep.log
  PP200_SLOTS_PER_SM=$SPS PP200_TRIP_BLOCK=$TB PP200_LIB=$L PATHS=${PATHS:-262144} OFFSET=${OFFSET:-1000000} \
    timeout 600 python scripts/profile_run.py >> $OUT/sweep.log 2>&1
done
