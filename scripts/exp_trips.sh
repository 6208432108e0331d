#!/bin/bash
# Per-trip timing logs (steady state vs tail) for launch-geometry variants. Lines on stdin:
# SLOTS_PER_SM TRIP_BLOCK LIB [EVAL_BLOCK [VAR=VALUE ...]]
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
while read -r SPS TB LIB EB EXTRA; do
  EB=${EB:-$TB}
  TAGX=$(echo "$EXTRA" | tr -c 'A-Za-z0-9' '_')
  [ -z "$SPS" ] && continue
  L=paper_1505_00383_b200/libpp200.so; [ "$LIB" != "main" ] && L=paper_1505_00383_b200/exp/libpp200_$LIB.so
  echo "== slots/SM $SPS block $TB lib $LIB eval-block $EB $EXTRA" >> $OUT/trips.log
  env $EXTRA PP200_KERNEL_TIMING=1 PP200_TRIP_LOG=$OUT/trips_${SPS}_${TB}_${LIB}_${EB}${TAGX}.txt PP200_EVAL_BLOCK=$EB PP200_SLOTS_PER_SM=$SPS PP200_TRIP_BLOCK=$TB PP200_LIB=$L \
    PATHS=${PATHS:-131072} OFFSET=${OFFSET:-1000000} timeout 600 python scripts/profile_run.py >> $OUT/trips.log 2>&1
done
