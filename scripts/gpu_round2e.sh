#!/bin/bash
mkdir -p gpurun_out/r2e
O=gpurun_out/r2e/ab.txt
for LIB in paper_1505_00383_b200/libpp200.so paper_1505_00383_b200/exp/libpp200_noinl.so; do
  echo "== $LIB" >> $O
  PP200_LIB=$PWD/$LIB timeout 300 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_COOP_GROUP=32,8 >> $O 2>&1
  PP200_LIB=$PWD/$LIB timeout 200 python scripts/ab.py cyclic5 qd 0 120 PP200_COOP_GROUP=32,8 >> $O 2>&1
done
timeout 600 python scripts/ab.py rand32 qd 0 16 PP200_COOP_GROUP=32,8 >> $O 2>&1
PP200_KERNEL_TIMING=1 PP200_TRIP_LOG=gpurun_out/r2e/trips_r32qd.txt PATHS=16 OFFSET=0 PREC=qd SYSTEM=rand32.sys timeout 300 python scripts/profile_run.py >> $O 2>&1
cat $O
