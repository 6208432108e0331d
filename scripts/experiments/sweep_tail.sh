mkdir -p gpurun_out/r01u
for cfg in "90 4736" "95 4736" "98 4736" "90 9472" "95 9472" "90 2368"; do
  set -- $cfg
  echo "== pct $1 tail $2" >> gpurun_out/r01u/tail.log
  PP200_COMPACT_PCT=$1 PP200_TAIL_SLOTS=$2 PATHS=262144 timeout 300 python scripts/profile_run.py >> gpurun_out/r01u/tail.log 2>&1
done
PP200_KERNEL_TIMING=1 PP200_TRIP_LOG=gpurun_out/r01u/trips_default.txt PATHS=262144 timeout 300 python scripts/profile_run.py >> gpurun_out/r01u/tail.log 2>&1
