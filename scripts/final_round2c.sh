#!/bin/bash
# round-2 re-check after pp_device_init's warm-up run: the acceptance suite (3 fresh processes),
# the drop-in and engine GPU tests, and the default bench with the updated ncu traffic figure
O=gpurun_out/r02y; mkdir -p $O
for i in 1 2 3; do
  POLYPATH_B200_TRACE=1 timeout 300 oracle/_ref/acceptance_b200 > $O/acceptance_b200_$i.txt 2>&1; echo "rc $?" >> $O/acceptance_b200_$i.txt
done
timeout 300 oracle/_ref/gpu_criteria > $O/gpu_criteria.txt 2>&1; echo "rc $?" >> $O/gpu_criteria.txt
timeout 1500 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_engine.py -q -x > $O/pytest_dropin_engine.log 2>&1; echo "pytest rc $?" >> $O/pytest_dropin_engine.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
ls $O
