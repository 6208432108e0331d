#!/bin/bash
# final build of round 2 (network-merge qd addition): the reference acceptance suite through the
# shim, criteria 4/6 on the device, pytest -m gpu, smoke, bench, and the qd solver under ncu
OUT=gpurun_out/r02f
mkdir -p $OUT
POLYPATH_B200_TRACE=1 timeout 600 oracle/_ref/acceptance_b200 > $OUT/acceptance_b200.txt 2>&1; echo "rc $?" >> $OUT/acceptance_b200.txt
timeout 600 oracle/_ref/gpu_criteria > $OUT/gpu_criteria.txt 2>&1; echo "rc $?" >> $OUT/gpu_criteria.txt
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
SYSTEM=katsura12.sys PREC=qd MAX_NEWTON=4 PATHS=4096 OFFSET=0 SKIP=200 bash scripts/gpu_round.sh r02f/qd prof:lsq_coop
tail -3 $OUT/pytest_gpu.log; cat $OUT/smoke.log; tail -c 300 $OUT/bench.json
