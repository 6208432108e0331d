#!/bin/bash
OUT=gpurun_out/r2l
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
POLYPATH_B200_TRACE=1 timeout 600 oracle/_ref/acceptance_b200 > $OUT/acceptance_b200.txt 2>&1; echo "rc $?" >> $OUT/acceptance_b200.txt
timeout 900 python scripts/track_full.py --prec dd > $OUT/full_cyclic10_dd.json 2> $OUT/full_dd.err
timeout 300 python scripts/track_full.py --prec d > $OUT/full_cyclic10_d.json 2> $OUT/full_d.err
tail -3 $OUT/pytest_gpu.log; cat $OUT/full_cyclic10_dd.json $OUT/full_cyclic10_d.json
