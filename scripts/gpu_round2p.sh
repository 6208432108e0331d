#!/bin/bash
OUT=gpurun_out/r2p
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python scripts/measure_configs.py --only cyclic8_d cyclic8_dd cyclic10_d cyclic10_dd katsura12_qd > $OUT/configs.jsonl 2> $OUT/configs.err
tail -3 $OUT/pytest_gpu.log; cat $OUT/smoke.log; tail -c 300 $OUT/bench.json
