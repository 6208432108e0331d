#!/bin/bash
# Validation of a kernel change: parity tests, steady-state trip timing, complex-double configs
# and ncu, bench.  bash scripts/validate_round.sh TAG
TAG=${1:-val}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "modes or properties or bench_eval or track_bitwise" > $OUT/pytest.log 2>&1
printf "512 128 main 128\n" | PATHS=131072 bash scripts/exp_trips.sh $TAG
timeout 900 python scripts/measure_configs.py --only cyclic8_d cyclic10_d rand32_d cyclic10_dd > $OUT/configs.jsonl 2> $OUT/configs.err
PREC=d PATHS=524288 SKIP=10 bash scripts/gpu_round.sh ${TAG}_d prof:lsq_trip prof:ctrl_eval_trip
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
