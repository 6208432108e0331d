#!/bin/bash
OUT=gpurun_out/r2m
mkdir -p $OUT
timeout 900 python bench.py --paths 393216 --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_393k.json 2>&1
timeout 900 python bench.py --paths 524288 --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_524k.json 2>&1
tail -c 400 $OUT/bench_393k.json; tail -c 400 $OUT/bench_524k.json
