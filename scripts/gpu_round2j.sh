#!/bin/bash
mkdir -p gpurun_out/r2j
O=gpurun_out/r2j/ab.txt
python scripts/ab.py cyclic10 dd 868928 262144 PP200_LSQ_FUSE=0,1 > $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2384256 262144 PP200_LSQ_FUSE=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_LSQ_FUSE=0,1 >> $O 2>&1
timeout 600 python bench.py --gpus 2 --steps 1 --warmup 1 --paths 16384 --no-cpu-baseline > gpurun_out/r2j/bench_gpus2.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -k "rand32" -q > gpurun_out/r2j/pytest_rand32.txt 2>&1
timeout 2400 python scripts/measure_configs.py --only rand32_d rand32_dd rand32_qd > gpurun_out/r2j/configs_rand32.jsonl 2> gpurun_out/r2j/configs_rand32.err
cat $O; tail -3 gpurun_out/r2j/bench_gpus2.txt gpurun_out/r2j/pytest_rand32.txt
