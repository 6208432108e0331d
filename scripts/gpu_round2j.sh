#!/bin/bash
mkdir -p gpurun_out/r2j
O=gpurun_out/r2j/ab.txt
python scripts/ab.py cyclic10 dd 868928 262144 PP200_LSQ_FUSE=0,1 > $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2384256 262144 PP200_LSQ_FUSE=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_LSQ_FUSE=0,1 >> $O 2>&1
AB_TIMING=0 timeout 300 python scripts/ab.py rand32 d 0 65536 PP200_LSQ_QCACHE=0,1 >> $O 2>&1
AB_TIMING=0 timeout 900 python scripts/ab.py rand32 dd 0 65536 PP200_COOP_WHOLE_RUN=0,1 >> $O 2>&1
timeout 600 python bench.py --gpus 2 --steps 1 --warmup 1 --paths 16384 --no-cpu-baseline > gpurun_out/r2j/bench_gpus2.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -k "rand32 or sink or acceptance" -q > gpurun_out/r2j/pytest_sel.txt 2>&1
cat $O; tail -3 gpurun_out/r2j/bench_gpus2.txt gpurun_out/r2j/pytest_sel.txt
