#!/bin/bash
mkdir -p gpurun_out/r2o
O=gpurun_out/r2o/ab.txt
python scripts/ab.py cyclic10 dd 868928 262144 PP200_STAGE_TABLES=0,1 > $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2384256 262144 PP200_STAGE_TABLES=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 d 1500000 524288 PP200_STAGE_TABLES=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_STAGE_TABLES=0,1 >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -k "staged or fuse" -q >> $O 2>&1
cat $O
