#!/bin/bash
mkdir -p gpurun_out/r2t
O=gpurun_out/r2t/ab.txt
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2000000 393216 PP200_STAGE_TABLES=0,1 > $O 2>&1
python scripts/ab.py cyclic10 dd 868928 262144 PP200_STAGE_TABLES=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_STAGE_TABLES=0,1 >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -k "staged or l2hint or production" -q >> $O 2>&1
cat $O
