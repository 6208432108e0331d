#!/bin/bash
mkdir -p gpurun_out/r2s
O=gpurun_out/r2s/ab.txt
python scripts/ab.py cyclic10 dd 868928 262144 PP200_LSQ_L2HINT=0,1 > $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2000000 393216 PP200_LSQ_L2HINT=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_LSQ_L2HINT=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2000000 393216 PP200_STAGE_TABLES=0,1 >> $O 2>&1
python scripts/ab.py cyclic10 dd 868928 262144 PP200_STAGE_TABLES=0,1 >> $O 2>&1
PP200_LSQ_L2HINT=1 PATHS=131072 SKIP=10 bash scripts/gpu_round.sh r2s prof:lsq_trip
timeout 600 python -m pytest tests/test_gpu_parity.py -k "l2hint or staged" -q >> $O 2>&1
cat $O
