#!/bin/bash
mkdir -p gpurun_out/r2f
O=gpurun_out/r2f/ab.txt
AB_TIMING=0 python scripts/ab.py cyclic10 dd 868928 262144 PP200_FUSED=0,1 > $O 2>&1
python scripts/ab.py cyclic10 dd 868928 262144 PP200_FUSED=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 d 1500000 524288 PP200_FUSED=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_FUSED=0,1 >> $O 2>&1
python -m pytest tests/test_gpu_engine.py tests/test_gpu_dropin.py -q -x >> $O 2>&1
python -m pytest tests/test_gpu_parity.py -q -x -k "fused or group" >> $O 2>&1
cat $O
