#!/bin/bash
mkdir -p gpurun_out/r2i
O=gpurun_out/r2i/ab.txt
python scripts/ab.py cyclic10 dd 868928 262144 PP200_LSQ_PRE=0,1 > $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2384256 262144 PP200_LSQ_PRE=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_LSQ_PRE=0,1 >> $O 2>&1
cat $O
