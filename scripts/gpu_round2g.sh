#!/bin/bash
mkdir -p gpurun_out/r2g
O=gpurun_out/r2g/ab.txt
AB_TIMING=0 python scripts/ab.py cyclic10 dd 868928 262144 PP200_FUSED=0,1 > $O 2>&1
python scripts/ab.py cyclic10 dd 868928 262144 PP200_FUSED=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_FUSED=0,1 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 868928 262144 PP200_FUSED=1 PP200_GRAPH_TRIPS=4,16,64 >> $O 2>&1
cat $O
