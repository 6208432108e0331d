#!/bin/bash
mkdir -p gpurun_out/r2d
O=gpurun_out/r2d/ab.txt
timeout 300 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_COOP_GROUP=32,8,4 > $O 2>&1
timeout 200 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_COOP_GROUP=8 PP200_COOP_GROUP_EVAL=8 >> $O 2>&1
timeout 300 python scripts/ab.py cyclic8 qd 0 2048 PP200_COOP_GROUP=32,8,4 >> $O 2>&1
timeout 200 python scripts/ab.py cyclic10 dd 1000000 4096 PP200_COOP_GROUP=32,8 >> $O 2>&1
timeout 300 python scripts/ab.py rand32 dd 0 8192 PP200_FORCE_COOP=0,1 >> $O 2>&1
timeout 200 python scripts/ab.py rand32 d 0 16384 PP200_FORCE_COOP=0,1 >> $O 2>&1
timeout 400 python scripts/ab.py rand32 qd 0 64 PP200_COOP_GROUP=32 >> $O 2>&1
cat $O
