#!/bin/bash
# tail-mode group thresholds for quad-double (katsura-12 qd, production engine)
O=gpurun_out/r2x; mkdir -p $O
AB_TIMING=0 timeout 900 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_COOP_G8_PER_SM=8,2,4,16 >> $O/ab.txt 2>&1
AB_TIMING=0 timeout 900 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_COOP_GROUP_EVAL=32,8 >> $O/ab.txt 2>&1
AB_TIMING=0 timeout 900 python scripts/ab.py cyclic8 qd 0 1024 PP200_COOP_G8_PER_SM=8,2 >> $O/ab.txt 2>&1
