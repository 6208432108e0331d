#!/bin/bash
# tail-mode lane groups of 16 (G = 32 / 8 / 16) with the network-merge qd addition; parity of the new modes
O=gpurun_out/r2w; mkdir -p $O
AB_TIMING=0 timeout 900 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_COOP_GROUP=8,16 >> $O/ab.txt 2>&1
AB_TIMING=1 timeout 900 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_COOP_GROUP=8,16 PP200_COOP_GROUP_EVAL=32,16 >> $O/ab.txt 2>&1
AB_TIMING=0 timeout 600 python scripts/ab.py cyclic10 dd 1000000 4096 PP200_COOP_GROUP=0,16 PP200_COOP_G8_PER_SM=8,4 >> $O/ab.txt 2>&1
AB_TIMING=0 timeout 900 python scripts/ab.py cyclic10 dd 1000000 131072 PP200_COOP_GROUP=0,16 >> $O/ab.txt 2>&1
AB_TIMING=0 timeout 900 python scripts/ab.py rand32 qd 0 148 PP200_COOP_GROUP=8,16 >> $O/ab.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -k "group16 or qd" > $O/pytest.log 2>&1; echo "rc $?" >> $O/pytest.log
