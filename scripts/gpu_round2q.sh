#!/bin/bash
mkdir -p gpurun_out/r2q
O=gpurun_out/r2q/ab.txt
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2000000 393216 PP200_PAIR_SLOTS=0,18944,37888 > $O 2>&1
python scripts/ab.py cyclic10 dd 2000000 393216 PP200_PAIR_SLOTS=0,18944 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic8 dd 0 40320 PP200_PAIR_SLOTS=0,18944,41000 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py katsura12 dd 0 4096 PP200_PAIR_SLOTS=0,18944 PP200_TAIL_SLOTS=0 >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -k "pair" -q >> $O 2>&1
cat $O
