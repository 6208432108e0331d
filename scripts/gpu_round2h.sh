#!/bin/bash
mkdir -p gpurun_out/r2h
O=gpurun_out/r2h/ab.txt
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2384256 262144 PP200_TAIL_SLOTS=4736,9472,18944,37888 > $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2384256 262144 PP200_TAIL_SLOTS=18944 PP200_COOP_GROUP=4,8 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2384256 262144 PP200_COMPACT_PCT=85,90,95,98 >> $O 2>&1
AB_TIMING=0 python scripts/ab.py cyclic10 d 1500000 524288 PP200_TAIL_SLOTS=4736,18944,75776 >> $O 2>&1
cat $O
