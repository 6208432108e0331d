#!/bin/bash
mkdir -p gpurun_out/r2c
python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_COOP_GROUP=32,8,4 > gpurun_out/r2c/k12qd_groups.txt 2>&1
python scripts/ab.py cyclic8 qd 0 2048 PP200_COOP_GROUP=32,8,4 >> gpurun_out/r2c/k12qd_groups.txt 2>&1
python scripts/ab.py cyclic10 dd 1000000 4096 PP200_COOP_GROUP=32,8,4 >> gpurun_out/r2c/k12qd_groups.txt 2>&1
python scripts/ab.py rand32 qd 0 512 PP200_COOP_GROUP=32,8,4 >> gpurun_out/r2c/k12qd_groups.txt 2>&1
cat gpurun_out/r2c/k12qd_groups.txt
