#!/bin/bash
# round-2 GPU batch b: q-cache A/B for the dd solver, ncu of the quad-double tail-mode kernels
mkdir -p gpurun_out/r2b
python scripts/lsq_experiment.py dd 131072 PP200_LSQ_QCACHE=0,1 > gpurun_out/r2b/qcache.txt 2>&1
PREC=qd SYSTEM=katsura12.sys MAX_NEWTON=4 PATHS=4096 OFFSET=0 timeout 900 ncu --set full --import-source on -k regex:lsq_coop -s 20 -c 1 -o gpurun_out/r2b/k12qd_lsq_coop python scripts/profile_run.py > gpurun_out/r2b/ncu_lsq_coop.log 2>&1
PREC=qd SYSTEM=katsura12.sys MAX_NEWTON=4 PATHS=4096 OFFSET=0 timeout 900 ncu --set full --import-source on -k regex:eval_coop -s 20 -c 1 -o gpurun_out/r2b/k12qd_eval_coop python scripts/profile_run.py > gpurun_out/r2b/ncu_eval_coop.log 2>&1
cat gpurun_out/r2b/qcache.txt
