#!/bin/bash
mkdir -p gpurun_out/r2k
O=gpurun_out/r2k/ab.txt
AB_TIMING=0 python scripts/ab.py cyclic10 dd 2384256 262144 PP200_LSQ_SPT=1,2 > $O 2>&1
python scripts/ab.py cyclic10 dd 868928 262144 PP200_LSQ_SPT=1,2 >> $O 2>&1
timeout 900 python bench.py > gpurun_out/r2k/bench.json 2> gpurun_out/r2k/bench.err
timeout 2700 python scripts/measure_configs.py --only cyclic10_dd rand32_d rand32_dd rand32_qd > gpurun_out/r2k/configs.jsonl 2> gpurun_out/r2k/configs.err
cat $O
