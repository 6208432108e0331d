#!/bin/bash
# final round-2 evidence, part B: ncu of the dominant kernels (dd and d), the launch list, configs
PATHS=131072 SKIP=10 bash scripts/gpu_round.sh r02z prof:lsq_trip prof:ctrl_eval_trip launches
mkdir -p gpurun_out/r02z/d
PREC=d PATHS=262144 OFFSET=1500000 SKIP=10 bash scripts/gpu_round.sh r02z/d prof:lsq_trip_reg prof:ctrl_eval_trip
timeout 2400 python scripts/measure_configs.py --only cyclic5_d cyclic5_dd cyclic5_qd cyclic8_d cyclic8_dd cyclic10_d cyclic10_dd katsura12_qd rand32_d rand32_dd > gpurun_out/r02z/configs.jsonl 2> gpurun_out/r02z/configs.err
ls gpurun_out/r02z
