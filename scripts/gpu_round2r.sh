#!/bin/bash
PATHS=131072 SKIP=10 bash scripts/gpu_round.sh r02f prof:lsq_trip prof:ctrl_eval_trip launches
