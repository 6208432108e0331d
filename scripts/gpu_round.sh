#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list and full captures.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_round.sh TAG [what...]
#   what: tests smoke bench launches prof:<kernel-regex> (default: all, profiling lsq_trip)
# ncu reports are reduced to CSV pages on the box (gpurun brings back <= 64 MiB).
TAG=${1:-r01}; shift
WHAT=${@:-tests smoke bench launches prof:track_fused}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
for W in $WHAT; do
  case $W in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $OUT/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?" >> $OUT/smoke.log ;;
    bench) timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?" >> $OUT/bench.err ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
        python bench.py --steps 1 --warmup 0 --paths 8192 --no-cpu-baseline > $OUT/launches.log 2>&1 ;;
    prof:*) K=${W#prof:}
      PATHS=${PATHS:-8192} timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-0} -c 1 \
        -o $OUT/prof_$K python scripts/profile_run.py > $OUT/prof_$K.log 2>&1
      ncu -i $OUT/prof_$K.ncu-rep --page raw --csv > $OUT/prof_${K}_raw.csv 2>&1
      ncu -i $OUT/prof_$K.ncu-rep --page details --csv > $OUT/prof_${K}_details.csv 2>&1
      ncu -i $OUT/prof_$K.ncu-rep --page source --csv > $OUT/prof_${K}_source.csv 2>&1
      gzip -f $OUT/prof_${K}_source.csv
      if [ $(stat -c %s $OUT/prof_$K.ncu-rep) -gt 20000000 ]; then rm -f $OUT/prof_$K.ncu-rep; fi ;;
    run:*) eval "${W#run:}" ;;
  esac
done
ls -la $OUT
