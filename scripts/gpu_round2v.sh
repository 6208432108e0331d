#!/bin/bash
# quad-double addition variants on katsura-12 qd (production engine), twice each
O=gpurun_out/r2v; mkdir -p $O
for rep in 1 2; do
for lib in libpp200_base.so libpp200_netonly.so libpp200_seqspec.so libpp200.so; do
  echo "== $lib" >> $O/ab.txt
  AB_TIMING=0 PP200_LIB=paper_1505_00383_b200/$lib timeout 600 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_X=0 >> $O/ab.txt 2>&1
done
done
