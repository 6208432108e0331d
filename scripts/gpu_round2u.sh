#!/bin/bash
# quad-double addition by merge network: A/B against the previous build (libpp200_base.so),
# records checked against the reference goldens; then the qd GPU parity tests
O=gpurun_out/r2u; mkdir -p $O
for lib in paper_1505_00383_b200/libpp200_base.so paper_1505_00383_b200/libpp200.so; do
  echo "== $lib" >> $O/ab.txt
  AB_TIMING=0 PP200_LIB=$lib timeout 600 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_X=0 >> $O/ab.txt 2>&1
  AB_TIMING=1 PP200_LIB=$lib timeout 600 python scripts/ab.py katsura12 qd 0 4096 max_newton=4 PP200_X=0 >> $O/ab.txt 2>&1
  AB_TIMING=0 PP200_LIB=$lib timeout 600 python scripts/ab.py cyclic5 qd 0 120 PP200_X=0 >> $O/ab.txt 2>&1
  AB_TIMING=0 PP200_LIB=$lib timeout 600 python scripts/ab.py cyclic8 qd 0 1024 PP200_X=0 >> $O/ab.txt 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -k "qd" > $O/pytest_qd.log 2>&1; echo "rc $?" >> $O/pytest_qd.log
