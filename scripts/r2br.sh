#!/bin/bash
# action kernel register tile A/B (columns per thread 1 / 2 / 4) + bitwise tests of the shipped one
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_action.py -m gpu -x -q > $OUT/pytest_action.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_action.log
echo "NB=2 (shipped)"; timeout 300 python scripts/action_sweep.py 2>&1 | tail -1
for nb in 1 4; do echo "NB=$nb"; MPFEM_B200_LIB=$PWD/paper_2410_12614_b200/lib/diag/libact_nb$nb.so timeout 300 python scripts/action_sweep.py 2>&1 | tail -1; done
