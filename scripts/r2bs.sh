#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_action.py tests/test_gpu_box.py tests/test_gpu_reference_suite.py -m gpu -x -q > $OUT/pytest_action.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_action.log
echo "shipped (NB=2 Poisson, 1 mass)"; timeout 300 python scripts/action_sweep.py 2>&1 | tail -1
