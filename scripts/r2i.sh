#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python scripts/k12_time.py 2>&1 | tee $OUT/k12.txt
timeout 900 python -m pytest tests/test_gpu_cells.py -m gpu -q -x -k "within_bound or full_config or batch or edge or high_degree" > $OUT/pytest_cells.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" $OUT/pytest_cells.log | tail -20
