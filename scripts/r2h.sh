#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
gcc -O1 -o /tmp/dg_test scripts/dbg/dg_test.c -Lpaper_2410_12614_b200/lib -lmpfem_b200 && LD_LIBRARY_PATH=paper_2410_12614_b200/lib CUDA_LAUNCH_BLOCKING=1 /tmp/dg_test
for c in "shared entries" "coordinate export" "mismatched" "global error" "continuous dofmap"; do oracle/_ref/shimtests/ref_tests_b200 "$c" 2>&1 | tail -3; done
timeout 300 python scripts/k12_time.py 2>&1 | head -3
timeout 900 python -m pytest tests/test_gpu_cells.py -m gpu -q -x -k "within_bound or full_config or batch or edge" > $OUT/pytest_cells.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" $OUT/pytest_cells.log | tail -20
