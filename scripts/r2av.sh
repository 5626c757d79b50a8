#!/bin/bash
set -u
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_distributed.py tests/test_gpu_reference_suite.py -m gpu -x -q > $OUT/pytest_asm.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_asm.log
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_assembly.py -m gpu -x -q -k "values_bitwise or row_lists" > $OUT/sanitizer_asm.log 2>&1; echo "sanitizer rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitizer_asm.log | tail -3
