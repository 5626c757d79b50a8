#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/sp3 scripts/store_probe3.cu && timeout 120 /tmp/sp3 > $OUT/store_probe3.txt 2>&1; cat $OUT/store_probe3.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" $OUT/pytest_gpu.log | tail -25
