#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 oracle/_ref/shimtests/ref_tests_b200 > $OUT/ref_tests_b200.txt 2>&1; echo "ref_tests_b200 rc=$?"; cat $OUT/ref_tests_b200.txt | tail -40
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" $OUT/pytest_gpu.log | tail -25
