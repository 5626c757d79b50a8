#!/bin/bash
set -u
OUT=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_assembly.py -m gpu -x -q -k "full_size" --durations=5 > $OUT/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -12 $OUT/pytest_full.log
oracle/_ref/shimtests/ref_tests_b200 > $OUT/ref_tests_b200.txt 2>&1; echo "ref tests rc=$?"; tail -1 $OUT/ref_tests_b200.txt
