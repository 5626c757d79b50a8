#!/bin/bash
set -u
MALLOC_CHECK_=3 timeout 600 oracle/_ref/shimtests/ref_tests_b200 2>&1 | tail -8; echo "rc=${PIPESTATUS[0]}"
timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x 2>&1 | tail -15
