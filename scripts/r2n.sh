#!/bin/bash
set -u
timeout 600 oracle/_ref/shimtests/ref_tests_b200 2>&1 | tail -40; echo "rc=${PIPESTATUS[0]}"
