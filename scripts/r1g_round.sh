#!/bin/bash
# Round-1g GPU session: all GPU tests, the default bench line, config-2 sweep + config-3
# robustness tables, then the ncu captures (scripts/r1g_ncu.sh).
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err
timeout 1200 python bench.py --steps 20 --no-cpu-baseline --no-assembly --no-modes --no-action --no-hex --sweep --robustness > $OUT/sweep.json 2> $OUT/sweep.err; echo "sweep rc=$?"; tail -3 $OUT/sweep.err
bash scripts/r1g_ncu.sh
