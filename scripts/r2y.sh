#!/bin/bash
# Round-2y GPU session (re-entry baseline): full GPU tests, default bench line, config-2 sweep.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -2 $OUT/bench.err; head -c 600 $OUT/bench.json; echo
timeout 1500 python bench.py --steps 5 --sweep --robustness --no-assembly --no-action --no-hex --no-modes --no-cpu-baseline > $OUT/bench_sweep.json 2> $OUT/bench_sweep.err; echo "sweep rc=$?"; tail -2 $OUT/bench_sweep.err
