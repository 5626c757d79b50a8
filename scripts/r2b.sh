#!/bin/bash
# Round-2b: GPU tests after the workspace / deferred-error refactor, store-stream probes,
# HBM direction probe, a short bench.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/sp2 scripts/store_probe2.cu && timeout 120 /tmp/sp2 > $OUT/store_probe2.txt 2>&1; cat $OUT/store_probe2.txt
timeout 120 python scripts/hbm_probe.py > $OUT/hbm_probe.txt 2>&1; cat $OUT/hbm_probe.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 50 --no-assembly --no-action --no-hex --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; head -c 1500 $OUT/bench.json
