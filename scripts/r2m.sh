#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fpp scripts/fp_peaks.cu && timeout 120 /tmp/fpp | tee $OUT/fp_peaks.json
timeout 300 python scripts/k12_time.py 2>&1 | head -3
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" $OUT/pytest_gpu.log | tail -20
timeout 600 python bench.py --steps 30 --no-assembly --no-action --no-hex --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("headline", d["value"], d["ms_per_step"], d["kernels_ms"])
for m in d.get("modes", []): print(m["config"], m["mode"], round(m["ms"], 4), m["max_err_over_u_s"])
PY
