#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 300 compute-sanitizer --print-limit 5 oracle/_ref/shimtests/ref_tests_b200 "discontinuous" > $OUT/sanitizer.txt 2>&1; echo "san rc=$?"; head -60 $OUT/sanitizer.txt
timeout 900 python -m pytest tests/test_gpu_cells.py -m gpu -q -x > $OUT/pytest_cells.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" $OUT/pytest_cells.log | tail -20
timeout 600 python bench.py --steps 30 --no-assembly --no-action --no-hex --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("headline", d["value"], d["ms_per_step"], d["kernels_ms"])
for m in d.get("modes", []): print(m["config"], m["mode"], round(m["ms"], 4), m["max_err_over_u_s"])
PY
