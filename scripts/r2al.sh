#!/bin/bash
# warp-per-row pull kernel (rows-restricted): assembly / distributed tests, bench assembly
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_distributed.py tests/test_gpu_reference_suite.py -m gpu -x -q > $OUT/pytest_asm.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_asm.log
timeout 1200 python bench.py --steps 20 --no-cpu-baseline --no-modes --no-action --no-hex > $OUT/bench_asm.json 2> $OUT/bench_asm.err; echo "bench rc=$?"; tail -2 $OUT/bench_asm.err
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_asm.json').read().strip().splitlines()[-1])
for r in d['assembly']['results']:
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()})
PY
