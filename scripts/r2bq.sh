#!/bin/bash
# K2-s bulk-copy store path: cell tests + modes table
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_cells.py tests/test_gpu_box.py tests/test_gpu_bounds.py -m gpu -x -q > $OUT/pytest_bulk.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_bulk.log
timeout 900 python bench.py --no-cpu-baseline --no-action --no-hex --no-assembly > $OUT/bench_bulk.json 2> $OUT/bench_bulk.err; echo "bench rc=$?"; tail -2 $OUT/bench_bulk.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_bulk.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kernels_ms'])
print([(m['config'],m['mode'],round(m['ms'],4)) for m in d['modes']])
PY
timeout 600 python scripts/sweep_mixed.py 2 3 4 5 > $OUT/sweep_bulk.txt 2>&1; echo "sweep rc=$?"; tail -20 $OUT/sweep_bulk.txt
