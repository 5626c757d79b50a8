#!/bin/bash
set -u
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_action.py tests/test_gpu_box.py tests/test_gpu_assembly.py -m gpu -x -q > $OUT/pytest_action.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_action.log
timeout 900 python bench.py --steps 20 --no-cpu-baseline --no-assembly --no-modes --no-hex > $OUT/bench_action.json 2> $OUT/bench_action.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_action.json').read().strip().splitlines()[-1])
for m in d['action']['results']:
    print(m['config'], m['mode'], round(m['ms'], 4), 'issue_frac', round(m['issue_frac'], 3), 'bound', (m.get('bound_check') or {}).get('max_err_over_S_bound_v'))
PY
