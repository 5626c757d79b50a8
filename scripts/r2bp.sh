#!/bin/bash
# compact scatter plan: assembly tests + bench assembly key
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_distributed.py -m gpu -x -q > $OUT/pytest_compact.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_compact.log
timeout 900 python bench.py --steps 50 --no-cpu-baseline --no-action --no-hex --no-modes > $OUT/bench_compact.json 2> $OUT/bench_compact.err; echo "bench rc=$?"; tail -3 $OUT/bench_compact.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_compact.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'])
for r in d['assembly']['results']: print({k:(round(v,3) if isinstance(v,float) else v) for k,v in r.items()})
PY
