#!/bin/bash
# PDL A/B: cell-kernel tests + bench with modes/assembly (no CPU baseline)
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_cells.py tests/test_gpu_assembly.py tests/test_gpu_box.py -m gpu -x -q > $OUT/pytest_pdl.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_pdl.log
timeout 900 python bench.py --no-cpu-baseline --no-action --no-hex > $OUT/bench_pdl.json 2> $OUT/bench_pdl.err; echo "bench rc=$?"; tail -2 $OUT/bench_pdl.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_pdl.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kernels_ms'])
print([(m['config'],m['mode'],round(m['ms'],4)) for m in d['modes']])
for r in d['assembly']['results']: print(r['p'], r['cell_kernels_ms'], r['fused_kernels_atomic_scatter_fp32_ms'])
PY
