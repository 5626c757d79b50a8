#!/bin/bash
set -u
OUT=gpurun_out
timeout 600 python scripts/fused_ab.py > $OUT/fused_new.json 2> $OUT/fused_new.err; echo "new rc=$?"; tail -2 $OUT/fused_new.err
MPFEM_B200_LIB=$PWD/paper_2410_12614_b200/lib/diag/libfusedbase.so timeout 600 python scripts/fused_ab.py > $OUT/fused_base.json 2> $OUT/fused_base.err; echo "base rc=$?"; tail -2 $OUT/fused_base.err
python - <<'PY'
import json
a = json.loads(open('gpurun_out/fused_new.json').read().strip().splitlines()[-1])
b = json.loads(open('gpurun_out/fused_base.json').read().strip().splitlines()[-1])
for x, y in zip(a['cases'], b['cases']):
    print(x['p'], x['form'], x['mode'], x['coef'], x['n'], 'path', x['path'], 'same bits' if x['digest'] == y['digest'] and x['flags'] == y['flags'] else 'DIFFERENT', 'new', x['ms'], 'base', y['ms'])
PY
timeout 900 python -m pytest tests/test_gpu_cells.py -m gpu -x -q 2>&1 | tail -2
