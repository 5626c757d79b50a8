#!/bin/bash
set -u
OUT=gpurun_out
timeout 600 python scripts/ffma_ab.py > $OUT/ffma_new.json 2> $OUT/ffma_new.err; echo "new rc=$?"; tail -2 $OUT/ffma_new.err
MPFEM_B200_LIB=$PWD/paper_2410_12614_b200/lib/diag/libsimtbase.so timeout 600 python scripts/ffma_ab.py > $OUT/ffma_base.json 2> $OUT/ffma_base.err; echo "base rc=$?"; tail -2 $OUT/ffma_base.err
python - <<'PY'
import json
a = json.loads(open('gpurun_out/ffma_new.json').read().strip().splitlines()[-1])
b = json.loads(open('gpurun_out/ffma_base.json').read().strip().splitlines()[-1])
for x, y in zip(a['cases'], b['cases']):
    print(x['p'], x['form'], x['n'], 'path', x['path'], 'same bits' if x['digest'] == y['digest'] and x['flags'] == y['flags'] else 'DIFFERENT', 'new', x['ms'], 'base', y['ms'])
PY
