#!/bin/bash
set -u
OUT=gpurun_out
timeout 600 python scripts/tc2s_ab.py > $OUT/tc2s_new.json 2> $OUT/tc2s_new.err; echo "new rc=$?"; tail -2 $OUT/tc2s_new.err
MPFEM_B200_LIB=$PWD/paper_2410_12614_b200/lib/diag/libtc2base.so timeout 600 python scripts/tc2s_ab.py > $OUT/tc2s_base.json 2> $OUT/tc2s_base.err; echo "base rc=$?"; tail -2 $OUT/tc2s_base.err
python - <<'PY'
import json
a = json.loads(open('gpurun_out/tc2s_new.json').read().strip().splitlines()[-1])
b = json.loads(open('gpurun_out/tc2s_base.json').read().strip().splitlines()[-1])
for x, y in zip(a['cases'], b['cases']):
    print(x['p'], x['form'], x['mode'], x['n'], 'same bits' if x['digest'] == y['digest'] else 'DIFFERENT', 'new', x['ms'], 'base', y['ms'])
PY
