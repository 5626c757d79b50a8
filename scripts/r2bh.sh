#!/bin/bash
# bench.py's N>1 branch, functionally: two ranks sharing the one GPU over gloo (no timing claim)
set -u
OUT=gpurun_out
MPFEM_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-modes --no-action --no-hex > $OUT/bench_n2_gloo.json 2> $OUT/bench_n2_gloo.err; echo "bench N=2 rc=$?"; tail -3 $OUT/bench_n2_gloo.err
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_n2_gloo.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('metric', 'value', 'n_gpus', 'ms_per_step', 'scaling')})
for r in d['assembly']['results']:
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()})
PY
