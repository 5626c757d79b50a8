#!/bin/bash
set -u
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cells.py tests/test_gpu_bounds.py -m gpu -x -q > $OUT/pytest_cells.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_cells.log
timeout 900 python bench.py --steps 50 --no-cpu-baseline --no-assembly --no-action --no-hex > $OUT/bench_modes.json 2> $OUT/bench_modes.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_modes.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kernels_ms'])
for m in d['modes']:
    print(m['config'], m['mode'], round(m['ms'], 4))
PY
timeout 600 python scripts/kernel_zoo.py mass_k2 1 > $OUT/zoo_mass_k2.plain 2>&1 && timeout 900 ncu --set full --clock-control none -k "regex:cellmat_tcs" -c 1 -o $OUT/zoo_mass_k2 -f python scripts/kernel_zoo.py mass_k2 1 > $OUT/zoo_mass_k2.ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/zoo_mass_k2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_write.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active 2>/dev/null | tail -2
