set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ; tail -2 gpurun_out/pytest_gpu.log
timeout 100 python bench.py --no-assembly --no-cpu-baseline --steps 200 > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'], d['ms_per_step'],d['kernels_ms'], d['accuracy']['max_err_rel'])"
timeout 300 python scripts/sweep_mixed.py 2 3 4 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except: print(l[:200]); continue
  print(d['p'], d['form'], d['ms'], d['roofline_frac'], [round(x,3) for x in d['kernels_ms']])"
