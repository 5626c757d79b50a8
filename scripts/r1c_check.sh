set -u
mkdir -p gpurun_out
for lib in "" paper_2410_12614_b200/lib/diag/libtc2s7.so; do
MPFEM_B200_LIB=$lib timeout 100 python bench.py --no-assembly --no-cpu-baseline --steps 200 > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$lib'[-12:], d['value'], d['ms_per_step'],d['kernels_ms'], d['accuracy']['max_err_rel'])"
MPFEM_B200_LIB=$lib timeout 300 python scripts/sweep_mixed.py 4 5 6 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except: print(l[:200]); continue
  print(d['p'], d['form'], d['ms'], d['roofline_frac'], [round(x,3) for x in d['kernels_ms']])"
done
