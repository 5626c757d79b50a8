set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ; tail -3 gpurun_out/pytest_gpu.log
for st in 1 0; do
MPFEM_B200_STAGED_EPI=$st timeout 100 python bench.py --no-assembly --no-cpu-baseline --steps 200 > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('staged=$st', d['value'], d['ms_per_step'],d['kernels_ms'], d['accuracy']['max_err_rel'])"
MPFEM_B200_STAGED_EPI=$st timeout 300 python scripts/sweep_mixed.py 3 4 5 8 2>&1 | cut -c1-100,300-420
done
