set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ; tail -3 gpurun_out/pytest_gpu.log
timeout 100 python bench.py --no-assembly --no-cpu-baseline --steps 200 > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bench', d['value'], d['ms_per_step'],d['kernels_ms'])"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-assembly"
ncu --set full --clock-control none --import-source on -k regex:"geom_w" -s 4 -c 1 -o gpurun_out/k1prof -f $CMD > gpurun_out/ncu_k1.log 2>&1; echo "ncu rc=$?"
