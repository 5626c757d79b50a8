set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-modes --steps 50 > gpurun_out/b.json 2>gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'))
print(d['value'], d['kernels_ms'])
for r in d['assembly']['results']: print({k:v for k,v in r.items()})"
