set -u
mkdir -p gpurun_out
timeout 600 python bench.py --no-assembly --no-cpu-baseline --robustness --steps 100 > gpurun_out/bm.json 2> gpurun_out/bm.err; echo "rc=$?"; tail -3 gpurun_out/bm.err
python -c "
import json;d=json.load(open('gpurun_out/bm.json'))
print(d['value'], d['kernels_ms'])
for r in d['modes']: print(r)
for r in d['robustness']: print(r)"
