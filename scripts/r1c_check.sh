set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/b.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/b.json'))
for r in d['assembly']['results']: print(r['p'], 'fp32 %.3f ms (%.3f)  fp64 %.3f ms (%.3f) atomic %.3f pattern %.1f' % (r['assemble_fp32_ms'], r['assemble_fp32_hbm_frac'], r['assemble_fp64_ms'], r['assemble_fp64_hbm_frac'], r['assemble_atomic_fp32_ms'], r['csr_pattern_ms']))"
