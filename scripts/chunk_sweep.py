import os, sys, json, subprocess
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
res = {}
for ch in ["1", "2", "3", "4", "8"]:
    env = dict(os.environ, MPFEM_B200_CHUNKS=ch)
    out = subprocess.run([sys.executable, "bench.py", "--steps", "100", "--no-cpu-baseline"], env=env, capture_output=True, text=True).stdout
    d = json.loads(out.strip().splitlines()[-1])
    res[ch] = (d["ms_per_step"], d["kernels_ms"])
    print(ch, res[ch], flush=True)
