"""Timeline of one concurrent K1/K2 call (MPFEM_B200_TRACE=1): spans, overlap, residency."""
import os, sys, json
os.environ["MPFEM_B200_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_12614_b200 as mp

cfg = mp.KernelConfig(form=1, u_p=2, u_g=3, u_q=2, u_s=1, engine=0)
s = mp.make_setup(4, cfg)
n = 65536
verts, _ = mp.gen_tets(0, 1, n)
vd = torch.from_numpy(verts).cuda()
out = torch.empty((n, 1225), dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    s.cell_matrices(vd, None, 1, out=out)
flush.zero_()
s.cell_matrices(vd, None, 1, out=out)
torch.cuda.synchronize()
k1, k2 = s.debug_trace()
t0 = min(k1[:, 0].min(), k2[:, 0].min())
k1 = k1.astype(np.float64); k2 = k2.astype(np.float64)
k1[:, :2] -= t0; k2[:, :2] -= t0
k1[:, :2] /= 1e3; k2[:, :2] /= 1e3
res = {"k1_ctas": len(k1), "k2_ctas": len(k2),
       "k1_start_us": [k1[:, 0].min(), float(np.median(k1[:, 0])), k1[:, 0].max()],
       "k1_end_us": [k1[:, 1].min(), float(np.median(k1[:, 1])), k1[:, 1].max()],
       "k2_start_us": [k2[:, 0].min(), float(np.median(k2[:, 0])), k2[:, 0].max()],
       "k2_end_us": [k2[:, 1].min(), float(np.median(k2[:, 1])), k2[:, 1].max()],
       "k1_sms": len(set(k1[:, 2].astype(int))), "k2_sms": len(set(k2[:, 2].astype(int)))}
print(json.dumps(res, indent=1))

# clocks / power under a sustained loop of the same call
import subprocess, time
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                      "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
t = time.time()
while time.time() - t < 2.0:
    for _ in range(50):
        s.cell_matrices(vd, None, 1, out=out)
    torch.cuda.synchronize()
p.terminate()
lines = p.stdout.read().strip().splitlines()
print("clocks/power samples (last 8):", lines[-8:])
