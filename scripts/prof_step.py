"""One config-1 step (unchunked) for ncu captures: python scripts/prof_step.py [p] [form] [mode]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2410_12614_b200 as mp
p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
form = int(sys.argv[2]) if len(sys.argv) > 2 else 1
mode = sys.argv[3] if len(sys.argv) > 3 else "mixed64g"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 65536
if mode == "mixed64g":
    cfg = mp.KernelConfig(form=form, u_p=2, u_g=3, u_q=2, u_s=1)
else:
    cfg = mp.mode_config(mode, form)
v, _ = mp.gen_tets(0, 1, n)
vd = torch.from_numpy(v).cuda()
s = mp.make_setup(p, cfg)
s.set_timing(True)  # one chunk: K1 then K2
for _ in range(3):
    out = s.cell_matrices(vd, None, 1)
torch.cuda.synchronize()
print("timings ms", s.last_timings())
