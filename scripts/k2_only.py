"""Runs K1+K2 for one config a few times (for ncu captures of K2)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, paper_2410_12614_b200 as mp
form = int(os.environ.get("FORM", "0")); p = int(os.environ.get("P", "4"))
v, _ = mp.gen_tets(0, 1, 65536); vd = torch.from_numpy(v).cuda()
s = mp.make_setup(p, mp.KernelConfig(form=form, u_p=2, u_g=3, u_q=2, u_s=1))
for _ in range(3):
    s.cell_matrices(vd, None, 1)
torch.cuda.synchronize()
print("ok")
