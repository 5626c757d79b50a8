import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, paper_2410_12614_b200 as mp
v, _ = mp.gen_tets(0, 1, 3000); vd = torch.from_numpy(v).cuda()
for form in (0, 1):
    s = mp.make_setup(4, mp.KernelConfig(form=form, u_p=2, u_g=3, u_q=2, u_s=1))
    a = s.cell_matrices(vd, None, 1); torch.cuda.synchronize()
    print("form", form, "ok", float(a.abs().max()), flush=True)
