import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, paper_2410_12614_b200 as mp
v, _ = mp.gen_tets(0, 1, 65536); vd = torch.from_numpy(v).cuda()
for form, kind in ((0, 0), (1, 0), (1, 1)):
    s = mp.make_setup(4, mp.KernelConfig(form=form, u_p=2, u_g=3, u_q=2, u_s=1))
    s.set_timing(True)
    for _ in range(2):
        s.cell_matrices(vd, None, kind)
    torch.cuda.synchronize()
