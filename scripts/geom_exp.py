import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, paper_2410_12614_b200 as mp
v, _ = mp.gen_tets(0, 1, 65536); vd = torch.from_numpy(v).cuda()
for ug in (3, 2):
    for kind in (0, 1):
        for form in (0, 1):
            s = mp.make_setup(4, mp.KernelConfig(form=form, u_p=2, u_g=ug, u_q=2, u_s=1))
            s.set_timing(True)
            ts = []
            for _ in range(10):
                s.cell_matrices(vd, None, kind); ts.append(s.last_timings())
            import numpy as np
            t = np.median(np.array(ts), axis=0)
            print(f"ug={ug} coef={kind} form={form} geom={t[0]*1e3:.1f}us gemm={t[1]*1e3:.1f}us", flush=True)
