"""K2 time vs output pitch (1225 = dense, 1228 = 16-B rows, 1280 = 512-B rows)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch, paper_2410_12614_b200 as mp
v, _ = mp.gen_tets(0, 1, 65536); vd = torch.from_numpy(v).cuda()
for form in (0, 1):
    s = mp.make_setup(4, mp.KernelConfig(form=form, u_p=2, u_g=3, u_q=2, u_s=1))
    s.set_timing(True)
    for pitch in (1225, 1228, 1232, 1280):
        out = torch.empty((65536, pitch), dtype=torch.float32, device="cuda")
        ts = []
        for _ in range(10):
            s.cell_matrices(vd, None, 1, out=out, out_pitch=pitch); ts.append(s.last_timings())
        t = np.median(np.array(ts), axis=0)
        print(f"form={form} pitch={pitch} gemm={t[1]*1e3:.1f}us", flush=True)
