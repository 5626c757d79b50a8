"""Quick GPU diagnostic: one small case per path vs the oracle (prints errors)."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2410_12614_b200 as mp
from oracle_lib import Oracle, MODES, nphi
O = Oracle()
v, _ = O.gen_tets(0, 1, 300)
vd = torch.from_numpy(v).cuda()
for mode in ["fp64", "fp32", "mixed", "mixed_bf16", "fp16"]:
    for form in (0, 1):
        for p in (1, 2, 4):
            up, ug, uq, us, eng = MODES[mode]
            cfg = mp.KernelConfig(form=form, u_p=up, u_g=ug, u_q=uq, u_s=us, engine=eng)
            t = time.time()
            s = mp.make_setup(p, cfg)
            a = s.cell_matrices(vd, None, 1)
            torch.cuda.synchronize()
            a = a.double().cpu().numpy()
            b, a64 = O.bound(p, form, (up, ug, uq, us, eng), v[0], 1)
            same, _ = O.bilinear(p, form, (up, ug, uq, us, eng), v[:1], 1)
            e = np.abs(a[0] - a64).max() / np.abs(a64).max()
            es = np.abs(a[0] - same[0]).max() / np.abs(a64).max()
            print(f"{mode:10s} form={form} p={p} path={s.path} err64={e:.3e} err_same={es:.3e} bound={b[0]:.3e} ratio={e/b[0]:.3f} t={time.time()-t:.2f}s", flush=True)
