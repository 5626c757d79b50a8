"""Times the action kernel (configs 0/1, mixed, 65,536 P4 tets) for the current environment."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2410_12614_b200 as mp  # noqa: E402

verts, _ = mp.gen_tets(0, 1, 65536)
vd = torch.from_numpy(verts).cuda()
res = []
for form in (0, 1):
    for mode in ("mixed", "fp64"):
        cfg = mp.mode_config(mode, form, geometry_fp64=(form == 1))
        cfg.mode = mp.ModeKind.action
        s = mp.make_setup(4, cfg)
        w = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (65536, s.n_phi))).cuda()
        out = mp.action_kernel(s, vd, w, coef_kind=mp.CoefKind.sincosexp)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            mp.action_kernel(s, vd, w, coef_kind=mp.CoefKind.sincosexp, out=out)
        e1.record()
        torch.cuda.synchronize()
        res.append(f"f{form} {mode} {e0.elapsed_time(e1) / 10 * 1e3:.0f}us")
print(os.environ.get("MPFEM_B200_ACT_THREADS", "256"), os.environ.get("MPFEM_B200_ACT_BUDGET_KB", "110"), " ".join(res))
