"""One action_kernel call per form (configs 0/1, mixed, 65,536 P4 tets) for ncu captures."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2410_12614_b200 as mp  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "mixed"
verts, _ = mp.gen_tets(0, 1, 65536)
vd = torch.from_numpy(verts).cuda()
for form in (0, 1):
    cfg = mp.mode_config(mode, form, geometry_fp64=(form == 1))
    cfg.mode = mp.ModeKind.action
    s = mp.make_setup(4, cfg)
    w = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (65536, s.n_phi))).cuda()
    for _ in range(2):
        mp.action_kernel(s, vd, w, coef_kind=mp.CoefKind.sincosexp)
    torch.cuda.synchronize()
print("ok")
