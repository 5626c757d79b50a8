"""K1/K2 durations (library CUDA events) for configs 0/1 in the mixed modes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2410_12614_b200 as mp  # noqa: E402

verts, _ = mp.gen_tets(0, 1, 65536)
vd = torch.from_numpy(verts).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for form in (0, 1):
    for mode in ("mixed", "mixed_bf16", "fp16"):
        cfg = mp.mode_config(mode, form, geometry_fp64=(form == 1))
        s = mp.make_setup(4, cfg)
        s.reserve(65536)
        out = torch.empty((65536, s.n_phi ** 2), dtype=torch.float32, device="cuda")
        s.set_timing(True)
        k = []
        for _ in range(30):
            flush.zero_()
            s.cell_matrices(vd, None, mp.CoefKind.sincosexp, out=out)
            k.append(s.last_timings())
        k = np.median(np.array(k), axis=0)
        print(f"form {form} {mode:10s} path {s.path} K1 {k[0]*1e3:7.1f} us  K2 {k[1]*1e3:7.1f} us  launches {s.last_launch_count()}")
