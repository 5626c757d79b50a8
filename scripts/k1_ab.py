"""K1 / K2 times of configs 0 and 1 for the library at MPFEM_B200_LIB (A/B of diagnostic builds)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_2410_12614_b200 as mp
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
v, _ = mp.gen_tets(0, 1, 65536)
vd = torch.from_numpy(v).cuda()
for form, g64 in ((0, False), (1, True)):
    s = mp.make_setup(4, mp.mode_config("mixed", form, geometry_fp64=g64))
    s.reserve(65536)
    out = torch.empty((65536, s.n_phi ** 2), dtype=torch.float32, device="cuda")
    for _ in range(3): s.cell_matrices(vd, None, 1, out=out)
    s.set_timing(True)
    k1, k2 = [], []
    for _ in range(20):
        flush.zero_(); s.cell_matrices(vd, None, 1, out=out); t = s.last_timings(); k1.append(t[0]); k2.append(t[1])
    print(os.environ.get("MPFEM_B200_LIB", "default").split("/")[-1], "form", form, "k1 %.1f us k2 %.1f us" % (np.median(k1) * 1e3, np.median(k2) * 1e3), flush=True)
