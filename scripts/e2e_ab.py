"""Times the host-buffer API (config 1, 65,536 P4 tets, pinned buffers) for the loaded library."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2410_12614_b200 as mp
verts, _ = mp.gen_tets(0, 1, 65536)
cfg = mp.mode_config("mixed", 1, geometry_fp64=True)
s = mp.make_setup(4, cfg)
vp = torch.from_numpy(verts).pin_memory().numpy()
out = torch.empty((65536, s.n_phi, s.n_phi), dtype=torch.float32).pin_memory().numpy()
s.cell_matrices_host(vp, None, mp.CoefKind.sincosexp, out=out)
ref = out.copy()
import time
res = []
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        s.cell_matrices_host(vp, None, mp.CoefKind.sincosexp, out=out)
    res.append((time.perf_counter() - t0) / 10 * 1e3)
print("ms per call", [round(r, 3) for r in res], "digest", hex(int(np.bitwise_xor.reduce(ref.view(np.uint32).ravel()))))
