"""Config 0 / 1 step times (65,536 P4 tets, mixed) + mass sweep K2 times for the loaded library."""
import json, sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2410_12614_b200 as mp
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
verts, _ = mp.gen_tets(0, 1, 65536)
vd = torch.from_numpy(verts).to(dev)
out = {}
for form in (0, 1):
    s = mp.make_setup(4, mp.mode_config("mixed", form, geometry_fp64=(form == 1)))
    s.reserve(65536)
    o = torch.empty((65536, s.n_phi ** 2), dtype=torch.float32, device=dev)
    out[f"config{form}_ms"] = round(bench.timed_ms(torch, lambda: s.cell_matrices(vd, None, mp.CoefKind.sincosexp, out=o), flush=flush), 4)
only = {(p, 0, "mixed") for p in (3, 4, 5)} | {(2, 1, "mixed")}
for r in bench.run_sweep(mp, torch, dev, only=only):
    out[f"p{r['p']}_{r['form']}_k2_ms"] = round(r["kernels_ms"][1], 4)
print(json.dumps(out))
