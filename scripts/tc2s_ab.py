"""A/B of the pair kernel's output paths: prints a digest of the cell matrices of several shapes and
the K1/K2 times; run once per library (MPFEM_B200_LIB) and compare the digests (same MMAs, same bits).
usage: tc2s_ab.py"""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_12614_b200 as mp
res = {"lib": os.environ.get("MPFEM_B200_LIB", "default").split("/")[-1], "cases": []}
cases = [(4, 1, "mixed", 65536), (4, 1, "fp16", 65536), (4, 1, "mixed_bf16", 5000), (3, 1, "mixed", 70001), (5, 1, "mixed", 20000),
         (6, 1, "mixed", 9999), (6, 0, "mixed", 30000), (7, 0, "mixed_bf16", 8000), (8, 1, "mixed", 3000), (4, 1, "mixed", 255), (4, 1, "mixed", 257)]
for p, form, mode, n in cases:
    v, _ = mp.gen_tets(0, 3, n)
    vd = torch.from_numpy(v).cuda()
    s = mp.make_setup(p, mp.mode_config(mode, form))
    s.reserve(n)
    out = s.cell_matrices(vd, None, mp.CoefKind.sincosexp)
    torch.cuda.synchronize()
    dig = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        s.cell_matrices(vd, None, mp.CoefKind.sincosexp, out=out)
    e0.record()
    for _ in range(20):
        s.cell_matrices(vd, None, mp.CoefKind.sincosexp, out=out)
    e1.record(); torch.cuda.synchronize()
    res["cases"].append({"p": p, "form": form, "mode": mode, "n": n, "digest": dig, "ms": round(e0.elapsed_time(e1) / 20, 4)})
    del s, out, vd
print(json.dumps(res))
