"""A/B of the fused small-p kernel: digest of the cell matrices and time per shape; run once per
library (MPFEM_B200_LIB) and compare (upper-triangle accumulation mirrors bit for bit)."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_12614_b200 as mp
res = {"lib": os.environ.get("MPFEM_B200_LIB", "default").split("/")[-1], "cases": []}
rng = np.random.default_rng(5)
for p, form, mode, n, ck in [(1, 1, "mixed", 4000000, "sincosexp"), (1, 0, "mixed", 4000000, "sincosexp"), (2, 0, "mixed", 2000000, "sincosexp"),
                             (1, 1, "mixed_bf16", 100001, "sincosexp"), (2, 0, "mixed_bf16", 99999, "one"), (2, 0, "fp32", 50000, "sincosexp"),
                             (1, 1, "fp32", 50000, "nodal"), (2, 0, "mixed", 50000, "nodal")]:
    v, _ = mp.gen_tets(0, 3, n)
    vd = torch.from_numpy(v).cuda()
    s = mp.make_setup(p, mp.mode_config(mode, form))
    s.reserve(n)
    kind = getattr(mp.CoefKind, ck)
    coef = None
    if ck == "nodal":
        coef = torch.from_numpy(rng.uniform(0.5, 2.0, size=(n, s.n_phi))).cuda()
    out, fl = s.cell_matrices(vd, None, kind, coef, want_flags=True)
    torch.cuda.synchronize()
    dig = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        s.cell_matrices(vd, None, kind, coef, out=out)
    e0.record()
    for _ in range(5):
        s.cell_matrices(vd, None, kind, coef, out=out)
    e1.record(); torch.cuda.synchronize()
    res["cases"].append({"p": p, "form": form, "mode": mode, "coef": ck, "n": n, "path": s.path, "flags": int(fl), "digest": dig, "ms": round(e0.elapsed_time(e1) / 5, 4)})
    del s, out, vd
print(json.dumps(res))
