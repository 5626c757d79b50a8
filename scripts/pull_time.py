"""Times the config-4 scatter variants (plan-based deterministic, atomic, row pull) with CUDA events.
usage: pull_time.py [p ...]   (MPFEM_B200_LIB selects a library variant)"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_12614_b200 as mp
from paper_2410_12614_b200 import assembly as am
ps = [int(a) for a in sys.argv[1:]] or [2, 3]
n = 96
verts, cells = mp.structured_tet_mesh(n, n, n, 1.0, 0.15, 1)
vd = torch.from_numpy(verts).cuda()
cd = torch.from_numpy(cells).cuda()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for p in ps:
    dm = am.build_dofmap(p, cd, verts.shape[0])
    pat = am.csr_pattern(dm)
    s = mp.make_setup(p, mp.mode_config("mixed_bf16", mp.FormKind.poisson))
    local = s.cell_matrices(vd, cd, mp.CoefKind.sincosexp)
    res = {"p": p, "lib": os.environ.get("MPFEM_B200_LIB", "default").split("/")[-1]}
    for fmt, name in ((2, "fp32"), (3, "fp64")):
        vals = torch.empty(pat.nnz, dtype=torch.float32 if fmt == 2 else torch.float64, device="cuda")
        res[f"pull_{name}_ms"] = round(timed(lambda: am.assemble_matrix(local, dm, pat, fmt, am.DETERMINISTIC, values=vals, pull=True)), 3)
        if "--all" in os.environ.get("PULL_TIME_ARGS", ""):
            res[f"plan_{name}_ms"] = round(timed(lambda: am.assemble_matrix(local, dm, pat, fmt, am.DETERMINISTIC, values=vals, pull=False)), 3)
        del vals
    print(json.dumps(res), flush=True)
    del dm, pat, s, local
    torch.cuda.empty_cache()
