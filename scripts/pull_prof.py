"""One config-4 row-pull deterministic assembly (P3 by default) for ncu captures.
usage: pull_prof.py [p] [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_12614_b200 as mp
from paper_2410_12614_b200 import assembly as am
p = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 96
verts, cells = mp.structured_tet_mesh(n, n, n, 1.0, 0.15, 1)
vd = torch.from_numpy(verts).cuda()
cd = torch.from_numpy(cells).cuda()
dm = am.build_dofmap(p, cd, verts.shape[0])
pat = am.csr_pattern(dm)
s = mp.make_setup(p, mp.mode_config("mixed_bf16", mp.FormKind.poisson))
local = s.cell_matrices(vd, cd, mp.CoefKind.sincosexp)
vals = torch.empty(pat.nnz, dtype=torch.float32, device="cuda")
for _ in range(2):
    am.assemble_matrix(local, dm, pat, 2, am.DETERMINISTIC, values=vals, pull=True)
torch.cuda.synchronize()
print("ok", pat.nnz)
