"""Runs one hot-path kernel family in isolation (for `ncu --set full` captures of every kernel
DESIGN.md cites). usage: python scripts/kernel_zoo.py KIND [reps]

KIND:
  mass_k2      config 0: 65,536 P4 tets, mass, mixed (fp16 storage), c(x) -> K1 + K2 (tcgen05)
  poisson_k2   config 1: the headline step (K1 + K2)
  simt_f32     config 1 in fp32 mode (FFMA GEMM)
  simt_f64     config 1 in fp64 mode (fp64 GEMM)
  fused_p1     p = 1 Poisson mixed, 4M cells (one-thread-per-cell fused kernel)
  action       config 1 as action_kernel (Algorithm 2), mixed
  bounds       kernel_bounds on 4,096 config-1 cells
  asm_p2/asm_p3  config 4 (96^3 x 6 tets): dofmap, CSR pattern + plan, deterministic / atomic
               scatter, fused kernel + scatter
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_12614_b200 as mp  # noqa: E402
from paper_2410_12614_b200 import assembly as am  # noqa: E402


def main():
    kind = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda", 0)
    if kind in ("mass_k2", "poisson_k2", "simt_f32", "simt_f64", "action", "bounds"):
        v, _ = mp.gen_tets(0, 1, 65536)
        vd = torch.from_numpy(v).to(dev)
        form = 0 if kind == "mass_k2" else 1
        mode = {"simt_f32": "fp32", "simt_f64": "fp64"}.get(kind, "mixed")
        cfg = mp.mode_config(mode, form, geometry_fp64=(form == 1))
        if kind == "action":
            cfg.mode = mp.ModeKind.action
            s = mp.make_setup(4, cfg)
            w = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (65536, s.n_phi))).to(dev)
            for _ in range(reps):
                mp.action_kernel(s, vd, w, coef_kind=mp.CoefKind.sincosexp)
        elif kind == "bounds":
            s = mp.make_setup(4, cfg)
            for _ in range(reps):
                s.cell_bounds(vd[:4096], coef_kind=mp.CoefKind.sincosexp)
        else:
            s = mp.make_setup(4, cfg)
            s.reserve(65536)
            for _ in range(reps):
                s.cell_matrices(vd, None, mp.CoefKind.sincosexp)
    elif kind == "fused_p1":
        n = 1 << 22
        v, _ = mp.gen_tets(0, 2, n)
        vd = torch.from_numpy(v).to(dev)
        s = mp.make_setup(1, mp.mode_config("mixed", 1))
        for _ in range(reps):
            s.cell_matrices(vd, None, mp.CoefKind.sincosexp)
    elif kind in ("asm_p2", "asm_p3"):
        p = 2 if kind == "asm_p2" else 3
        verts, cells = mp.structured_tet_mesh(96, 96, 96, 1.0, 0.15, 1)
        vd = torch.from_numpy(verts).to(dev)
        cd = torch.from_numpy(cells).to(dev)
        dm = am.build_dofmap(p, cd, verts.shape[0])
        pat = am.csr_pattern(dm)
        s = mp.make_setup(p, mp.mode_config("mixed_bf16", 1))
        s.reserve(cells.shape[0])
        local = s.cell_matrices(vd, cd, mp.CoefKind.sincosexp)
        vals = torch.zeros(pat.nnz, dtype=torch.float32, device=dev)
        for _ in range(reps):
            am.assemble_matrix(local, dm, pat, am.FP32, am.DETERMINISTIC, values=vals)
            am.assemble_matrix(local, dm, pat, am.FP32, am.ATOMIC, values=vals)
            am.assemble_cells(s, vd, cd, dm, pat, am.FP32, mp.CoefKind.sincosexp, values=vals)
    else:
        raise SystemExit(f"unknown kind {kind}")
    torch.cuda.synchronize()
    print("ok", kind)


if __name__ == "__main__":
    main()
