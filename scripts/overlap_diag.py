"""Concurrent K1/K2 diagnostic: per-call wall time and error status at several batch sizes,
plus a comparison against the sequential path (MPFEM_B200_OVERLAP=0 in a subprocess)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_12614_b200 as mp

cfg = mp.KernelConfig(form=1, u_p=2, u_g=3, u_q=2, u_s=1, engine=0)
s = mp.make_setup(4, cfg)
res = {}
for n in [int(a) for a in (sys.argv[1:] or ["1000", "9000", "65536"])]:
    verts, _ = mp.gen_tets(0, 1, n)
    vd = torch.from_numpy(verts).cuda()
    outs = []
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        try:
            a, fl = s.cell_matrices(vd, None, 1, want_flags=True)
            torch.cuda.synchronize()
            st = "ok"
        except Exception as e:
            st = str(e)[:200]
            a = None
        outs.append((time.perf_counter() - t, st))
    ck = float(a.double().sum().item()) if a is not None else None
    res[n] = {"calls": outs, "checksum": ck}
    print(n, outs, ck, flush=True)
print(json.dumps({"overlap": os.environ.get("MPFEM_B200_OVERLAP", "1"), "res": {str(k): v for k, v in res.items()}}))
