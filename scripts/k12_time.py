"""K1 / K2 durations (library CUDA events, L2 flushed) for the configs-0/1 workloads and a few
sweep points: python scripts/k12_time.py"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_2410_12614_b200 as mp

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(p, form, mode, n, g64=False):
    v, _ = mp.gen_tets(0, 1, n)
    vd = torch.from_numpy(v).cuda()
    s = mp.make_setup(p, mp.mode_config(mode, form, geometry_fp64=g64))
    s.reserve(n)
    out = torch.empty((n, s.n_phi ** 2), dtype=torch.float64 if s.path == 2 else torch.float32, device="cuda")
    for _ in range(3): s.cell_matrices(vd, None, 1, out=out)
    s.set_timing(True)
    k1, k2, tot = [], [], []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); s.cell_matrices(vd, None, 1, out=out); e1.record(); torch.cuda.synchronize()
        t = s.last_timings(); k1.append(t[0]); k2.append(t[1] if len(t) > 1 else 0); tot.append(e0.elapsed_time(e1))
    s.synchronize()
    by = n * (96 + out.element_size() * s.n_phi ** 2)
    print(f"p={p} form={form} mode={mode} n={n} path={s.path} k1={np.median(k1)*1e3:.1f}us k2={np.median(k2)*1e3:.1f}us "
          f"step={np.median(tot)*1e3:.1f}us hbm_frac={by/(np.median(tot)*1e-3)/6.5437e12:.3f}", flush=True)

run(4, 0, "mixed", 65536)
run(4, 1, "mixed", 65536, g64=True)
for p in (1, 2, 3, 4, 5, 6):
    n = (1 << 32) // (4 * mp.nphi(p) ** 2)
    run(p, 0, "mixed", n)
for p in (2, 3):
    n = (1 << 32) // (4 * mp.nphi(p) ** 2)
    run(p, 1, "mixed", n)
