"""A/B of the fp32-mode GEMM: digest of the cell matrices and time per shape; run once per library
(MPFEM_B200_LIB) and compare (same accumulation order, same bits)."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_12614_b200 as mp
res = {"lib": os.environ.get("MPFEM_B200_LIB", "default").split("/")[-1], "cases": []}
for p, form, n in [(4, 1, 65536), (4, 0, 65536), (1, 1, 100000), (2, 1, 50001), (3, 0, 33333), (5, 1, 9000), (6, 0, 5000), (8, 1, 777), (4, 1, 127), (4, 1, 129)]:
    v, _ = mp.gen_tets(0, 3, n)
    vd = torch.from_numpy(v).cuda()
    s = mp.make_setup(p, mp.mode_config("fp32", form))
    s.reserve(n)
    out, fl = s.cell_matrices(vd, None, mp.CoefKind.sincosexp, want_flags=True)
    torch.cuda.synchronize()
    dig = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        s.cell_matrices(vd, None, mp.CoefKind.sincosexp, out=out)
    e0.record()
    for _ in range(5):
        s.cell_matrices(vd, None, mp.CoefKind.sincosexp, out=out)
    e1.record(); torch.cuda.synchronize()
    res["cases"].append({"p": p, "form": form, "n": n, "path": s.path, "flags": int(fl), "digest": dig, "ms": round(e0.elapsed_time(e1) / 5, 4)})
    del s, out, vd
print(json.dumps(res))
