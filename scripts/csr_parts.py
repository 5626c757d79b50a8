"""Breakdown of the CSR pattern + scatter plan build at BASELINE config 4 (96^3 x 6 tets)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, paper_2410_12614_b200 as mp
from paper_2410_12614_b200 import assembly as am
from paper_2410_12614_b200 import lib, _ptr, check
n = int(os.environ.get("N", "96"))
verts, cells = mp.structured_tet_mesh(n, n, n, 1.0, 0.15, 1)
cdev = torch.from_numpy(cells).cuda()
def ev(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3, r
for p in (2, 3):
    dm = am.build_dofmap(p, cdev, verts.shape[0]); torch.cuda.synchronize()
    t_inc, _ = ev(lambda: am.incidence(dm))
    row_ptr = torch.empty(dm.n_dofs + 1, dtype=torch.int64, device="cuda")
    nnz = C.c_int64(0)
    t_cnt, _ = ev(lambda: check(lib().mpfem_b200_csr_pattern(_ptr(dm.cell_dofs), dm.n_cells, dm.n_local, dm.n_dofs, _ptr(row_ptr), None, C.byref(nnz), None)))
    col = torch.empty(nnz.value, dtype=torch.int32, device="cuda")
    t_fill, _ = ev(lambda: check(lib().mpfem_b200_csr_pattern(_ptr(dm.cell_dofs), dm.n_cells, dm.n_local, dm.n_dofs, _ptr(row_ptr), _ptr(col), C.byref(nnz), None)))
    nk = dm.n_cells * dm.n_local ** 2
    pos = torch.empty(nk, dtype=torch.int32, device="cuda")
    t_pos, _ = ev(lambda: check(lib().mpfem_b200_scatter_plan(_ptr(dm.cell_dofs), dm.n_cells, dm.n_local, dm.n_dofs, _ptr(row_ptr), _ptr(col), _ptr(pos), None, None, None)))
    seg = torch.empty(nnz.value + 1, dtype=torch.int64, device="cuda"); perm = torch.empty(nk, dtype=torch.int32, device="cuda")
    t_plan, _ = ev(lambda: check(lib().mpfem_b200_scatter_plan(_ptr(dm.cell_dofs), dm.n_cells, dm.n_local, dm.n_dofs, _ptr(row_ptr), _ptr(col), _ptr(pos), _ptr(seg), _ptr(perm), None)))
    t_all, _ = ev(lambda: am.csr_pattern(dm))
    print(f"p={p} n_dofs={dm.n_dofs} nnz={nnz.value} incidence={t_inc:.1f} count={t_cnt:.1f} fill={t_fill:.1f} "
          f"pos_map={t_pos:.1f} full_plan={t_plan:.1f} csr_pattern_total={t_all:.1f} ms", flush=True)
    del pos, seg, perm, col
    torch.cuda.empty_cache()
