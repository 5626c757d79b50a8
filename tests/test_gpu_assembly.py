"""GPU dof map / CSR / scatter-add against the reference algorithm (oracle, pinned to the
compiled reference). Bars: dof map and sparsity bitwise; deterministic values bitwise;
atomic values within gamma_{m+1}(fmt) * sum|contrib| of the exact sum (test_assembly.cpp:165-167).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2410_12614_b200 as mp  # noqa: E402
from paper_2410_12614_b200 import assembly as am  # noqa: E402
from oracle_lib import nphi  # noqa: E402


def gpu_dofmap(p, verts, cells):
    return am.build_dofmap(p, torch.from_numpy(np.ascontiguousarray(cells)).cuda(), verts.shape[0])


@pytest.mark.parametrize("dims,p", [((3, 2, 2), 1), ((3, 2, 2), 2), ((3, 2, 2), 3), ((2, 2, 2), 4),
                                    ((2, 1, 1), 6), ((1, 1, 2), 8), ((6, 5, 4), 2), ((5, 4, 4), 3)])
def test_dofmap_bitwise(oracle, dims, p):
    verts, cells = oracle.structured_tet_mesh(*dims, 1.0, 0.15, 7)
    cd, nd, mm = oracle.build_dofmap(p, verts, cells)
    dm = gpu_dofmap(p, verts, cells)
    assert dm.n_dofs == nd and dm.max_multiplicity == mm
    assert np.array_equal(dm.cell_dofs.cpu().numpy(), cd)


def test_dofmap_known_answers(oracle):
    # test_mesh.cpp:194-199: 2x2x2 tet mesh, P1: 27 dofs, max multiplicity 24
    verts, cells = oracle.structured_tet_mesh(2, 2, 2, 1.0, 0.15, 7)
    dm = gpu_dofmap(1, verts, cells)
    assert (dm.n_dofs, dm.max_multiplicity) == (27, 24)
    # (p n + 1)^3 dofs on an n^3 Kuhn mesh
    for n, p in ((4, 2), (3, 3)):
        verts, cells = oracle.structured_tet_mesh(n, n, n, 1.0, 0.15, 3)
        assert gpu_dofmap(p, verts, cells).n_dofs == (p * n + 1) ** 3


@pytest.mark.parametrize("p,dims", [(1, (4, 3, 3)), (2, (4, 3, 3)), (3, (4, 3, 3)), (4, (2, 2, 2)),
                                    (6, (2, 2, 1)), (8, (1, 1, 1))])
def test_csr_pattern_and_values_bitwise(oracle, p, dims):
    # the row-pull kernel's variants: 16 / 8 / 4-byte copies (n_loc = 4, 20, 84 / 10 / 35, 165), 128- and
    # 256-entry chunks (n_loc <= 64 / above); p >= 6 rows exceed the shared-memory caps, so the
    # global-memory replay is exercised too. The pattern carries seg_ptr/perm so that the default
    # call takes the segment-gather kernel and pull=True the row-pull kernel.
    verts, cells = oracle.structured_tet_mesh(*dims, 1.0, 0.15, 11)
    cd, nd, _ = oracle.build_dofmap(p, verts, cells)
    dm = gpu_dofmap(p, verts, cells)
    pat = am.csr_pattern(dm, deterministic_plan=True)
    rng = np.random.default_rng(p)
    loc32 = rng.uniform(-1, 1, size=(cells.shape[0], nphi(p), nphi(p))).astype(np.float32)
    for fmt in (2, 3):
        rows, cols, vals, _ = oracle.assemble_matrix(cd, nd, loc32.astype(np.float64), fmt)
        rp = pat.row_ptr.cpu().numpy()
        assert pat.nnz == rows.size
        assert np.array_equal(np.repeat(np.arange(nd), np.diff(rp)), rows)
        assert np.array_equal(pat.col_idx.cpu().numpy(), cols)
        v = am.assemble_matrix(torch.from_numpy(loc32).cuda(), dm, pat, fmt, am.DETERMINISTIC)
        torch.cuda.synchronize()
        got = v.double().cpu().numpy()
        assert np.array_equal(got.view(np.uint64), vals.view(np.uint64)), fmt
        # the plan-free row-pull path gives the same bits
        vs = am.assemble_matrix(torch.from_numpy(loc32).cuda(), dm, pat, fmt, am.DETERMINISTIC,
                                pull=True)
        assert np.array_equal(vs.double().cpu().numpy().view(np.uint64), vals.view(np.uint64)), fmt
        # atomic mode: gamma_{m+1} * sum |contrib|
        va = am.assemble_matrix(torch.from_numpy(loc32).cuda(), dm, pat, fmt, am.ATOMIC)
        torch.cuda.synchronize()
        absum = oracle.assemble_matrix(cd, nd, np.abs(loc32.astype(np.float64)), 3)[2]
        u = 2.0**-24 if fmt == 2 else 2.0**-53
        m = 25
        assert np.all(np.abs(va.double().cpu().numpy() - vals) <= (m + 1) * u / (1 - (m + 1) * u) * absum * 2)
    # fp64 locals into fp32 values (cast at fmt, assembly.cpp:57)
    loc64 = rng.uniform(-1, 1, size=(cells.shape[0], nphi(p), nphi(p)))
    rows, cols, vals, _ = oracle.assemble_matrix(cd, nd, loc64, 2)
    for pull in (False, True):
        v = am.assemble_matrix(torch.from_numpy(loc64).cuda(), dm, pat, 2, am.DETERMINISTIC, pull=pull)
        assert np.array_equal(v.double().cpu().numpy().view(np.uint64), vals.view(np.uint64)), pull
    # patterns without seg_ptr/perm (the default) take the row-pull kernel: with its own uint16
    # position stream (pull_pos, with and without the int32 pos_map beside it) or with pos_map only
    for kw in ({}, {"pos_map": False}, {"pull_plan": False}):
        pat0 = am.csr_pattern(dm, **kw)
        assert pat0.seg_ptr is None
        assert (pat0.pull_pos is None) == (kw.get("pull_plan") is False)
        assert (pat0.pos_map is None) == (kw.get("pos_map") is False)
        for loc in (loc64, loc32):
            ref = oracle.assemble_matrix(cd, nd, loc.astype(np.float64), 2)[2]
            v = am.assemble_matrix(torch.from_numpy(loc).cuda(), dm, pat0, 2)
            assert np.array_equal(v.double().cpu().numpy().view(np.uint64), ref.view(np.uint64)), kw


def test_row_pull_row_lists_bitwise(oracle):
    """Rows-restricted row pull (the multi-GPU slab pass): a list with runs of consecutive rows,
    isolated rows and a reversed tail writes exactly those rows, bitwise the full assembly."""
    p = 3
    verts, cells = oracle.structured_tet_mesh(4, 3, 3, 1.0, 0.15, 7)
    dm = gpu_dofmap(p, verts, cells)
    pat = am.csr_pattern(dm)
    rng = np.random.default_rng(3)
    loc = torch.from_numpy(rng.uniform(-1, 1, size=(cells.shape[0], 20, 20)).astype(np.float32)).cuda()
    full = am.assemble_matrix(loc, dm, pat, 2)
    nd = dm.n_dofs
    pick = np.concatenate([np.arange(5, 75), np.arange(100, 400, 7), np.arange(nd - 40, nd)[::-1]]).astype(np.int32)
    rows = torch.from_numpy(pick).cuda()
    vals = torch.full((pat.nnz,), 123.0, dtype=torch.float32, device="cuda")
    am.assemble_matrix(loc, dm, pat, 2, rows=rows, values=vals)
    torch.cuda.synchronize()
    rp = pat.row_ptr.cpu().numpy()
    mask = np.zeros(pat.nnz, dtype=bool)
    for r in pick:
        mask[rp[r]:rp[r + 1]] = True
    got, ref = vals.cpu().numpy(), full.cpu().numpy()
    assert np.array_equal(got[mask].view(np.uint32), ref[mask].view(np.uint32))
    assert np.all(got[~mask] == 123.0)


def test_partial_cell_ranges_compose_bitwise(oracle):
    """Assembling cells [0, k) then continuing with [k, n) (accumulate) equals one pass:
    the multi-GPU interface exchange invariant."""
    p = 2
    verts, cells = oracle.structured_tet_mesh(3, 3, 4, 1.0, 0.15, 5)
    dm = gpu_dofmap(p, verts, cells)
    pat = am.csr_pattern(dm, deterministic_plan=True)
    rng = np.random.default_rng(9)
    loc = torch.from_numpy(rng.uniform(-1, 1, size=(cells.shape[0], 10, 10)).astype(np.float32)).cuda()
    full = am.assemble_matrix(loc, dm, pat, 2)
    k = cells.shape[0] // 2
    for pull in (False, True):
        part = am.assemble_matrix(loc[:k], dm, pat, 2, cell_begin=0, cell_end=k, pull=pull)
        part = am.assemble_matrix(loc[k:], dm, pat, 2, cell_begin=k, cell_end=cells.shape[0],
                                  accumulate=True, values=part, pull=pull)
        torch.cuda.synchronize()
        assert torch.equal(full.view(torch.int32), part.view(torch.int32)), pull


def test_config4_reduced_end_to_end(oracle):
    """BASELINE config 4 at 12^3 x 6 tets: GPU Poisson P2 locals (mixed) -> GPU assembly,
    bitwise equal to the reference assembly of the same locals; global Poisson rows sum to
    ~0 (constants in the kernel)."""
    n, p = 12, 2
    verts, cells = mp.structured_tet_mesh(n, n, n, 1.0, 0.15, 1)
    vd = torch.from_numpy(verts).cuda()
    cdev = torch.from_numpy(cells).cuda()
    s = mp.make_setup(p, mp.mode_config("mixed_bf16", mp.FormKind.poisson))
    loc = s.cell_matrices(vd, cdev, mp.CoefKind.sincosexp)
    dm = am.build_dofmap(p, cdev, verts.shape[0])
    pat = am.csr_pattern(dm)
    vals = am.assemble_matrix(loc, dm, pat, 3)
    torch.cuda.synchronize()
    cd, nd, _ = oracle.build_dofmap(p, verts, cells)
    assert nd == dm.n_dofs and np.array_equal(cd, dm.cell_dofs.cpu().numpy())
    rows, cols, rv, _ = oracle.assemble_matrix(cd, nd, loc.double().cpu().numpy(), 3)
    assert np.array_equal(vals.cpu().numpy().view(np.uint64), rv.view(np.uint64))
    rp = pat.row_ptr.cpu().numpy()
    rs = np.add.reduceat(rv, rp[:-1])
    scale = np.abs(rv).max()
    assert np.abs(rs).max() <= 1e-2 * scale


@pytest.mark.slow
def test_config4_full_size_p2_properties():
    """96^3 x 6 = 5,308,416 tets, P2: dof count, symmetric pattern, sampled rows."""
    n, p = 96, 2
    verts, cells = mp.structured_tet_mesh(n, n, n, 1.0, 0.15, 1)
    cdev = torch.from_numpy(cells).cuda()
    dm = am.build_dofmap(p, cdev, verts.shape[0])
    assert dm.n_dofs == (p * n + 1) ** 3 == 7189057
    pat = am.csr_pattern(dm)
    rp = pat.row_ptr
    assert int(rp[-1]) == pat.nnz
    nnz_row = (rp[1:] - rp[:-1]).double()
    assert 20 < float(nnz_row.mean()) < 40
    # pattern symmetry: multiset of (row, col) equals (col, row)
    rows = torch.repeat_interleave(torch.arange(dm.n_dofs, device="cuda"), rp[1:] - rp[:-1])
    key = rows.to(torch.int64) * dm.n_dofs + pat.col_idx.to(torch.int64)
    keyt = pat.col_idx.to(torch.int64) * dm.n_dofs + rows.to(torch.int64)
    assert torch.equal(torch.sort(key).values, torch.sort(keyt).values)


@pytest.mark.slow
def test_config4_full_size_p2_bitwise_pin(oracle):
    """BASELINE config 4 at its full size (96^3 x 6 = 5,308,416 tets, P2, Poisson, mixed-bf16
    cell kernels): the GPU dof map equals the reference restatement's (mesh.cpp:204-298) entry
    for entry, and the deterministic CSR assembly (fp32 and fp64 values) equals the reference
    assembly (assembly.cpp:41-88) bit for bit on windows of rows at the start, in the middle and
    at the end of the matrix. A window's rows are complete in the sub-assembly of exactly the
    cells incident to it, taken in ascending order, so the oracle sums each entry's contributions
    in the same order as the full assembly would; rows outside the window are ignored. Whole-
    matrix properties on top: the sum of all entries equals the sum of all local entries, and
    the Poisson rows sum to ~0."""
    n, p = 96, 2
    verts, cells = oracle.structured_tet_mesh(n, n, n, 1.0, 0.15, 1)
    cd, nd, mm = oracle.build_dofmap(p, verts, cells)
    vd = torch.from_numpy(verts).cuda()
    cdev = torch.from_numpy(cells).cuda()
    dm = am.build_dofmap(p, cdev, verts.shape[0])
    assert dm.n_dofs == nd == 7189057 and dm.max_multiplicity == mm
    assert torch.equal(dm.cell_dofs.cpu(), torch.from_numpy(cd))
    s = mp.make_setup(p, mp.mode_config("mixed_bf16", mp.FormKind.poisson))
    loc = s.cell_matrices(vd, cdev, mp.CoefKind.sincosexp).view(-1, 10, 10)
    pat = am.csr_pattern(dm)
    rp = pat.row_ptr.cpu().numpy()
    col = pat.col_idx.cpu().numpy()
    w = 20000
    for fmt in (2, 3):
        vals = am.assemble_matrix(loc, dm, pat, fmt)
        torch.cuda.synchronize()
        v = vals.double().cpu().numpy()
        for r0 in (0, nd // 2 - w // 2, nd - w):
            r1 = r0 + w
            touched = np.nonzero(((cd >= r0) & (cd < r1)).any(axis=1))[0]  # ascending cells
            lsub = loc[torch.from_numpy(touched).cuda()].double().cpu().numpy()
            rows, cols, rv, _ = oracle.assemble_matrix(cd[touched], nd, lsub, fmt)
            keep = (rows >= r0) & (rows < r1)
            a, b = rp[r0], rp[r1]
            assert keep.sum() == b - a
            assert np.array_equal(cols[keep], col[a:b])
            assert np.array_equal(rows[keep], np.repeat(np.arange(r0, r1), np.diff(rp[r0:r1 + 1])))
            assert np.array_equal(rv[keep].view(np.uint64), v[a:b].view(np.uint64)), (fmt, r0)
        if fmt == 3:
            total, ltotal = float(vals.sum()), float(loc.double().sum())
            scale = float(loc.double().abs().sum())
            assert abs(total - ltotal) <= 1e-9 * scale
            rs = torch.segment_reduce(vals, "sum", lengths=pat.row_ptr[1:] - pat.row_ptr[:-1])
            assert float(rs.abs().max()) <= 1e-2 * float(vals.abs().max())
        del vals


@pytest.mark.parametrize("mode,p", [("mixed", 2), ("mixed_bf16", 3), ("fp64", 2), ("mixed", 1)])
def test_fused_cell_kernels_scatter(oracle, mode, p):
    """assemble_cells (cell kernels fused with the atomic scatter; on the tcgen05 path K2 adds
    from TMEM) against the deterministic assembly of the same cell matrices: per entry within
    gamma_{m+1}(fmt) * sum|contrib| (test_assembly.cpp:165-167), and with cell ranges that
    compose (z-slab style)."""
    verts, cells = oracle.structured_tet_mesh(4, 3, 3, 1.0, 0.15, 11)
    dm = gpu_dofmap(p, verts, cells)
    pat = am.csr_pattern(dm)
    s = mp.make_setup(p, mp.mode_config(mode, mp.FormKind.poisson))
    vd = torch.from_numpy(verts).cuda()
    cd = torch.from_numpy(np.ascontiguousarray(cells)).cuda()
    local = s.cell_matrices(vd, cd, mp.CoefKind.sincosexp)
    ab = local.abs().double()
    for fmt in (2, 3):
        det = am.assemble_matrix(local, dm, pat, fmt, am.DETERMINISTIC).double()
        mag = am.assemble_matrix(ab.to(local.dtype), dm, pat, fmt, am.DETERMINISTIC).double()
        u = 2.0 ** -24 if fmt == 2 else 2.0 ** -53
        m = dm.max_multiplicity
        tol = (m + 1) * u / (1 - (m + 1) * u) * mag + 1e-300
        fused = am.assemble_cells(s, vd, cd, dm, pat, fmt, mp.CoefKind.sincosexp).double()
        assert bool(((fused - det).abs() <= tol).all()), (mode, fmt)
        k = cells.shape[0] // 3
        part = am.assemble_cells(s, vd, cd[:k], dm, pat, fmt, mp.CoefKind.sincosexp)
        part = am.assemble_cells(s, vd, cd[k:], dm, pat, fmt, mp.CoefKind.sincosexp, cell_begin=k,
                                 accumulate=True, values=part).double()
        assert bool(((part - det).abs() <= tol).all()), (mode, fmt)


@pytest.mark.parametrize("mode,p", [("mixed", 2), ("mixed_bf16", 3), ("fp64", 2), ("mixed", 1)])
def test_fused_scatter_vs_oracle_assembly(oracle, mode, p):
    """The fused kernel + atomic scatter against the reference assembly (oracle
    assemble_matrix, assembly.cpp:41-88) of the binary64 oracle cell matrices. Per entry:
    |fused - ref| <= gamma_{m+1}(fmt) sum|contrib| (test_assembly.cpp:165-167) plus, summed
    over the contributing cells, each cell's own S * bound_a * max|A_c| (the kernel bound of
    kernel_bounds, bounds.cpp:255-266, which the cell matrices meet)."""
    from oracle_lib import COEF_SINCOSEXP, MODES, UNIT_ROUNDOFF
    verts, cells = oracle.structured_tet_mesh(3, 3, 2, 1.0, 0.15, 13)
    cdn, nd, mm = oracle.build_dofmap(p, verts, cells)
    dm = gpu_dofmap(p, verts, cells)
    pat = am.csr_pattern(dm)
    cfg = mp.mode_config(mode, mp.FormKind.poisson)
    s = mp.make_setup(p, cfg)
    ct = (int(cfg.u_p), int(cfg.u_g), int(cfg.u_q), int(cfg.u_s), int(cfg.engine))
    us = UNIT_ROUNDOFF[int(cfg.u_s)]
    S = 4.0 if all(us > UNIT_ROUNDOFF[int(f)] for f in (cfg.u_p, cfg.u_g, cfg.u_q)) else 1.0
    a64 = np.zeros((cells.shape[0], nphi(p), nphi(p)))
    tol_loc = np.zeros_like(a64)
    for c in range(cells.shape[0]):
        b, a = oracle.bound(p, 1, ct, verts[cells[c]], COEF_SINCOSEXP)
        a64[c] = a
        tol_loc[c] = S * b[0] * np.max(np.abs(a))
    _, _, ref, _ = oracle.assemble_matrix(cdn, nd, a64, 3)
    _, _, mag, _ = oracle.assemble_matrix(cdn, nd, np.abs(a64), 3)
    _, _, cell_tol, _ = oracle.assemble_matrix(cdn, nd, tol_loc, 3)
    vd = torch.from_numpy(verts).cuda()
    cd = torch.from_numpy(np.ascontiguousarray(cells)).cuda()
    for fmt in (2, 3):
        u = 2.0 ** -24 if fmt == 2 else 2.0 ** -53
        g = (mm + 1) * u / (1 - (mm + 1) * u)
        fused = am.assemble_cells(s, vd, cd, dm, pat, fmt, mp.CoefKind.sincosexp).double().cpu().numpy()
        assert pat.nnz == ref.size
        bad = np.abs(fused - ref) > g * mag * 1.0001 + cell_tol
        assert not bad.any(), (mode, fmt, int(bad.sum()))
