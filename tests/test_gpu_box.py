"""Hexahedral (box) cells on the GPU, through the C-ABI.

The geometry is evaluated at every rule point (trilinear map), so K1 writes per-point scaled
weights; K2 (the tcgen05 / SIMT GEMM) is unchanged. Bars (tolerances written here):
  * W (build_C with per-point G): BITWISE the reference's (oracle restatement pinned to the
    compiled reference, tests/test_oracle_golden.py::test_box_cells_bitwise), constant and nodal
    coefficients, every mode, p = 1..4;
  * cell matrices vs the fp64 oracle: err_rel <= S bound_a per cell (kernel_bounds on the box
    cell, S = 4 when u_s is coarser than every compute format), vs same mode <= 2 S bound_a;
  * fp64 mode equals the oracle to rounding (<= 1e-13 relative); mesh-indexed == private.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2410_12614_b200 as mp  # noqa: E402
from oracle_lib import (COEF_NODAL, COEF_ONE, MASS, MODES, POISSON, UNIT_ROUNDOFF,  # noqa: E402
                        box_mesh_cells)

PACK = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]


def kconfig(mode, form):
    up, ug, uq, us, eng = MODES[mode]
    return mp.KernelConfig(form=mp.FormKind(form), u_p=mp.Fmt(up), u_g=mp.Fmt(ug), u_q=mp.Fmt(uq),
                           u_s=mp.Fmt(us), engine=mp.EngineKind(eng))


def cfg_tuple(c):
    return (int(c.u_p), int(c.u_g), int(c.u_q), int(c.u_s), int(c.engine))


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.fixture(scope="module")
def hexes(oracle):
    verts, _ = oracle.structured_tet_mesh(3, 3, 3, 1.0, 0.15, 11)
    cells = box_mesh_cells(3, 3, 3)
    return verts, cells, verts[cells]


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_box_scaled_weights_bitwise(oracle, hexes, mode, form):
    _, _, hx = hexes
    rng = np.random.default_rng(5 + form)
    cfg = kconfig(mode, form)
    nd = 3 if form == POISSON else 1
    blocks = PACK if form == POISSON else [(0, 0)]
    for p in (1, 2, 3, 4):
        s = mp.make_setup(p, cfg, cell_kind=1)
        n, nq = 5, (p + 1) ** 3
        for kind in (COEF_ONE, COEF_NODAL):
            z = rng.uniform(0.5, 1.5, size=(n, s.n_phi)) if kind == COEF_NODAL else None
            w, _ = s.scaled_weights(dev(hx[:n]), None, kind, None if z is None else dev(z))
            nqp = s.k // len(blocks)
            w = w.cpu().numpy().reshape(n, len(blocks), nqp)
            assert np.all(w[:, :, nq:] == 0.0)
            w = np.ascontiguousarray(w[:, :, :nq]).reshape(n, -1)
            for c in range(n):
                ref, _ = oracle.build_C_box(p, form, cfg_tuple(cfg), hx[c], kind, None if z is None else z[c])
                ref = ref.reshape(nd, nd, nq)
                want = np.concatenate([ref[a, b] for a, b in blocks])
                assert np.array_equal(w[c].view(np.uint64), want.view(np.uint64)), (mode, form, p, kind, c)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_box_cell_matrices_within_bound(oracle, hexes, mode, form):
    _, _, hx = hexes
    rng = np.random.default_rng(9)
    cfg = kconfig(mode, form)
    us = UNIT_ROUNDOFF[int(cfg.u_s)]
    S = 4.0 if all(us > UNIT_ROUNDOFF[int(f)] for f in (cfg.u_p, cfg.u_g, cfg.u_q)) else 1.0
    for p in (1, 2, 3):
        s = mp.make_setup(p, cfg, cell_kind=1)
        n = 6
        for kind in (COEF_ONE, COEF_NODAL):
            z = rng.uniform(0.5, 1.5, size=(n, s.n_phi)) if kind == COEF_NODAL else None
            a = s.cell_matrices(dev(hx[:n]), None, kind, None if z is None else dev(z))
            a = a.double().cpu().numpy()
            same, _ = oracle.bilinear_box(p, form, cfg_tuple(cfg), hx[:n], kind, z)
            for c in range(n):
                b, a64 = oracle.bound_box(p, form, cfg_tuple(cfg), hx[c], kind, None if z is None else z[c])
                scale = np.max(np.abs(a64))
                e64 = np.max(np.abs(a[c] - a64)) / scale
                esm = np.max(np.abs(a[c] - same[c])) / scale
                assert e64 <= S * b[0], (mode, form, p, kind, c, e64, b[0])
                assert esm <= 2 * S * b[0], (mode, form, p, kind, c, esm, b[0])
                if mode == "fp64":
                    assert e64 <= 1e-13


def test_box_mesh_indexed_and_host_api(oracle, hexes):
    verts, cells, hx = hexes
    for mode in ("mixed", "fp64"):
        s = mp.make_setup(2, kconfig(mode, POISSON), cell_kind=1)
        a_mesh = s.cell_matrices(dev(verts), dev(cells, torch.int32), COEF_ONE)
        a_priv = s.cell_matrices(dev(hx), None, COEF_ONE)
        assert torch.equal(a_mesh, a_priv)
        a_host = s.cell_matrices_host(hx, None, COEF_ONE)
        assert np.array_equal(a_host, a_priv.cpu().numpy())
    with pytest.raises(mp.ConfigError):  # analytic coefficients are defined for tets only
        s.cell_matrices(dev(hx), None, 1)
    with pytest.raises(mp.ConfigError):
        mp.make_setup(5, kconfig("mixed", MASS), cell_kind=1)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_box_bounds_bitwise(oracle, hexes, mode, form):
    """kernel_bounds on hexahedra (per-point geometry diagnostics) on the GPU: bound_a, the
    kappas and the exact A bitwise the reference's (oracle restatement pinned by
    test_box_cells_bitwise), p = 1..3; then every cell of the mesh against its bound."""
    _, _, hx = hexes
    rng = np.random.default_rng(2 + form)
    cfg = kconfig(mode, form)
    for p in (1, 2, 3):
        s = mp.make_setup(p, cfg, cell_kind=1)
        n = 3
        for kind in (COEF_ONE, COEF_NODAL):
            z = rng.uniform(0.5, 1.5, size=(n, s.n_phi)) if kind == COEF_NODAL else None
            out, a64 = s.cell_bounds(dev(hx[:n]), coef_kind=kind, coef=None if z is None else dev(z),
                                     want_a64=True)
            out, a64 = out.cpu().numpy(), a64.cpu().numpy()
            for c in range(n):
                ref, ra = oracle.bound_box(p, form, cfg_tuple(cfg), hx[c], kind, None if z is None else z[c])
                assert np.array_equal(out[c].view(np.uint64), ref.view(np.uint64)), (mode, form, p, kind, c)
                assert np.array_equal(a64[c].view(np.uint64), ra.view(np.uint64)), (mode, form, p, kind, c)
    us = UNIT_ROUNDOFF[int(cfg.u_s)]
    S = 4.0 if all(us > UNIT_ROUNDOFF[int(f)] for f in (cfg.u_p, cfg.u_g, cfg.u_q)) else 1.0
    s = mp.make_setup(2, cfg, cell_kind=1)
    a = s.cell_matrices(dev(hx), None, COEF_ONE).double()
    b, a64 = s.cell_bounds(dev(hx), want_a64=True)
    err = (a - a64).abs().amax(dim=(1, 2)) / a64.abs().amax(dim=(1, 2))
    assert float((err / (S * b[:, 0])).max()) <= 1.0


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_box_action_bitwise(oracle, hexes, mode, form):
    """Algorithm 2 on hexahedra (geometry at every rule point in the r stage): bitwise the
    reference's action_kernel (oracle restatement pinned to ref_action_box), p = 1..3."""
    verts, cells, hx = hexes
    rng = np.random.default_rng(21 + form)
    up, ug, uq, us, eng = MODES[mode]
    cfg = mp.KernelConfig(form=mp.FormKind(form), mode=mp.ModeKind.action, u_p=mp.Fmt(up),
                          u_g=mp.Fmt(ug), u_q=mp.Fmt(uq), u_s=mp.Fmt(us), engine=mp.EngineKind(eng))
    for p in (1, 2, 3):
        s = mp.make_setup(p, cfg, cell_kind=1)
        n = 9
        w = rng.uniform(-1, 1, size=(n, s.n_phi))
        for kind in (COEF_ONE, COEF_NODAL):
            z = rng.uniform(0.5, 1.5, size=(n, s.n_phi)) if kind == COEF_NODAL else None
            v = mp.action_kernel(s, dev(hx[:n]), dev(w), coef_kind=kind, coef=None if z is None else dev(z))
            ref, _ = oracle.action_box(p, form, cfg_tuple(cfg), hx[:n], w, kind, z)
            got = v.double().cpu().numpy()
            assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (mode, form, p, kind)
    vm = s.action(dev(verts), dev(rng.uniform(-1, 1, size=(cells.shape[0], s.n_phi))),
                  cells=dev(cells, torch.int32))
    assert torch.isfinite(vm).all()


@pytest.mark.parametrize("form", [MASS, POISSON])
def test_box_scaled_weights_rare_inputs_bitwise(oracle, hexes, form):
    """K1-box's fp32-u_g fast paths (per-point inputs for p = 1, warp-shared vertices for
    nq_pad % 32 == 0) screen each vertex and fall back to the flagged emulation for
    fp32-subnormal coordinates and for geometry that overflows fp32: W and the batch's FP flags
    bitwise the reference's."""
    _, _, hx = hexes
    cells = np.array(hx[:6], dtype=np.float64)
    cells[1, 3, 0] = 1e-40          # fp32-subnormal coordinate
    cells[2, 5, 2] = -3e-39         # fp32-subnormal, negative
    cells[3] *= 1e30                # det and G overflow fp32
    cells[4] *= 1e-30               # G underflows fp32
    cfg = kconfig("mixed", form)
    nd = 3 if form == POISSON else 1
    blocks = PACK if form == POISSON else [(0, 0)]
    for p in (1, 2, 3):
        s = mp.make_setup(p, cfg, cell_kind=1)
        n, nq = cells.shape[0], (p + 1) ** 3
        w, fl = s.scaled_weights(dev(cells), None, COEF_ONE, None)
        nqp = s.k // len(blocks)
        w = np.ascontiguousarray(w.cpu().numpy().reshape(n, len(blocks), nqp)[:, :, :nq]).reshape(n, -1)
        want_fl = 0
        for c in range(n):
            ref, f = oracle.build_C_box(p, form, cfg_tuple(cfg), cells[c], COEF_ONE, None)
            want_fl |= f
            ref = ref.reshape(nd, nd, nq)
            want = np.concatenate([ref[a, b] for a, b in blocks])
            assert np.array_equal(w[c].view(np.uint64), want.view(np.uint64)), (form, p, c)
        assert fl == want_fl, (form, p, fl, want_fl)
