"""GPU bound evaluation: kernel_bounds (bounds.cpp:29-281, bilinear part) per cell
on the device, through the C-ABI.

Bars (tolerances written here):
  * constant and nodal coefficients: bound_a, kappa_q/p/g and the exact binary64 A are BITWISE
    the oracle's kernel_bounds restatement (itself pinned bitwise to the compiled reference by
    tests/test_oracle_golden.py::test_bounds_bitwise), modes x forms x p = 1..5;
  * analytic coefficients (c(x_q) through CUDA's vs glibc's transcendentals): <= 1e-12 relative;
  * SPEC acceptance #6 at BASELINE scale: on all 65,536 config-0/1 cells, the mixed-precision
    cell matrices stay within S * bound_a of the exact A (S = 4 when u_s is coarser than every
    compute format, test_bounds.cpp:52-77) -- every cell, not a host-side sample.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2410_12614_b200 as mp  # noqa: E402
from oracle_lib import (COEF_EXP10_AFFINE, COEF_NODAL, COEF_ONE, COEF_SINCOSEXP, MASS,  # noqa: E402
                        MODES, POISSON, UNIT_ROUNDOFF, nphi)


def kconfig(mode, form, geometry_fp64=False):
    up, ug, uq, us, eng = MODES[mode]
    if geometry_fp64:
        ug = 3
    return mp.KernelConfig(form=mp.FormKind(form), u_p=mp.Fmt(up), u_g=mp.Fmt(ug), u_q=mp.Fmt(uq),
                           u_s=mp.Fmt(us), engine=mp.EngineKind(eng))


def cfg_tuple(c):
    return (int(c.u_p), int(c.u_g), int(c.u_q), int(c.u_s), int(c.engine))


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_bounds_bitwise_vs_kernel_bounds(oracle, mode, form):
    verts, _ = oracle.gen_tets(0, 1, 8)
    rng = np.random.default_rng(3 + form)
    cfg = kconfig(mode, form)
    for p in range(1, 6):
        s = mp.make_setup(p, cfg)
        n = 3
        for kind in (COEF_ONE, COEF_NODAL):
            z = rng.uniform(0.5, 1.5, size=(n, nphi(p))) if kind == COEF_NODAL else None
            out, a64 = s.cell_bounds(dev(verts[:n]), coef_kind=kind, coef=None if z is None else dev(z),
                                     want_a64=True)
            out, a64 = out.cpu().numpy(), a64.cpu().numpy()
            for c in range(n):
                ref, ra = oracle.bound(p, form, cfg_tuple(cfg), verts[c], kind, None if z is None else z[c])
                assert np.array_equal(bits(out[c]), bits(ref)), (mode, form, p, kind, c, out[c], ref)
                assert np.array_equal(bits(a64[c]), bits(ra)), (mode, form, p, kind, c)


def test_bounds_analytic_coefficients(oracle):
    verts, _ = oracle.gen_tets(0, 1, 6)
    av, au = oracle.gen_tets(1, 3, 6)
    for form in (MASS, POISSON):
        cfg = kconfig("mixed", form, geometry_fp64=(form == POISSON))
        for p in (2, 4):
            s = mp.make_setup(p, cfg)
            for kind, vv, cf in ((COEF_SINCOSEXP, verts, None), (COEF_EXP10_AFFINE, av, au)):
                out = s.cell_bounds(dev(vv), coef_kind=kind, coef=None if cf is None else dev(cf)).cpu().numpy()
                for c in range(vv.shape[0]):
                    ref, _ = oracle.bound(p, form, cfg_tuple(cfg), vv[c], kind, None if cf is None else cf[c])
                    assert np.allclose(out[c], ref, rtol=1e-12, atol=0), (form, p, kind, c, out[c], ref)


def test_bounds_singular_cell_is_check_error():
    s = mp.make_setup(2, kconfig("mixed", POISSON))
    with pytest.raises(mp.CheckError):
        s.cell_bounds(dev(np.zeros((1, 4, 3))))


@pytest.mark.parametrize("form", [MASS, POISSON])
@pytest.mark.parametrize("mode", ["mixed", "mixed_bf16", "fp16"])
def test_bound_dominance_every_cell_at_baseline_size(oracle, form, mode):
    """SPEC #6 at config scale: every one of the 65,536 config-0/1 cells (P4, c(x) at the
    quadrature points) satisfies err_rel(A_gpu) <= S bound_a against the exact binary64 A of
    kernel_bounds (report.a), both computed on the GPU."""
    verts, _ = oracle.gen_tets(0, 1, 65536)
    dv = dev(verts)
    cfg = kconfig(mode, form, geometry_fp64=(form == POISSON))
    us = UNIT_ROUNDOFF[int(cfg.u_s)]
    S = 4.0 if all(us > UNIT_ROUNDOFF[int(f)] for f in (cfg.u_p, cfg.u_g, cfg.u_q)) else 1.0
    s = mp.make_setup(4, cfg)
    a = s.cell_matrices(dv, None, COEF_SINCOSEXP).double()
    b, a64 = s.cell_bounds(dv, coef_kind=COEF_SINCOSEXP, want_a64=True)
    err = (a - a64).abs().amax(dim=(1, 2)) / a64.abs().amax(dim=(1, 2))
    ratio = (err / (S * b[:, 0])).cpu().numpy()
    assert np.isfinite(ratio).all()
    assert ratio.max() <= 1.0, (mode, form, float(ratio.max()), int(ratio.argmax()))
    # sampled cross-check of the device bounds against the host restatement
    for c in (0, 4097, 65535):
        ref, _ = oracle.bound(4, form, cfg_tuple(cfg), verts[c], COEF_SINCOSEXP)
        assert np.allclose(b[c].cpu().numpy(), ref, rtol=1e-12)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_action_bounds_bitwise(oracle, mode, form):
    """bound_v and the exact v (bounds.cpp:128-279 action part) bitwise the restatement's
    (pinned to ref_action_bound, tests/test_oracle_golden.py::test_action_bounds_bitwise)."""
    verts, _ = oracle.gen_tets(0, 1, 8)
    rng = np.random.default_rng(8 + form)
    cfg = kconfig(mode, form)
    for p in range(1, 6):
        s = mp.make_setup(p, cfg)
        n = 3
        w = rng.uniform(-1, 1, size=(n, nphi(p)))
        for kind in (COEF_ONE, COEF_NODAL):
            z = rng.uniform(0.5, 1.5, size=(n, nphi(p))) if kind == COEF_NODAL else None
            out, v64 = s.action_bounds(dev(verts[:n]), dev(w), coef_kind=kind,
                                       coef=None if z is None else dev(z), want_v64=True)
            out, v64 = out.cpu().numpy(), v64.cpu().numpy()
            for c in range(n):
                ref, rv = oracle.action_bound(p, form, cfg_tuple(cfg), verts[c], w[c], kind,
                                              None if z is None else z[c])
                assert np.array_equal(bits(out[c]), bits(ref)), (mode, form, p, kind, c, out[c], ref)
                assert np.array_equal(bits(v64[c]), bits(rv)), (mode, form, p, kind, c)


@pytest.mark.parametrize("form", [MASS, POISSON])
def test_action_bound_dominance_every_cell(oracle, form):
    """Algorithm 2 at config scale: every one of the 65,536 config-0/1 cells satisfies
    err_rel(v_gpu) <= S bound_v against the exact v of kernel_bounds, both on the GPU."""
    verts, _ = oracle.gen_tets(0, 1, 65536)
    dv = dev(verts)
    w = dev(np.random.default_rng(12).uniform(-1, 1, size=(65536, nphi(4))))
    for mode in ("mixed", "mixed_bf16"):
        up, ug, uq, us, eng = MODES[mode]
        cfg = mp.KernelConfig(form=mp.FormKind(form), mode=mp.ModeKind.action, u_p=mp.Fmt(up),
                              u_g=mp.Fmt(3 if form == POISSON else ug), u_q=mp.Fmt(uq),
                              u_s=mp.Fmt(us), engine=mp.EngineKind(eng))
        s = mp.make_setup(4, cfg)
        v = mp.action_kernel(s, dv, w, coef_kind=COEF_SINCOSEXP).double()
        b, v64 = s.action_bounds(dv, w, coef_kind=COEF_SINCOSEXP, want_v64=True)
        err = (v - v64).abs().amax(dim=1) / v64.abs().amax(dim=1)
        ratio = (err / (4.0 * b[:, 0])).cpu().numpy()
        assert np.isfinite(ratio).all() and ratio.max() <= 1.0, (mode, form, float(ratio.max()))
