"""GPU parity tests of Algorithm 2 (action_kernel, kernels.cpp:269-304), through the C-ABI.

Bars (tolerances written here):
  * constant and nodal coefficients: BITWISE equal to the reference's action_kernel (the
    oracle restatement, itself pinned bitwise to the compiled reference by
    tests/test_oracle_golden.py::test_action_bitwise) in every precision mode, p = 1..8;
  * analytic coefficients (c(x_q) through CUDA's vs glibc's transcendentals): vs the same-mode
    oracle max|v_gpu - v_ref| / max|v| <= 2 S bound_v, and vs the fp64 oracle
    err_rel <= S bound_v per cell (bound_v = kernel_bounds' action bound, bounds.cpp:269-279;
    S = 4 when u_s is coarser than every compute format, test_bounds.cpp:52-77);
  * at BASELINE size (65,536 tets): v = A w against the GPU's own fp64 cell matrices (a
    size-independent identity), batched == per-cell bitwise, mesh-indexed == private vertices.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2410_12614_b200 as mp  # noqa: E402
from oracle_lib import (COEF_EXP10_AFFINE, COEF_NODAL, COEF_ONE, COEF_SINCOSEXP, MASS,  # noqa: E402
                        MODES, POISSON, UNIT_ROUNDOFF, nphi)


def aconfig(mode, form, geometry_fp64=False):
    up, ug, uq, us, eng = MODES[mode]
    if geometry_fp64:
        ug = 3
    return mp.KernelConfig(form=mp.FormKind(form), mode=mp.ModeKind.action, u_p=mp.Fmt(up),
                           u_g=mp.Fmt(ug), u_q=mp.Fmt(uq), u_s=mp.Fmt(us),
                           engine=mp.EngineKind(eng))


def cfg_tuple(c):
    return (int(c.u_p), int(c.u_g), int(c.u_q), int(c.u_s), int(c.engine))


def slack(c) -> float:
    us = UNIT_ROUNDOFF[int(c.u_s)]
    return 4.0 if all(us > UNIT_ROUNDOFF[int(f)] for f in (c.u_p, c.u_g, c.u_q)) else 1.0


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def tets(oracle):
    v, _ = oracle.gen_tets(0, 1, 512)
    return v


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
@pytest.mark.parametrize("gfp64", [False, True])
def test_action_bitwise_vs_reference(oracle, tets, mode, form, gfp64):
    if gfp64 and mode == "fp64":
        pytest.skip("u_g is already fp64")
    rng = np.random.default_rng(11 + form)
    cfg = aconfig(mode, form, gfp64)
    for p in range(1, 9):
        n = 37 if p <= 4 else 9
        s = mp.make_setup(p, cfg)
        w = rng.uniform(-1.0, 1.0, size=(n, nphi(p)))
        for kind in (COEF_ONE, COEF_NODAL):
            z = rng.uniform(0.5, 1.5, size=(n, nphi(p))) if kind == COEF_NODAL else None
            v = mp.action_kernel(s, dev(tets[:n]), dev(w), coef_kind=kind,
                                 coef=None if z is None else dev(z))
            ref, _ = oracle.action(p, form, cfg_tuple(cfg), tets[:n], w, kind, z)
            got = v.double().cpu().numpy()
            assert np.array_equal(bits(got), bits(ref)), (mode, form, p, kind,
                                                          np.max(np.abs(got - ref)))
        assert s.last_launch_count() == 1


def test_action_shared_nodal_z_and_mesh_indexing(oracle):
    """The reference's action_kernel takes one z for the batch (kernels.hpp:90-92): a 1-D
    coefficient is shared; mesh-indexed vertices give the same bits as private copies."""
    verts, cells = oracle.structured_tet_mesh(3, 3, 2, 1.0, 0.15, 5)
    rng = np.random.default_rng(2)
    for mode in ("fp64", "mixed", "fp16"):
        cfg = aconfig(mode, POISSON)
        p = 3
        s = mp.make_setup(p, cfg)
        n = cells.shape[0]
        w = rng.uniform(-1, 1, size=(n, nphi(p)))
        z = rng.uniform(0.5, 1.5, size=nphi(p))
        v_mesh = s.action(dev(verts), dev(w), cells=dev(cells, torch.int32), coef_kind=COEF_NODAL,
                          coef=dev(z)).double().cpu().numpy()
        priv = verts[cells]  # (n, 4, 3)
        v_priv = s.action(dev(priv), dev(w), coef_kind=COEF_NODAL,
                          coef=dev(np.tile(z, (n, 1)))).double().cpu().numpy()
        ref, _ = oracle.action(p, POISSON, cfg_tuple(cfg), priv, w, COEF_NODAL, np.tile(z, (n, 1)))
        assert np.array_equal(bits(v_mesh), bits(v_priv))
        assert np.array_equal(bits(v_mesh), bits(ref))


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_action_analytic_coefficient_within_bound(oracle, tets, mode, form):
    rng = np.random.default_rng(5)
    cfg = aconfig(mode, form, geometry_fp64=(form == POISSON))
    S = slack(cfg)
    aniso_v, aniso_u = oracle.gen_tets(1, 3, 16)
    for p in (1, 2, 4, 6):
        n = 12
        s = mp.make_setup(p, cfg)
        w = rng.uniform(-1.0, 1.0, size=(n, nphi(p)))
        for kind, vv, cf in ((COEF_SINCOSEXP, tets[:n], None), (COEF_EXP10_AFFINE, aniso_v[:n], aniso_u[:n])):
            if kind == COEF_EXP10_AFFINE and mode == "fp16":
                continue  # c up to 1e6 overflows fp16 storage by design (config 3)
            got = s.action(dev(vv), dev(w), coef_kind=kind,
                           coef=None if cf is None else dev(cf)).double().cpu().numpy()
            same, _ = oracle.action(p, form, cfg_tuple(cfg), vv, w, kind, cf)
            for c in range(n):
                b, v64 = oracle.action_bound(p, form, cfg_tuple(cfg), vv[c], w[c], kind,
                                             None if cf is None else cf[c])
                scale = np.max(np.abs(v64))
                fin = np.isfinite(same[c])
                if not fin.all():  # u_s overflow (fp16 storage, config 3): same events as the reference
                    assert np.array_equal(np.isfinite(got[c]), fin), (mode, form, p, c)
                    assert np.array_equal(got[c][~fin], same[c][~fin], equal_nan=True)
                    continue
                err64 = np.max(np.abs(got[c] - v64)) / scale
                errsm = np.max(np.abs(got[c] - same[c])) / scale
                assert errsm <= 2 * S * b[0], (mode, form, p, kind, c, errsm, b[0])
                if kind == COEF_SINCOSEXP:
                    assert err64 <= S * b[0], (mode, form, p, kind, c, err64, b[0])
                # Config-3 cells (10^6 coefficient range, aspect ratios to 10^4): the
                # reference's own same-mode action exceeds bound_v there (r underflows u_s on
                # the tiny cells; the u_s-rounded w is amplified by the ill-conditioned G),
                # which is the paper's robustness finding, so only the same-mode bar applies.


def test_action_known_answer_and_errors():
    # test_kernels.cpp:281-290: reference tet, P1 mass action of w = 1 -> 1/24 each
    ref = np.array([[[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]], dtype=np.float64)
    s = mp.make_setup(1, aconfig("fp64", MASS))
    v = mp.action_kernel(s, dev(ref), dev(np.ones((1, 4)))).cpu().numpy()
    assert np.max(np.abs(v - 1.0 / 24.0)) <= 1e-13
    # zero input gives a bitwise zero result (test_kernels.cpp:300-303)
    v0 = mp.action_kernel(s, dev(ref), dev(np.zeros((1, 4)))).cpu().numpy()
    assert np.all(v0 == 0.0)
    with pytest.raises(mp.ConfigError):
        mp.action_kernel(s, dev(ref), dev(np.ones((1, 3))))
    bil = mp.make_setup(1, mp.reference_config(mp.FormKind.mass))
    with pytest.raises(mp.ConfigError):
        mp.action_kernel(bil, dev(ref), dev(np.ones((1, 4))))
    # singular cell -> CheckError (geometry.cpp:42)
    flat = np.zeros((1, 4, 3))
    with pytest.raises(mp.CheckError):
        s.action(dev(flat), dev(np.ones((1, 4))), want_flags=True)


def test_action_host_api_matches_device(oracle, tets):
    rng = np.random.default_rng(9)
    cfg = aconfig("mixed", POISSON, True)
    s = mp.make_setup(4, cfg)
    n = 300
    w = rng.uniform(-1, 1, size=(n, nphi(4)))
    vd = s.action(dev(tets[:n]), dev(w), coef_kind=COEF_SINCOSEXP).cpu().numpy()
    vh = s.action_host(tets[:n], w, coef_kind=COEF_SINCOSEXP)
    assert np.array_equal(vd.view(np.uint32), vh.view(np.uint32))


@pytest.mark.parametrize("form", [MASS, POISSON])
def test_action_at_baseline_size_equals_cell_matrix_product(oracle, form):
    """65,536 config-0/1 tets, P4: the fp64 action equals A w with A the GPU's fp64 cell
    matrices (reference identity v = A w, test_kernels.cpp:319-365, to 1e-12 relative); batches
    of 1 reproduce the batched result bit for bit (test_kernels.cpp:367-405); the mixed-mode
    action stays within S bound_v of the fp64 oracle on sampled cells."""
    verts, _ = oracle.gen_tets(0, 1, 65536)
    rng = np.random.default_rng(4)
    p = 4
    w = rng.uniform(-1, 1, size=(65536, nphi(p)))
    dv, dw = dev(verts), dev(w)
    s64 = mp.make_setup(p, aconfig("fp64", form))
    v64 = s64.action(dv, dw, coef_kind=COEF_SINCOSEXP)
    b64 = mp.make_setup(p, mp.KernelConfig(form=mp.FormKind(form)))
    a64 = b64.cell_matrices(dv, None, COEF_SINCOSEXP)
    av = torch.einsum("cij,cj->ci", a64, dw)
    rel = (v64 - av).abs().amax(dim=1) / av.abs().amax(dim=1)
    assert float(rel.max()) <= 1e-12
    for c in (0, 777, 65535):
        v1 = s64.action(dv[c:c + 1], dw[c:c + 1], coef_kind=COEF_SINCOSEXP)
        assert torch.equal(v1[0], v64[c])
    cfg = aconfig("mixed", form, geometry_fp64=(form == POISSON))
    sm = mp.make_setup(p, cfg)
    vm = sm.action(dv, dw, coef_kind=COEF_SINCOSEXP).double().cpu().numpy()
    for c in rng.choice(65536, 8, replace=False):
        b, ex = oracle.action_bound(p, form, cfg_tuple(cfg), verts[c], w[c], COEF_SINCOSEXP)
        err = np.max(np.abs(vm[c] - ex)) / np.max(np.abs(ex))
        assert err <= slack(cfg) * b[0], (c, err, b[0])
