"""GPU parity tests of the cell-matrix hot path, through the C-ABI.

Bars (tolerances written here):
  * rule / scaled weights W: bitwise equal to the reference build_C (oracle, pinned to the
    compiled reference) for constant and nodal coefficients; analytic coefficients allow a
    last-place difference where CUDA's and glibc's sin/cos/exp/pow differ by an ulp.
  * cell matrices vs the fp64 oracle: err_rel <= S * bound_a per cell, S = 4 when u_s is
    coarser than the compute formats else 1 (test_bounds.cpp:52-77);
  * vs the reference same-mode output: max|A_gpu - A_ref| / max|A| <= 2 S bound_a.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2410_12614_b200 as mp  # noqa: E402
from oracle_lib import (COEF_EXP10_AFFINE, COEF_NODAL, COEF_ONE, COEF_SINCOSEXP, MASS,  # noqa: E402
                        MODES, POISSON, UNIT_ROUNDOFF, nphi, nq, rel_err)

PACK = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]


def kconfig(mode, form, geometry_fp64=False):
    up, ug, uq, us, eng = MODES[mode]
    if geometry_fp64:
        ug = 3
    return mp.KernelConfig(form=mp.FormKind(form), u_p=mp.Fmt(up), u_g=mp.Fmt(ug), u_q=mp.Fmt(uq),
                           u_s=mp.Fmt(us), engine=mp.EngineKind(eng))


def cfg_tuple(c: mp.KernelConfig):
    return (int(c.u_p), int(c.u_g), int(c.u_q), int(c.u_s), int(c.engine))


def slack(c: mp.KernelConfig) -> float:
    us = UNIT_ROUNDOFF[int(c.u_s)]
    coarser = all(us > UNIT_ROUNDOFF[int(f)] for f in (c.u_p, c.u_g, c.u_q))
    return 4.0 if coarser else 1.0


@pytest.fixture(scope="module")
def tets(oracle):
    v, _ = oracle.gen_tets(0, 1, 1024)
    return v


@pytest.fixture(scope="module")
def aniso(oracle):
    return oracle.gen_tets(1, 3, 256)


def coef_for(kind, p, n, rng):
    if kind == COEF_NODAL:
        return rng.uniform(0.5, 1.5, size=(n, nphi(p)))
    return None


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.mark.parametrize("p", range(1, 9))
def test_setup_rule_bitwise(oracle, p):
    s = mp.make_setup(p, kconfig("mixed", POISSON))
    pts, w = s.rule()
    opts, ow = oracle.rule(p)
    assert np.array_equal(pts.view(np.uint64), opts.view(np.uint64))
    assert np.array_equal(w.view(np.uint64), ow.view(np.uint64))
    assert s.n_phi == nphi(p) and s.n_q == nq(p)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
@pytest.mark.parametrize("kind", [COEF_ONE, COEF_NODAL, COEF_SINCOSEXP])
def test_scaled_weights_match_build_C(oracle, tets, mode, form, kind):
    rng = np.random.default_rng(7)
    for p in (1, 2, 4):
        cfg = kconfig(mode, form)
        s = mp.make_setup(p, cfg)
        n = 6
        coef = coef_for(kind, p, n, rng)
        w, _ = s.scaled_weights(dev(tets[:n]), None, kind, None if coef is None else dev(coef))
        nd = 3 if form == POISSON else 1
        blocks = PACK if form == POISSON else [(0, 0)]
        # W layout: blocks of nq_pad = round_up(n_q, 8) entries, zero beyond n_q
        nqp = s.k // len(blocks)
        w = w.cpu().numpy().reshape(n, len(blocks), nqp)
        assert np.all(w[:, :, nq(p):] == 0.0)
        w = np.ascontiguousarray(w[:, :, :nq(p)]).reshape(n, -1)
        us = UNIT_ROUNDOFF[int(cfg.u_s)]
        for c in range(n):
            ref, _ = oracle.build_C(p, form, cfg_tuple(cfg), tets[c], kind,
                                    None if coef is None else coef[c])
            ref = ref.reshape(nd, nd, nq(p))
            want = np.concatenate([ref[s_, t_] for s_, t_ in blocks])
            if kind in (COEF_ONE, COEF_NODAL):
                assert np.array_equal(w[c].view(np.uint64), want.view(np.uint64)), (p, c)
            else:
                # The analytic coefficient is evaluated on the GPU by polynomial kernels at
                # u_g (fp32 for u_g = fp32, fp64 otherwise) within ~2 ulp of the correctly
                # rounded value the oracle uses: W may differ in the last place of u_s.
                diff = np.abs(w[c] - want)
                wide = int(cfg.u_s) >= 2
                tol = 8.0 * us if wide else 2.0 * us
                tol = max(tol, 16 * 2.0**-53)
                min_sub = {0: 2.0**-133, 1: 2.0**-24, 2: 2.0**-149, 3: 2.0**-1074}[int(cfg.u_s)]
                assert np.all(diff <= tol * np.abs(want) + min_sub), (p, c)  # 1 subnormal ulp
                if not wide:  # a ~2-ulp(u_g) coefficient difference rarely survives rounding to u_s
                    assert np.mean(diff > 0) <= 0.02, (p, c)


def run_gpu(setup, verts, kind, coef):
    out = setup.cell_matrices(dev(verts), None, kind, None if coef is None else dev(coef))
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_cell_matrices_within_bound(oracle, tets, mode, form):
    rng = np.random.default_rng(11)
    for p in (1, 2, 3, 4):
        for kind in (COEF_SINCOSEXP, COEF_NODAL, COEF_ONE):
            cfg = kconfig(mode, form)
            s = mp.make_setup(p, cfg)
            n = 4 if p >= 4 else 6
            coef = coef_for(kind, p, n, rng)
            a_gpu = run_gpu(s, tets[:n], kind, coef)
            a_same, _ = oracle.bilinear(p, form, cfg_tuple(cfg), tets[:n], kind, coef)
            S = slack(cfg)
            for c in range(n):
                b, a64 = oracle.bound(p, form, cfg_tuple(cfg), tets[c], kind,
                                      None if coef is None else coef[c])
                err = np.max(np.abs(a_gpu[c] - a64)) / np.max(np.abs(a64))
                assert err <= S * b[0], (p, kind, c, err, b[0])
                d_same = np.max(np.abs(a_gpu[c] - a_same[c])) / np.max(np.abs(a64))
                assert d_same <= 2 * S * b[0], (p, kind, c, d_same, b[0])


@pytest.mark.parametrize("mode", ["fp64", "mixed"])
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_extreme_geometry_fp_events_match_build_C(oracle, tets, mode, form):
    """Cells whose fp64 geometry overflows (1e160 coordinates), underflows |det| to zero
    while inv(J) overflows (1e-160: |det| * inf -> NaN), or carries a NaN vertex: the
    fast binary64 geometry must hand these to the flagged sequence, so W and the FP-event
    flags equal build_C's (kernels.cpp:177-197, geometry.cpp:12-118) bit for bit."""
    cfg = kconfig(mode, form, geometry_fp64=True)
    s = mp.make_setup(2, cfg)
    nan_cell = tets[1].copy()
    nan_cell[2, 1] = np.nan
    cases = [tets[0] * 1e160, tets[2] * 1e-160, nan_cell, tets[3] * 1e150, tets[4]]
    for i, cell in enumerate(cases):
        w, fl = s.scaled_weights(dev(cell[None]), None, COEF_ONE)
        ref, rfl = oracle.build_C(2, form, cfg_tuple(cfg), cell, COEF_ONE)
        nd = 3 if form == POISSON else 1
        blocks = PACK if form == POISSON else [(0, 0)]
        ref = ref.reshape(nd, nd, nq(2))
        want = np.concatenate([ref[a, b] for a, b in blocks])
        got = w.cpu().numpy().reshape(len(blocks), -1)[:, :nq(2)].reshape(-1)
        same = (got.view(np.uint64) == want.view(np.uint64)) | (np.isnan(got) & np.isnan(want))
        assert np.all(same), (i, got[:4], want[:4])
        assert fl == rfl, (i, hex(fl), hex(rfl))


@pytest.mark.parametrize("p", [5, 6, 7, 8])
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_high_degree_all_modes(oracle, tets, p, form):
    """p = 5..8 (56 to 165 dofs, up to 729 rule points) in every mode, 8 cells each: every
    cell within S * bound_a of the fp64 oracle; BASELINE's "mixed" (fp16 storage, fp32
    accumulation, the scalar-engine config of test_bounds.cpp:75-76) and fp16 also within
    2 S bound_a of the reference's same-mode output (kernels.cpp:242-267). Where the
    reference itself fails -- fp16 evaluation of the p >= 7 basis raises invalid and its
    matrices are NaN -- the GPU must fail the same way (NaN matrices, invalid flag)."""
    n = 8
    for mode in ("mixed", "fp16", "mixed_bf16", "fp64"):
        cfg = kconfig(mode, form)
        s = mp.make_setup(p, cfg)
        a_t, fl = s.cell_matrices(dev(tets[:n]), None, COEF_SINCOSEXP, want_flags=True)
        a_gpu = a_t.double().cpu().numpy()
        same = mode in ("mixed", "fp16")
        if same:
            a_same, rfl = oracle.bilinear(p, form, cfg_tuple(cfg), tets[:n], COEF_SINCOSEXP, None)
            if not np.all(np.isfinite(a_same)):
                assert mode == "fp16" and p >= 7, (mode, p)
                assert rfl & 4 and fl & 4, (hex(rfl), hex(fl))
                assert np.array_equal(np.isfinite(a_gpu), np.isfinite(a_same))
                continue
        S = slack(cfg)
        for c in range(n):
            b, a64 = oracle.bound(p, form, cfg_tuple(cfg), tets[c], COEF_SINCOSEXP, None)
            scale = np.max(np.abs(a64))
            err = np.max(np.abs(a_gpu[c] - a64)) / scale
            assert err <= S * b[0], (mode, c, err, b[0])
            if same:
                d_same = np.max(np.abs(a_gpu[c] - a_same[c])) / scale
                assert d_same <= 2 * S * b[0], (mode, c, d_same, b[0])


def test_fp16_storage_high_degree_reports_underflow(oracle, tets):
    # Collapsed Gauss-Jacobi weights fall below fp16's normal range from p = 3;
    # the reference raises underflow there, and so must the GPU path.
    s = mp.make_setup(4, kconfig("mixed", MASS))
    _, fl = s.cell_matrices(dev(tets[:8]), None, COEF_SINCOSEXP, want_flags=True)
    assert fl & 2


def test_config3_anisotropic(oracle, aniso):
    verts, u4 = aniso
    rng = np.random.default_rng(3)
    idx = rng.choice(verts.shape[0], 6, replace=False)
    for p in (1, 2, 3):
        for form in (MASS, POISSON):
            for mode in ("mixed_bf16", "fp32", "fp64"):
                cfg = kconfig(mode, form)
                s = mp.make_setup(p, cfg)
                a_gpu = run_gpu(s, verts[idx], COEF_EXP10_AFFINE, u4[idx])
                for j, c in enumerate(idx):
                    b, a64 = oracle.bound(p, form, cfg_tuple(cfg), verts[c], COEF_EXP10_AFFINE, u4[c])
                    err = np.max(np.abs(a_gpu[j] - a64)) / np.max(np.abs(a64))
                    assert err <= slack(cfg) * b[0], (p, form, mode, err, b[0])


@pytest.mark.parametrize("mode", ["mixed", "fp32", "fp64"])
def test_batch_neutrality_bitwise(tets, mode):
    # A cell's matrix does not depend on its batch or its position in a tile
    # (test_kernels.cpp:367-404 analogue).
    for form in (MASS, POISSON):
        s = mp.make_setup(3, kconfig(mode, form))
        full = run_gpu(s, tets[:600], COEF_SINCOSEXP, None)
        part = run_gpu(s, tets[300:301], COEF_SINCOSEXP, None)
        part2 = run_gpu(s, tets[255:520], COEF_SINCOSEXP, None)
        assert np.array_equal(full[300], part[0])
        assert np.array_equal(full[255:520], part2)


def test_mesh_indexed_equals_private_vertices(oracle):
    verts, cells = oracle.structured_tet_mesh(4, 3, 2, 1.0, 0.15, 5)
    priv = verts[cells]  # (n, 4, 3)
    for mode in ("mixed", "fp64"):
        s = mp.make_setup(2, kconfig(mode, POISSON))
        a = s.cell_matrices(dev(verts), torch.from_numpy(cells).cuda(), COEF_SINCOSEXP)
        b = s.cell_matrices(dev(priv), None, COEF_SINCOSEXP)
        torch.cuda.synchronize()
        assert torch.equal(a, b)


def test_host_api_matches_device(tets):
    s = mp.make_setup(4, kconfig("mixed_bf16", POISSON))
    d = run_gpu(s, tets[:300], COEF_SINCOSEXP, None)
    h = s.cell_matrices_host(tets[:300], None, COEF_SINCOSEXP)
    assert np.array_equal(d, h.astype(np.float64))


def test_edge_cases(oracle, tets):
    s = mp.make_setup(2, kconfig("mixed", POISSON))
    # empty batch
    out = s.cell_matrices(dev(tets[:0]), None, COEF_ONE)
    assert out.shape == (0, 10, 10)
    # ragged sizes around the 256-cell tile and a padded output pitch
    for n in (1, 255, 257):
        a = run_gpu(s, tets[:n], COEF_ONE, None)
        b = run_gpu(s, tets[:1], COEF_ONE, None)
        assert np.array_equal(a[0], b[0]) and a.shape[0] == n
    pitch = 128
    o = torch.full((5, pitch), -7.0, device="cuda")
    s.cell_matrices(dev(tets[:5]), None, COEF_ONE, out=o, out_pitch=pitch)
    torch.cuda.synchronize()
    ref = run_gpu(s, tets[:5], COEF_ONE, None).reshape(5, 100)
    assert np.array_equal(o[:, :100].double().cpu().numpy(), ref)
    assert torch.all(o[:, 100:] == -7.0)
    # singular cell -> CheckError (geometry.cpp:42)
    bad = tets[:3].copy()
    bad[1, 3] = bad[1, 0]
    with pytest.raises(mp.CheckError):
        s.cell_matrices(dev(bad), None, COEF_ONE, want_flags=True)
    # config errors (kernels.cpp:29-40, 120-122)
    with pytest.raises(mp.ConfigError):
        mp.make_setup(2, mp.KernelConfig(u_s=mp.Fmt.fp16, u_q=mp.Fmt.fp32, engine=mp.EngineKind.matrix))
    with pytest.raises(mp.ConfigError):
        mp.make_setup(9, kconfig("mixed", MASS))
    with pytest.raises(mp.ConfigError):
        s.cell_matrices(dev(tets[:2]), None, COEF_NODAL, dev(np.ones((2, 3))))


def test_full_config_sizes_properties(oracle):
    """BASELINE configs 0/1 at full size (65,536 tets, P4): size-independent properties
    plus sampled cells against the oracle bound."""
    v, _ = oracle.gen_tets(0, 1, 65536)
    vd = dev(v)
    rng = np.random.default_rng(5)
    sample = rng.choice(65536, 3, replace=False)
    for form, mode in ((MASS, "mixed"), (POISSON, "mixed_bf16"), (POISSON, "mixed")):
        cfg = kconfig(mode, form, geometry_fp64=(form == POISSON))
        s = mp.make_setup(4, cfg)
        a = s.cell_matrices(vd, None, COEF_SINCOSEXP)
        w, _ = s.scaled_weights(vd, None, COEF_SINCOSEXP)
        torch.cuda.synchronize()
        a64 = a.double()
        scale = a64.abs().amax(dim=(1, 2))
        # symmetry of every cell matrix
        skew = (a64 - a64.transpose(1, 2)).abs().amax(dim=(1, 2)) / scale
        assert float(skew.max()) <= 8 * UNIT_ROUNDOFF[int(cfg.u_s)]
        if form == MASS:
            # partition of unity: sum_ij A_ij = sum_q W_q (exact products, fp32 sums)
            tot = a64.sum(dim=(1, 2))
            want = w.sum(dim=1)
            assert float(((tot - want).abs() / want.abs()).max()) <= 1e-4
        else:
            # stiffness annihilates constants (test_kernels.cpp:146-166)
            rows = a64.sum(dim=2).abs().amax(dim=1) / scale
            assert float(rows.max()) <= 64 * UNIT_ROUNDOFF[int(cfg.u_s)]
        an = a64.cpu().numpy()
        for c in sample:
            b, ref = oracle.bound(4, form, cfg_tuple(cfg), v[c], COEF_SINCOSEXP)
            err = np.max(np.abs(an[c] - ref)) / np.max(np.abs(ref))
            assert err <= slack(cfg) * b[0]
        assert np.all(np.isfinite(an))


def test_singular_cell_check_error_without_flags(tets):
    """geometry.cpp:42 throws CheckError on a singular pivot. The asynchronous call without
    flags cannot throw in place: the singular cell's row is NaN and the CheckError is raised
    by synchronize() (or by the next call on the setup), after which the setup is usable."""
    s = mp.make_setup(2, kconfig("mixed", POISSON))
    bad = tets[:3].copy()
    bad[1, 3] = bad[1, 0]
    out = s.cell_matrices(dev(bad), None, COEF_ONE)
    with pytest.raises(mp.CheckError):
        s.synchronize()
    a = out.double().cpu().numpy()
    assert np.all(np.isnan(a[1])) and np.all(np.isfinite(a[[0, 2]]))
    s.synchronize()  # reported once
    s.cell_matrices(dev(bad), None, COEF_ONE)
    torch.cuda.synchronize()
    with pytest.raises(mp.CheckError):  # the next call reports it
        s.cell_matrices(dev(tets[:2]), None, COEF_ONE)
    ok = run_gpu(s, tets[:2], COEF_ONE, None)
    assert np.all(np.isfinite(ok))
    # host-buffer call synchronizes: raises in place
    with pytest.raises(mp.CheckError):
        s.cell_matrices_host(bad, None, COEF_ONE)


def test_two_streams_share_one_setup(tets):
    """One setup used concurrently from two streams (per-stream workspaces: W scratch, K1
    tile counter, flags): every result equals the single-stream result bit for bit."""
    s = mp.make_setup(4, kconfig("mixed", POISSON, geometry_fp64=True))
    va, vb = dev(tets[:700]), dev(tets[300:1000])
    ref_a = s.cell_matrices(va, None, COEF_SINCOSEXP).clone()
    ref_b = s.cell_matrices(vb, None, COEF_SINCOSEXP).clone()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for _ in range(8):
        with torch.cuda.stream(sa):
            oa = s.cell_matrices(va, None, COEF_SINCOSEXP, stream=sa)
        with torch.cuda.stream(sb):
            ob = s.cell_matrices(vb, None, COEF_SINCOSEXP, stream=sb)
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        assert torch.equal(oa, ref_a) and torch.equal(ob, ref_b)


@pytest.mark.parametrize("form", [MASS, POISSON])
def test_cuda_graph_replay_bitwise(tets, form):
    """K1 -> K2 captured in a CUDA graph after reserve() (mpfem_b200_reserve: no allocation in
    later calls) and replayed: the programmatic dependent launch edge between the two kernels
    (K2's griddepcontrol.wait) must survive capture; every replay equals the eager result bit
    for bit. Mass takes the staged K2-s kernel, Poisson the CTA-pair kernel."""
    s = mp.make_setup(4, kconfig("mixed", form, geometry_fp64=(form == POISSON)))
    v = dev(tets[:900])
    ref = s.cell_matrices(v, None, COEF_SINCOSEXP).clone()
    st = torch.cuda.Stream()
    out = torch.empty_like(ref)
    with torch.cuda.stream(st):
        s.reserve(v.shape[0], stream=st)
        s.cell_matrices(v, None, COEF_SINCOSEXP, out=out, stream=st)  # warm: attributes, modules
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        s.cell_matrices(v, None, COEF_SINCOSEXP, out=out, stream=st)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
