"""Pins the C restatement (oracle/mpfem_oracle.c) against fixtures produced by the
compiled, unmodified reference (tests/golden/make_golden.py) and against known answers
from the reference's own test suite. CPU only."""
import hashlib

import numpy as np
import pytest

from oracle_lib import COEF_NODAL, COEF_ONE, MASS, MODES, POISSON, nphi


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_rng_matches_mt19937_64(oracle, golden):
    # std::mt19937_64 default seed 5489: first draw 14514284786278117030 (C++ standard).
    assert int(oracle.rng_draws(5489, 1)[0]) == 14514284786278117030
    assert np.array_equal(oracle.rng_draws(1, 64), golden["rng_seed1"])


@pytest.mark.parametrize("p", range(1, 9))
def test_rule_and_nodes_bitwise(oracle, golden, p):
    pts, w = oracle.rule(p)
    assert np.array_equal(bits(pts), bits(golden[f"rule_pts_p{p}"]))
    assert np.array_equal(bits(w), bits(golden[f"rule_w_p{p}"]))
    assert np.array_equal(oracle.basis_nodes(p), golden[f"nodes_p{p}"])
    # exactness 2p+1 on the unit tet: integral of 1 = 1/6 (quadrature.cpp:171-224)
    assert abs(w.sum() - 1.0 / 6.0) < 1e-15


def test_tabulations_bitwise(oracle, golden):
    for entry in golden["tab_hashes"]:
        key, digest = str(entry).split(":")
        p, e, s, g = (int(x[1:]) for x in key.split("_")[1:])
        t = oracle.tabulate(p, e, s, g)
        assert hashlib.sha256(t.tobytes()).hexdigest() == digest, key
        if p <= 3:
            assert np.array_equal(bits(t), bits(golden[key])), key


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_basis_conditioning(oracle, golden, p):
    leb, gleb, gk, gkm = oracle.basis_conditioning(p)
    assert np.array_equal(np.concatenate([[leb], gleb, gkm, gk.ravel()]), golden[f"cond_p{p}"])


def test_cell_geometry_bitwise(oracle, golden):
    V = golden["verts"]
    for c in range(V.shape[0]):
        for form in (MASS, POISSON):
            for fmt in range(4):
                g, fl = oracle.cell_geometry(V[c], form, fmt)
                assert np.array_equal(bits(g), bits(golden["geometry"][c, form, fmt])), (c, form, fmt)
                assert fl == golden["geometry_flags"][c, form, fmt]


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_bilinear_and_scaled_weights_bitwise(oracle, golden, mode, form):
    V = golden["verts"]
    cfg = MODES[mode]
    for p in (1, 2, 3, 4):
        for kind in (COEF_ONE, 1, COEF_NODAL):
            key = f"A_{mode}_f{form}_p{p}_k{kind}"
            coef = golden[key + "_coef"] if kind == COEF_NODAL else None
            a, fl = oracle.bilinear(p, form, cfg, V[:2], kind, coef)
            assert np.array_equal(bits(a), bits(golden[key])), key
            assert fl == golden[key + "_flags"][0], key
            c, _ = oracle.build_C(p, form, cfg, V[0], kind, None if coef is None else coef[0])
            assert np.array_equal(bits(c), bits(golden[f"C_{mode}_f{form}_p{p}_k{kind}"]))


def test_bounds_bitwise(oracle, golden):
    V = golden["verts"]
    for form in (MASS, POISSON):
        for mode, cfg in MODES.items():
            for p in (1, 2, 3):
                for kind in (COEF_ONE, COEF_NODAL):
                    key = f"bound_{mode}_f{form}_p{p}_k{kind}"
                    coef = golden[key + "_coef"] if kind == COEF_NODAL else None
                    b, a64 = oracle.bound(p, form, cfg, V[5], kind, coef)
                    assert np.array_equal(bits(b), bits(golden[key])), key
                    assert np.array_equal(bits(a64), bits(golden[key + "_a64"])), key


def test_mesh_dofmap_assembly_bitwise(oracle, golden):
    verts, cells = oracle.structured_tet_mesh(3, 2, 2, 1.0, 0.15, 7)
    assert np.array_equal(bits(verts), bits(golden["mesh322_verts"]))
    assert np.array_equal(cells, golden["mesh322_cells"])
    for p in (1, 2, 3):
        cd, nd, mm = oracle.build_dofmap(p, verts, cells)
        assert np.array_equal(cd, golden[f"dofmap322_p{p}"])
        assert [nd, mm] == list(golden[f"dofmap322_p{p}_meta"])
        loc = golden[f"locals322_p{p}"]
        for fmt in (1, 2, 3):
            r, c, v, _ = oracle.assemble_matrix(cd, nd, loc, fmt)
            ref = golden[f"coo322_p{p}_fmt{fmt}"]
            assert np.array_equal(r, ref[0].astype(np.int32))
            assert np.array_equal(c, ref[1].astype(np.int32))
            assert np.array_equal(bits(v), bits(ref[2]))


def test_reference_known_answers(oracle, golden):
    # test_mesh.cpp:194-199: tet mesh 2x2x2 seed 7, P1 -> 27 dofs, max multiplicity 24
    v, c = oracle.structured_tet_mesh(2, 2, 2, 1.0, 0.15, 7)
    _, nd, mm = oracle.build_dofmap(1, v, c)
    assert (nd, mm) == (27, 24) == tuple(golden["dofmap222_p1_meta"])
    # reference tet P1 mass: |K|/20 (1 + delta_ij) with |K| = 1/6
    ref = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    a, _ = oracle.bilinear(1, MASS, MODES["fp64"], ref[None])
    want = (np.ones((4, 4)) + np.eye(4)) / 120.0
    assert np.max(np.abs(a[0] - want)) <= 1e-15
    # Poisson stiffness annihilates constants (test_kernels.cpp:146-166)
    V = golden["verts"]
    for p in (1, 2, 3):
        a, _ = oracle.bilinear(p, POISSON, MODES["fp64"], V[:2])
        assert np.max(np.abs(a.sum(axis=2))) <= 1e-12
    # golden COO text of test_assembly.cpp:173-201 (cells {2,1} and {1,0})
    cd = np.array([[2, 1], [1, 0]], dtype=np.int32)
    loc = np.array([[[4.0, 0.5], [-1.0, 2.0]], [[1.0, 3.0], [0.25, -2.0]]])
    r, cc, vv, _ = oracle.assemble_matrix(cd, 3, loc, 3)
    text = "".join(f"{a} {b} {x:.17g}\n" for a, b, x in zip(r, cc, vv))
    assert text == "0 0 -2\n0 1 0.25\n1 0 3\n1 1 3\n1 2 -1\n2 1 0.5\n2 2 4\n"


def test_config0_generator_properties(oracle):
    v, _ = oracle.gen_tets(0, 1, 2048)
    ref = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    assert np.all(np.abs(v - ref) < 0.15 + 1e-15)
    e = v[:, 1:, :] - v[:, :1, :]
    det = np.linalg.det(np.transpose(e, (0, 2, 1)))
    assert np.all(det >= 1e-3)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("form", [MASS, POISSON])
def test_action_bitwise(oracle, golden, mode, form):
    """Algorithm 2 (action_kernel, kernels.cpp:269-304) restated bit for bit, FP flags too."""
    V = golden["verts"]
    cfg = MODES[mode]
    for p in (1, 2, 3, 4):
        for kind in (COEF_ONE, 1, COEF_NODAL):
            key = f"V_{mode}_f{form}_p{p}_k{kind}"
            coef = golden[key + "_coef"] if kind == COEF_NODAL else None
            v, fl = oracle.action(p, form, cfg, V[:2], golden[key + "_w"], kind, coef)
            assert np.array_equal(bits(v), bits(golden[key])), key
            assert fl == golden[key + "_flags"][0], key


def test_action_bounds_bitwise(oracle, golden):
    """kernel_bounds with w: bound_v and the exact v (bounds.cpp:128-279)."""
    V = golden["verts"]
    for form in (MASS, POISSON):
        for mode, cfg in MODES.items():
            for p in (1, 2, 3):
                for kind in (COEF_ONE, COEF_NODAL):
                    key = f"vbound_{mode}_f{form}_p{p}_k{kind}"
                    coef = golden[key + "_coef"] if kind == COEF_NODAL else None
                    b, v64 = oracle.action_bound(p, form, cfg, V[7], golden[key + "_w"], kind, coef)
                    assert np.array_equal(bits(b), bits(golden[key])), key
                    assert np.array_equal(bits(v64), bits(golden[key + "_v64"])), key


def test_action_known_answers(oracle, golden):
    # test_kernels.cpp:281-290: reference tet, P1 mass action of w = 1 -> 1/24 per function
    ref = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    v, _ = oracle.action(1, MASS, MODES["fp64"], ref[None], np.ones((1, 4)))
    assert np.max(np.abs(v - 1.0 / 24.0)) <= 1e-13
    # the action is the bilinear matrix applied to w (fp64: both are exact to rounding)
    V = golden["verts"]
    rng = np.random.default_rng(3)
    for form in (MASS, POISSON):
        for p in (2, 3):
            w = rng.uniform(-1, 1, size=(2, nphi(p)))
            v, _ = oracle.action(p, form, MODES["fp64"], V[:2], w)
            a, _ = oracle.bilinear(p, form, MODES["fp64"], V[:2])
            av = np.einsum("cij,cj->ci", a, w)
            assert np.max(np.abs(v - av)) <= 1e-13 * np.max(np.abs(av))


@pytest.mark.parametrize("mode", list(MODES))
def test_box_cells_bitwise(oracle, golden, mode):
    """Hexahedra: bilinear_kernel, build_C and kernel_bounds with per-point
    geometry through the trilinear map, bit for bit the reference's (flags too)."""
    hexes = golden["hex_verts"]
    cfg = MODES[mode]
    for form in (MASS, POISSON):
        for p in (1, 2, 3):
            for kind in (COEF_ONE, COEF_NODAL):
                key = f"Ahex_{mode}_f{form}_p{p}_k{kind}"
                coef = golden[key + "_coef"] if kind == COEF_NODAL else None
                a, fl = oracle.bilinear_box(p, form, cfg, hexes[:2], kind, coef)
                assert np.array_equal(bits(a), bits(golden[key])), key
                assert fl == golden[key + "_flags"][0], key
                c, _ = oracle.build_C_box(p, form, cfg, hexes[0], kind, None if coef is None else coef[0])
                assert np.array_equal(bits(c), bits(golden[f"Chex_{mode}_f{form}_p{p}_k{kind}"]))
                vkey = f"Vhex_{mode}_f{form}_p{p}_k{kind}"
                v, vfl = oracle.action_box(p, form, cfg, hexes[4:6], golden[vkey + "_w"], kind, coef)
                assert np.array_equal(bits(v), bits(golden[vkey])), vkey
                assert vfl == golden[vkey + "_flags"][0], vkey
                if p <= 2:
                    b, a64 = oracle.bound_box(p, form, cfg, hexes[3], kind, None if coef is None else coef[1])
                    assert np.array_equal(bits(b), bits(golden[f"boundhex_{mode}_f{form}_p{p}_k{kind}"]))
                    assert np.array_equal(bits(a64), bits(golden[f"boundhex_{mode}_f{form}_p{p}_k{kind}_a64"]))
    # known answer: unit cube Q1 mass in closed form, prod_a (1 + delta_a) / 216 with
    # delta_a = 1 when the two vertices share their axis-a coordinate
    cube = np.array([[(b & 1), (b >> 1) & 1, (b >> 2) & 1] for b in range(8)], dtype=np.float64)
    a, _ = oracle.bilinear_box(1, MASS, MODES["fp64"], cube[None])
    want = np.array([[np.prod([2.0 if ((i >> k) & 1) == ((j >> k) & 1) else 1.0 for k in range(3)]) / 216.0
                      for j in range(8)] for i in range(8)])
    assert np.max(np.abs(a[0] - want)) <= 1e-15
