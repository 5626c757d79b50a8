"""Generates tests/golden/reference_golden.npz from the UNMODIFIED reference library
compiled out-of-tree (oracle/_ref/libmpfem_ref.so, built by `make -C oracle ref` from
/root/reference/proj/src). Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

The fixture pins the C restatement in oracle/mpfem_oracle.c (tests/test_oracle_golden.py)
and travels to the GPU box, where /root/reference does not exist.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import (COEF_NODAL, COEF_ONE, MODES, MASS, POISSON, Oracle, Reference,  # noqa: E402
                        box_mesh_cells, ensure_built, nphi)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    ensure_built(ref=True)
    R = Reference()
    # Synthetic tets from the product's config-0 generator definition (restated in the
    # oracle): the reference has no such generator, its inputs are the vertex arrays.
    V, _ = Oracle().gen_tets(0, 1, 16)
    out: dict[str, np.ndarray] = {}
    out["rng_seed1"] = R.rng_draws(1, 64)
    out["rng_seed5489"] = R.rng_draws(5489, 4)
    out["verts"] = V
    for p in range(1, 9):
        pts, w = R.rule(p)
        out[f"rule_pts_p{p}"] = pts
        out[f"rule_w_p{p}"] = w
        out[f"nodes_p{p}"] = R.basis_nodes(p)
    tab_hashes = []
    for p in range(1, 9):
        for ef, sf in [(3, 3), (2, 2), (2, 1), (2, 0), (1, 1)]:
            for g in (0, 1):
                t = R.tabulate(p, ef, sf, g)
                key = f"tab_p{p}_e{ef}_s{sf}_g{g}"
                if p <= 3:
                    out[key] = t
                tab_hashes.append(f"{key}:{sha(t)}")
    out["tab_hashes"] = np.array(tab_hashes)
    for p in (1, 2, 3, 4):
        leb, gleb, gk, gkm = R.basis_conditioning(p)
        out[f"cond_p{p}"] = np.concatenate([[leb], gleb, gkm, gk.ravel()])
    geo = np.zeros((16, 2, 4, 40))
    geo_flags = np.zeros((16, 2, 4), dtype=np.uint32)
    for c in range(16):
        for form in (MASS, POISSON):
            for fmt in range(4):
                g, fl = R.cell_geometry(V[c], form, fmt)
                geo[c, form, fmt] = g
                geo_flags[c, form, fmt] = fl
    out["geometry"] = geo
    out["geometry_flags"] = geo_flags
    rng = np.random.default_rng(20241016)
    for mode, cfg in MODES.items():
        for form in (MASS, POISSON):
            for p in (1, 2, 3, 4):
                for kind in (COEF_ONE, 1, COEF_NODAL):
                    m = 2
                    coef = rng.uniform(0.5, 1.5, size=(m, nphi(p))) if kind == COEF_NODAL else None
                    a, fl = R.bilinear(p, form, cfg, V[:m], kind, coef)
                    key = f"A_{mode}_f{form}_p{p}_k{kind}"
                    out[key] = a
                    out[key + "_flags"] = np.array([fl], dtype=np.uint32)
                    if coef is not None:
                        out[key + "_coef"] = coef
                    cz, _ = R.build_C(p, form, cfg, V[0], kind, None if coef is None else coef[0])
                    out[f"C_{mode}_f{form}_p{p}_k{kind}"] = cz
    for form in (MASS, POISSON):
        for mode, cfg in MODES.items():
            for p in (1, 2, 3):
                for kind in (COEF_ONE, COEF_NODAL):
                    coef = rng.uniform(0.5, 1.5, size=nphi(p)) if kind == COEF_NODAL else None
                    b, a64 = R.bound(p, form, cfg, V[5], kind, coef)
                    key = f"bound_{mode}_f{form}_p{p}_k{kind}"
                    out[key] = b
                    out[key + "_a64"] = a64
                    if coef is not None:
                        out[key + "_coef"] = coef
    verts, cells = R.structured_tet_mesh(3, 2, 2, 1.0, 0.15, 7)
    out["mesh322_verts"] = verts
    out["mesh322_cells"] = cells
    for p in (1, 2, 3):
        cd, nd, mm = R.build_dofmap(p, verts, cells)
        out[f"dofmap322_p{p}"] = cd
        out[f"dofmap322_p{p}_meta"] = np.array([nd, mm], dtype=np.int64)
        loc = rng.uniform(-1, 1, size=(cells.shape[0], nphi(p), nphi(p)))
        out[f"locals322_p{p}"] = loc
        for fmt in (1, 2, 3):
            r, c, v, fl = R.assemble_matrix(cd, nd, loc, fmt)
            out[f"coo322_p{p}_fmt{fmt}"] = np.stack([r.astype(np.float64), c.astype(np.float64), v])
    # reference test fixture (test_mesh.cpp:196-201): tet mesh 2x2x2 seed 7 P1 -> 27 dofs, m_K 24
    v2, c2 = R.structured_tet_mesh(2, 2, 2, 1.0, 0.15, 7)
    cd2, nd2, mm2 = R.build_dofmap(1, v2, c2)
    out["dofmap222_p1_meta"] = np.array([nd2, mm2], dtype=np.int64)
    # Algorithm 2 (action_kernel, kernels.cpp:269-304) and its bound (bounds.cpp:128-279).
    arng = np.random.default_rng(2410)
    for mode, cfg in MODES.items():
        for form in (MASS, POISSON):
            for p in (1, 2, 3, 4):
                for kind in (COEF_ONE, 1, COEF_NODAL):
                    m = 2
                    w = arng.uniform(-1.0, 1.0, size=(m, nphi(p)))
                    coef = arng.uniform(0.5, 1.5, size=(m, nphi(p))) if kind == COEF_NODAL else None
                    v, fl = R.action(p, form, cfg, V[:m], w, kind, coef)
                    key = f"V_{mode}_f{form}_p{p}_k{kind}"
                    out[key] = v
                    out[key + "_w"] = w
                    out[key + "_flags"] = np.array([fl], dtype=np.uint32)
                    if coef is not None:
                        out[key + "_coef"] = coef
            for p in (1, 2, 3):
                for kind in (COEF_ONE, COEF_NODAL):
                    w = arng.uniform(-1.0, 1.0, size=nphi(p))
                    coef = arng.uniform(0.5, 1.5, size=nphi(p)) if kind == COEF_NODAL else None
                    b, v64 = R.action_bound(p, form, cfg, V[7], w, kind, coef)
                    key = f"vbound_{mode}_f{form}_p{p}_k{kind}"
                    out[key] = b
                    out[key + "_v64"] = v64
                    out[key + "_w"] = w
                    if coef is not None:
                        out[key + "_coef"] = coef
    # Hexahedra: jittered 2x2x2 lattice, constant / nodal coefficients.
    brng = np.random.default_rng(8)
    lv, _ = R.structured_tet_mesh(2, 2, 2, 1.0, 0.15, 7)
    hexes = lv[box_mesh_cells(2, 2, 2)]
    out["hex_verts"] = hexes
    for mode, cfg in MODES.items():
        for form in (MASS, POISSON):
            for p in (1, 2, 3):
                n = (p + 1) ** 3
                for kind in (COEF_ONE, COEF_NODAL):
                    coef = brng.uniform(0.5, 1.5, size=(2, n)) if kind == COEF_NODAL else None
                    a, fl = R.bilinear_box(p, form, cfg, hexes[:2], kind, coef)
                    key = f"Ahex_{mode}_f{form}_p{p}_k{kind}"
                    out[key] = a
                    out[key + "_flags"] = np.array([fl], dtype=np.uint32)
                    if coef is not None:
                        out[key + "_coef"] = coef
                    c, _ = R.build_C_box(p, form, cfg, hexes[0], kind, None if coef is None else coef[0])
                    out[f"Chex_{mode}_f{form}_p{p}_k{kind}"] = c
                    wv = brng.uniform(-1.0, 1.0, size=(2, n))
                    v, vfl = R.action_box(p, form, cfg, hexes[4:6], wv, kind, coef)
                    out[f"Vhex_{mode}_f{form}_p{p}_k{kind}"] = v
                    out[f"Vhex_{mode}_f{form}_p{p}_k{kind}_w"] = wv
                    out[f"Vhex_{mode}_f{form}_p{p}_k{kind}_flags"] = np.array([vfl], dtype=np.uint32)
                    if p <= 2:
                        b, a64 = R.bound_box(p, form, cfg, hexes[3], kind, None if coef is None else coef[1])
                        out[f"boundhex_{mode}_f{form}_p{p}_k{kind}"] = b
                        out[f"boundhex_{mode}_f{form}_p{p}_k{kind}_a64"] = a64
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
