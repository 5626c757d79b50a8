"""ctypes bindings to the parity checker (oracle/liboracle.so) and, where it was built,
the compiled reference (oracle/_ref/libmpfem_ref.so).

Test infrastructure only: the product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libmpfem_ref.so")

BF16, FP16, FP32, FP64 = 0, 1, 2, 3
MASS, POISSON = 0, 1
COEF_ONE, COEF_SINCOSEXP, COEF_EXP10_AFFINE, COEF_NODAL = 0, 1, 2, 3
UNIT_ROUNDOFF = {BF16: 2.0**-8, FP16: 2.0**-11, FP32: 2.0**-24, FP64: 2.0**-53}

# Precision modes of BASELINE.json -> (u_p, u_g, u_q, u_s, engine); SURVEY 8.0.
MODES = {
    "fp64": (FP64, FP64, FP64, FP64, 0),
    "fp32": (FP32, FP32, FP32, FP32, 0),
    "fp16": (FP16, FP32, FP16, FP16, 0),
    "mixed": (FP32, FP32, FP32, FP16, 0),
    "mixed_bf16": (FP32, FP32, FP32, BF16, 2),
}

_d = C.POINTER(C.c_double)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)
_u32 = C.POINTER(C.c_uint32)
_u64 = C.POINTER(C.c_uint64)
_int = C.POINTER(C.c_int)


def nphi(p: int) -> int:
    return (p + 1) * (p + 2) * (p + 3) // 6


def nq(p: int) -> int:
    return (p + 1) ** 3


def _ptr(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def ensure_built(ref: bool = False) -> None:
    target = "ref" if ref else "all"
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, target], check=True)


class _Lib:
    prefix = ""

    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self._sig("round", C.c_double, [C.c_double, C.c_int, C.c_int, _u32])
        self._sig("rng_draws", None, [C.c_uint64, C.c_int, _u64])
        self._sig("rule_simplex3", C.c_int, [C.c_int, _d, _d])
        self._sig("tabulate", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _d] +
                  ([_u32] if prefix == "orc_" else []))
        self._sig("basis_nodes", C.c_int, [C.c_int, _d])
        self._sig("basis_conditioning", C.c_int, [C.c_int, _d, _d, _d, _d])
        self._sig("cell_geometry", C.c_int, [_d, C.c_int, C.c_int, _d, _u32])
        self._sig("build_C", C.c_int, [C.c_int, C.c_int, _int, _d, C.c_int, _d, _d, _u32])
        self._sig("bilinear", C.c_int, [C.c_int, C.c_int, _int, C.c_int64, _d, C.c_int, _d,
                                         C.c_int, _d, _u32])
        self._sig("bound", C.c_int, [C.c_int, C.c_int, _int, _d, C.c_int, _d, _d, _d])
        self._sig("bilinear_box", C.c_int, [C.c_int, C.c_int, _int, C.c_int64, _d, C.c_int, _d,
                                            C.c_int, _d, _u32])
        self._sig("build_C_box", C.c_int, [C.c_int, C.c_int, _int, _d, C.c_int, _d, _d, _u32])
        self._sig("action_box", C.c_int, [C.c_int, C.c_int, _int, C.c_int64, _d, C.c_int, _d,
                                          C.c_int, _d, C.c_int, _d, _u32])
        self._sig("bound_box", C.c_int, [C.c_int, C.c_int, _int, _d, C.c_int, _d, _d, _d])
        self._sig("action", C.c_int, [C.c_int, C.c_int, _int, C.c_int64, _d, C.c_int, _d,
                                      C.c_int, _d, C.c_int, _d, _u32])
        self._sig("action_bound", C.c_int, [C.c_int, C.c_int, _int, _d, C.c_int, _d, _d, _d,
                                            _d])
        self._sig("structured_tet_mesh", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double,
                                                   C.c_double, C.c_uint64, _d, _i32])
        self._sig("build_dofmap", C.c_int, [C.c_int, C.c_int64, _d, C.c_int64, _i32, _i32,
                                            _i32, _i32])
        self._sig("assemble_matrix", C.c_int, [C.c_int64, C.c_int, _i32, C.c_int32, _d,
                                               C.c_int, _i64, _i32, _i32, _d, _u32])
        self._sig("last_error", C.c_char_p, [])

    def _sig(self, name, res, args):
        f = getattr(self.lib, self.prefix + name)
        f.restype = res
        f.argtypes = args
        setattr(self, "_" + name, f)

    def _check(self, st):
        if st != 0:
            raise RuntimeError(f"status {st}: {self._last_error().decode()}")

    # -- API
    def round(self, x: float, fmt: int, ftz: int = 0):
        fl = C.c_uint32(0)
        v = self._round(x, fmt, ftz, C.byref(fl))
        return v, fl.value

    def rng_draws(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint64)
        self._rng_draws(seed, n, _ptr(out, _u64))
        return out

    def rule(self, p: int):
        pts = np.zeros((nq(p), 3))
        w = np.zeros(nq(p))
        self._check(self._rule_simplex3(p, _ptr(pts, _d), _ptr(w, _d)))
        return pts, w

    def tabulate(self, p, ef, sf, grads):
        nd = 3 if grads else 1
        out = np.zeros((nd, nphi(p), nq(p)))
        args = [p, ef, sf, int(grads), _ptr(out, _d)]
        if self.prefix == "orc_":
            args.append(None)
        self._check(self._tabulate(*args))
        return out

    def basis_nodes(self, p):
        out = np.zeros((nphi(p), 3))
        self._check(self._basis_nodes(p, _ptr(out, _d)))
        return out

    def basis_conditioning(self, p):
        leb = np.zeros(1)
        gleb = np.zeros(3)
        gk = np.zeros((nphi(p), 3))
        gkm = np.zeros(3)
        self._check(self._basis_conditioning(p, _ptr(leb, _d), _ptr(gleb, _d), _ptr(gk, _d),
                                             _ptr(gkm, _d)))
        return leb[0], gleb, gk, gkm

    def cell_geometry(self, verts, form, fmt):
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(12)
        out = np.zeros(40)
        fl = C.c_uint32(0)
        self._check(self._cell_geometry(_ptr(v, _d), form, fmt, _ptr(out, _d), C.byref(fl)))
        return out, fl.value

    def build_C(self, p, form, cfg, verts, kind=COEF_ONE, coef=None):
        nd = 3 if form == POISSON else 1
        out = np.zeros(nd * nd * nq(p))
        c = (C.c_int * 5)(*cfg)
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(12)
        cf = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
        fl = C.c_uint32(0)
        self._check(self._build_C(p, form, c, _ptr(v, _d), kind, _ptr(cf, _d), _ptr(out, _d),
                                  C.byref(fl)))
        return out, fl.value

    def bilinear(self, p, form, cfg, verts, kind=COEF_ONE, coef=None):
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 12)
        m = v.shape[0]
        n = nphi(p)
        out = np.zeros((m, n, n))
        c = (C.c_int * 5)(*cfg)
        cf = None
        stride = 0
        if coef is not None:
            cf = np.ascontiguousarray(coef, dtype=np.float64).reshape(m, -1)
            stride = cf.shape[1]
        fl = C.c_uint32(0)
        self._check(self._bilinear(p, form, c, m, _ptr(v, _d), kind, _ptr(cf, _d), stride,
                                   _ptr(out, _d), C.byref(fl)))
        return out, fl.value

    def bound(self, p, form, cfg, verts, kind=COEF_ONE, coef=None):
        out = np.zeros(4)
        a64 = np.zeros((nphi(p), nphi(p)))
        c = (C.c_int * 5)(*cfg)
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(12)
        cf = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
        self._check(self._bound(p, form, c, _ptr(v, _d), kind, _ptr(cf, _d), _ptr(out, _d),
                                _ptr(a64, _d)))
        return out, a64

    def bilinear_box(self, p, form, cfg, verts, kind=COEF_ONE, coef=None):
        """bilinear_kernel on hexahedra (verts (m, 8, 3)): A (m, (p+1)^3, (p+1)^3), flags."""
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 24)
        m, n = v.shape[0], (p + 1) ** 3
        out = np.zeros((m, n, n))
        c = (C.c_int * 5)(*cfg)
        cf, stride = None, 0
        if coef is not None:
            cf = np.ascontiguousarray(coef, dtype=np.float64).reshape(m, -1)
            stride = cf.shape[1]
        fl = C.c_uint32(0)
        self._check(self._bilinear_box(p, form, c, m, _ptr(v, _d), kind, _ptr(cf, _d), stride,
                                       _ptr(out, _d), C.byref(fl)))
        return out, fl.value

    def build_C_box(self, p, form, cfg, verts, kind=COEF_ONE, coef=None):
        nd = 3 if form == POISSON else 1
        out = np.zeros(nd * nd * (p + 1) ** 3)
        c = (C.c_int * 5)(*cfg)
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(24)
        cf = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
        fl = C.c_uint32(0)
        self._check(self._build_C_box(p, form, c, _ptr(v, _d), kind, _ptr(cf, _d), _ptr(out, _d),
                                      C.byref(fl)))
        return out, fl.value

    def action_box(self, p, form, cfg, verts, w, kind=COEF_ONE, coef=None):
        """action_kernel on hexahedra: v (m, (p+1)^3), flags."""
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 24)
        m = v.shape[0]
        wv = np.ascontiguousarray(w, dtype=np.float64).reshape(m, -1)
        out = np.zeros((m, (p + 1) ** 3))
        c = (C.c_int * 5)(*cfg)
        cf, stride = None, 0
        if coef is not None:
            cf = np.ascontiguousarray(coef, dtype=np.float64).reshape(m, -1)
            stride = cf.shape[1]
        fl = C.c_uint32(0)
        self._check(self._action_box(p, form, c, m, _ptr(v, _d), kind, _ptr(cf, _d), stride,
                                     _ptr(wv, _d), wv.shape[1], _ptr(out, _d), C.byref(fl)))
        return out, fl.value

    def bound_box(self, p, form, cfg, verts, kind=COEF_ONE, coef=None):
        n = (p + 1) ** 3
        out = np.zeros(4)
        a64 = np.zeros((n, n))
        c = (C.c_int * 5)(*cfg)
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(24)
        cf = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
        self._check(self._bound_box(p, form, c, _ptr(v, _d), kind, _ptr(cf, _d), _ptr(out, _d),
                                    _ptr(a64, _d)))
        return out, a64

    def action(self, p, form, cfg, verts, w, kind=COEF_ONE, coef=None):
        """action_kernel (kernels.cpp:269-304): v (m, n_phi) and the FP flag mask."""
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 12)
        m = v.shape[0]
        wv = np.ascontiguousarray(w, dtype=np.float64).reshape(m, -1)
        out = np.zeros((m, nphi(p)))
        c = (C.c_int * 5)(*cfg)
        cf = None
        stride = 0
        if coef is not None:
            cf = np.ascontiguousarray(coef, dtype=np.float64).reshape(m, -1)
            stride = cf.shape[1]
        fl = C.c_uint32(0)
        self._check(self._action(p, form, c, m, _ptr(v, _d), kind, _ptr(cf, _d), stride,
                                 _ptr(wv, _d), wv.shape[1], _ptr(out, _d), C.byref(fl)))
        return out, fl.value

    def action_bound(self, p, form, cfg, verts, w, kind=COEF_ONE, coef=None):
        """kernel_bounds action part: ({bound_v, kappa_q, kappa_p, kappa_g}, exact v)."""
        out = np.zeros(4)
        v64 = np.zeros(nphi(p))
        c = (C.c_int * 5)(*cfg)
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(12)
        wv = np.ascontiguousarray(w, dtype=np.float64).reshape(-1)
        cf = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
        self._check(self._action_bound(p, form, c, _ptr(v, _d), kind, _ptr(cf, _d), _ptr(wv, _d),
                                       _ptr(out, _d), _ptr(v64, _d)))
        return out, v64

    def structured_tet_mesh(self, nx, ny, nz, extent=1.0, jitter=0.15, seed=1):
        nv = (nx + 1) * (ny + 1) * (nz + 1)
        ncell = nx * ny * nz * 6
        verts = np.zeros((nv, 3))
        cells = np.zeros((ncell, 4), dtype=np.int32)
        self._check(self._structured_tet_mesh(nx, ny, nz, extent, jitter, seed,
                                              _ptr(verts, _d), _ptr(cells, _i32)))
        return verts, cells

    def build_dofmap(self, p, verts, cells):
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        cells = np.ascontiguousarray(cells, dtype=np.int32)
        cd = np.zeros((cells.shape[0], nphi(p)), dtype=np.int32)
        nd = C.c_int32(0)
        mm = C.c_int32(0)
        self._check(self._build_dofmap(p, verts.shape[0], _ptr(verts, _d), cells.shape[0],
                                       _ptr(cells, _i32), _ptr(cd, _i32), C.byref(nd),
                                       C.byref(mm)))
        return cd, nd.value, mm.value

    def assemble_matrix(self, cell_dofs, n_dofs, locals_, fmt):
        cd = np.ascontiguousarray(cell_dofs, dtype=np.int32)
        loc = np.ascontiguousarray(locals_, dtype=np.float64)
        ncell, nloc = cd.shape
        nnz = C.c_int64(0)
        fl = C.c_uint32(0)
        self._check(self._assemble_matrix(ncell, nloc, _ptr(cd, _i32), n_dofs, _ptr(loc, _d),
                                          fmt, C.byref(nnz), None, None, None, C.byref(fl)))
        rows = np.zeros(nnz.value, dtype=np.int32)
        cols = np.zeros(nnz.value, dtype=np.int32)
        vals = np.zeros(nnz.value)
        self._check(self._assemble_matrix(ncell, nloc, _ptr(cd, _i32), n_dofs, _ptr(loc, _d),
                                          fmt, C.byref(nnz), _ptr(rows, _i32), _ptr(cols, _i32),
                                          _ptr(vals, _d), C.byref(fl)))
        return rows, cols, vals, fl.value


class Oracle(_Lib):
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            ensure_built(False)
        super().__init__(ORACLE_SO, "orc_")
        self._sig("gen_tets", C.c_int, [C.c_int, C.c_uint64, C.c_int64, _d, _d])
        self._sig("coef_at_q", C.c_int, [C.c_int, _d, C.c_int, _d, _d])

    def gen_tets(self, kind: int, seed: int, m: int):
        v = np.zeros((m, 4, 3))
        coef = np.zeros((m, 4))
        self._check(self._gen_tets(kind, seed, m, _ptr(v, _d), _ptr(coef, _d)))
        return v, coef

    def coef_at_q(self, p, verts, kind, coef=None):
        out = np.zeros(nq(p))
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(12)
        cf = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
        self._check(self._coef_at_q(p, _ptr(v, _d), kind, _ptr(cf, _d), _ptr(out, _d)))
        return out


class Reference(_Lib):
    """The compiled, unmodified reference (oracle/_ref). Only exists where it was built."""

    def __init__(self):
        super().__init__(REF_SO, "ref_")
        self._sig("cpu_baseline", C.c_int, [C.c_int, C.c_int, _int, C.c_int64, _d, C.c_int, _d,
                                             C.c_int, C.c_int, _d, _d])

    def cpu_baseline(self, p, form, cfg, verts, kind, coef, threads):
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 12)
        m = v.shape[0]
        c = (C.c_int * 5)(*cfg)
        cf = None
        stride = 0
        if coef is not None:
            cf = np.ascontiguousarray(coef, dtype=np.float64).reshape(m, -1)
            stride = cf.shape[1]
        secs = C.c_double(0)
        chk = C.c_double(0)
        self._check(self._cpu_baseline(p, form, c, m, _ptr(v, _d), kind, _ptr(cf, _d), stride,
                                       threads, C.byref(secs), C.byref(chk)))
        return secs.value, chk.value


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def box_mesh_cells(nx: int, ny: int, nz: int) -> np.ndarray:
    """Hexahedra of the jittered lattice (mesh.cpp:78-123), vertex b = (x, y, z) bits."""
    cells = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                cells.append([(i + (b & 1)) + (nx + 1) * ((j + ((b >> 1) & 1)) + (ny + 1) * (k + ((b >> 2) & 1)))
                              for b in range(8)])
    return np.array(cells, dtype=np.int32)


def rel_err(approx: np.ndarray, exact: np.ndarray) -> np.ndarray:
    """err_rel(cell) = max|A^ - A| / max|A| (errorlab.cpp:90-99); NaN counts as +inf."""
    a = approx.reshape(approx.shape[0], -1)
    e = exact.reshape(exact.shape[0], -1)
    num = np.max(np.abs(a - e), axis=1)
    den = np.max(np.abs(e), axis=1)
    r = num / den
    r[~np.isfinite(r)] = np.inf
    return r
