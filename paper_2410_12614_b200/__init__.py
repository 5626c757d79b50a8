"""B200-native hot path of arXiv 2410.12614: batched mass/Poisson cell matrices on affine
tetrahedra (Lagrange P1-P8) and CSR assembly, behind the reference's kernel API.

This module is the Python host mirror of the reference's C++ interface
(/root/reference/proj/include/mpfem/kernels.hpp, mesh.hpp, assembly.hpp): the same names,
argument meaning and error behaviour (ConfigError / CheckError), on top of the C-ABI in
include/mpfem_b200.h (paper_2410_12614_b200/lib/libmpfem_b200.so). There is no CPU
fallback: without the CUDA library or a GPU every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Fmt", "FormKind", "ModeKind", "EngineKind", "CoefKind", "KernelConfig", "KernelSetup",
    "ConfigError", "CheckError", "RuntimeFailure", "reference_config", "make_setup",
    "bilinear_kernel", "action_kernel", "mode_config", "lib", "LIB_PATH",
]

LIB_PATH = os.environ.get("MPFEM_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libmpfem_b200.so")


class Fmt(enum.IntEnum):  # softfloat.hpp:17
    bf16 = 0
    fp16 = 1
    fp32 = 2
    fp64 = 3


class FormKind(enum.IntEnum):  # geometry.hpp:107
    mass = 0
    poisson = 1


class ModeKind(enum.IntEnum):  # kernels.hpp:11
    bilinear = 0
    action = 1


class EngineKind(enum.IntEnum):  # mm_units.hpp:31
    scalar = 0
    vector = 1
    matrix = 2


class CoefKind(enum.IntEnum):
    one = 0            # empty z: multiplication skipped
    sincosexp = 1      # c(x) = 1 + 0.5 sin(2 pi x) cos(2 pi y) e^z (BASELINE configs 0-2, 4)
    exp10_affine = 2   # c = 10^(6 u(x)), u affine per cell (BASELINE config 3)
    nodal = 3          # nodal FE coefficient z (kernels.cpp:114-136)


class ConfigError(ValueError):
    """Invalid user input (common.hpp:10-12); C-ABI status 2."""


class CheckError(RuntimeError):
    """A verification failed: singular cell, bad dof (common.hpp:15-17); C-ABI status 3."""


class RuntimeFailure(RuntimeError):
    """CUDA or device failure (no GPU, launch error); C-ABI status 4."""


@dataclass
class KernelConfig:  # kernels.hpp:20-29
    form: FormKind = FormKind.mass
    mode: ModeKind = ModeKind.bilinear
    u_p: Fmt = Fmt.fp64
    u_g: Fmt = Fmt.fp64
    u_q: Fmt = Fmt.fp64
    u_s: Fmt = Fmt.fp64
    engine: EngineKind = EngineKind.scalar
    n_batch: int = 64


def reference_config(form: FormKind, mode: ModeKind = ModeKind.bilinear) -> KernelConfig:
    """kernels.cpp:48-53: all-fp64, scalar engine."""
    return KernelConfig(form=FormKind(form), mode=ModeKind(mode))


# BASELINE.json precision modes -> KernelConfig
_MODES = {
    "fp64": (Fmt.fp64, Fmt.fp64, Fmt.fp64, Fmt.fp64, EngineKind.scalar),
    "fp32": (Fmt.fp32, Fmt.fp32, Fmt.fp32, Fmt.fp32, EngineKind.scalar),
    "fp16": (Fmt.fp16, Fmt.fp32, Fmt.fp16, Fmt.fp16, EngineKind.scalar),
    "mixed": (Fmt.fp32, Fmt.fp32, Fmt.fp32, Fmt.fp16, EngineKind.scalar),
    "mixed_bf16": (Fmt.fp32, Fmt.fp32, Fmt.fp32, Fmt.bf16, EngineKind.matrix),
}


def mode_config(mode: str, form: FormKind, geometry_fp64: bool = False) -> KernelConfig:
    up, ug, uq, us, eng = _MODES[mode]
    if geometry_fp64:
        ug = Fmt.fp64  # BASELINE config 1: G_K computed in fp64
    return KernelConfig(form=FormKind(form), u_p=up, u_g=ug, u_q=uq, u_s=us, engine=eng)


_lib = None


def lib():
    """Loads the CUDA product library; raises if it is missing (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeFailure(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, i32p, i64p, u32p, dp = (C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                C.POINTER(C.c_uint32), C.POINTER(C.c_double))
    sig = {
        "mpfem_b200_last_error": (C.c_char_p, []),
        "mpfem_b200_version": (C.c_char_p, []),
        "mpfem_b200_setup_create": (C.c_int, [C.c_int] * 10 + [C.POINTER(vp)]),
        "mpfem_b200_setup_destroy": (C.c_int, [vp]),
        "mpfem_b200_setup_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), i64p, i64p, C.POINTER(C.c_int)]),
        "mpfem_b200_setup_rule": (C.c_int, [vp, dp, dp]),
        "mpfem_b200_cell_matrices": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, vp, C.c_int64, vp,
                                               C.c_int64, vp, u32p]),
        "mpfem_b200_cell_matrices_scatter": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, vp, C.c_int64,
                                                       vp, vp, C.c_int, vp, u32p]),
        "mpfem_b200_cell_matrices_host": (C.c_int, [vp, vp, C.c_int64, vp, C.c_int64, C.c_int, vp,
                                                    C.c_int64, vp, C.c_int64, vp, u32p]),
        "mpfem_b200_reserve": (C.c_int, [vp, C.c_int64, vp]),
        "mpfem_b200_synchronize": (C.c_int, [vp, vp]),
        "mpfem_b200_action": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, vp, C.c_int64, vp,
                                        C.c_int64, vp, C.c_int64, vp, u32p]),
        "mpfem_b200_cell_bounds": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, vp, C.c_int64, vp, vp,
                                             vp]),
        "mpfem_b200_action_bounds": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, vp, C.c_int64, vp,
                                               C.c_int64, vp, vp, vp]),
        "mpfem_b200_action_host": (C.c_int, [vp, vp, C.c_int64, vp, C.c_int64, C.c_int, vp,
                                             C.c_int64, vp, C.c_int64, vp, C.c_int64, vp, u32p]),
        "mpfem_b200_scaled_weights": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int, vp, C.c_int64, vp,
                                                vp, u32p]),
        "mpfem_b200_last_launch_count": (C.c_int, [vp]),
        "mpfem_b200_set_timing": (C.c_int, [vp, C.c_int]),
        "mpfem_b200_last_timings": (C.c_int, [vp, C.POINTER(C.c_float), C.c_int]),
        "mpfem_b200_gen_tets": (C.c_int, [C.c_int, C.c_uint64, C.c_int64, vp, vp]),
        "mpfem_b200_structured_tet_mesh": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double,
                                                     C.c_double, C.c_uint64, vp, vp]),
        "mpfem_b200_dofmap": (C.c_int, [C.c_int, vp, C.c_int64, C.c_int64, vp, i32p, i32p, vp]),
        "mpfem_b200_csr_pattern": (C.c_int, [vp, C.c_int64, C.c_int, C.c_int32, vp, vp, i64p, vp]),
        "mpfem_b200_incidence": (C.c_int, [vp, C.c_int64, C.c_int, C.c_int32, vp, vp, vp]),
        "mpfem_b200_scatter_plan": (C.c_int, [vp, C.c_int64, C.c_int, C.c_int32, vp, vp, vp, vp,
                                              vp, vp]),
        "mpfem_b200_assemble": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int64, C.c_int, vp,
                                          C.c_int32, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int,
                                          vp, C.c_int64, vp]),
        "mpfem_b200_assemble_pull": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int64, C.c_int, vp,
                                               C.c_int32, vp, vp, vp, vp, vp, C.c_int, C.c_int, vp,
                                               C.c_int64, vp]),
        "mpfem_b200_scatter_plan_pull": (C.c_int, [vp, vp, C.c_int64, C.c_int, C.c_int32, vp, vp, vp,
                                                   vp, vp, vp, vp]),
        "mpfem_b200_csr_pattern_cols": (C.c_int, [vp, vp, C.c_int64, C.c_int, C.c_int32, vp, vp, i64p, vp]),
        "mpfem_b200_scatter_plan_cols": (C.c_int, [vp, vp, C.c_int64, C.c_int, C.c_int32, vp, vp, vp,
                                                   vp, vp, vp]),
        "mpfem_b200_dofmap_table": (C.c_int, [vp, vp, C.c_int64, vp, vp]),
        "mpfem_b200_dofmap_globalize": (C.c_int, [vp, C.c_int64, vp, C.c_int32, C.c_int32, vp, vp]),
        "mpfem_b200_csr_find": (C.c_int, [vp, vp, vp, vp, C.c_int64, vp, vp]),
        "mpfem_b200_dofmap_cells": (C.c_int, [C.c_int, C.c_int, vp, C.c_int64, C.c_int64, vp, i32p, i32p, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name, None)
        if f is None:
            continue
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().mpfem_b200_last_error().decode()
    if status == 2:
        raise ConfigError(msg)
    if status == 3:
        raise CheckError(msg)
    raise RuntimeFailure(msg)


def _ptr(t) -> int | None:
    """Raw device/host address of a torch tensor or numpy array (None passes through)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream_handle(stream) -> int | None:
    if stream is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:
            return None
    return getattr(stream, "cuda_stream", stream)


def nphi(p: int) -> int:
    return (p + 1) * (p + 2) * (p + 3) // 6


class KernelSetup:
    """Device-resident counterpart of the reference KernelSetup (kernels.hpp:47-58):
    rule, tabulations and the shared basis-product operand, immutable per config."""

    def __init__(self, p: int, config: KernelConfig, cell_kind: int = 0, dim: int = 3):
        self.p = p
        self.config = config
        h = C.c_void_p()
        check(lib().mpfem_b200_setup_create(cell_kind, dim, p, int(config.form), int(config.u_p),
                                            int(config.u_g), int(config.u_q), int(config.u_s),
                                            int(config.engine), int(config.n_batch), C.byref(h)))
        self._h = h
        n_phi, n_q, n_d, path = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        k, k_pad = C.c_int64(), C.c_int64()
        check(lib().mpfem_b200_setup_info(h, C.byref(n_phi), C.byref(n_q), C.byref(n_d),
                                          C.byref(k), C.byref(k_pad), C.byref(path)))
        self.n_phi, self.n_q, self.n_d = n_phi.value, n_q.value, n_d.value
        self.k, self.k_pad, self.path = k.value, k_pad.value, path.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().mpfem_b200_setup_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def out_dtype(self):
        return np.float64 if self.path == 2 else np.float32

    def rule(self):
        pts = np.zeros((self.n_q, 3))
        w = np.zeros(self.n_q)
        check(lib().mpfem_b200_setup_rule(self._h, pts.ctypes.data_as(C.POINTER(C.c_double)),
                                          w.ctypes.data_as(C.POINTER(C.c_double))))
        return pts, w

    def reserve(self, n_cells: int, stream=None) -> None:
        """Pre-sizes the scratch of `stream`'s workspace (graph-capture safe calls after)."""
        check(lib().mpfem_b200_reserve(self._h, int(n_cells), _stream_handle(stream)))

    def synchronize(self, stream=None) -> None:
        """Waits for `stream`; raises CheckError if a call on this setup met a singular cell
        since the last report (asynchronous calls without want_flags report it here or on
        the next call, see include/mpfem_b200.h)."""
        check(lib().mpfem_b200_synchronize(self._h, _stream_handle(stream)))

    def cell_matrices(self, verts, cells=None, coef_kind: int = CoefKind.one, coef=None, out=None,
                      out_pitch: int | None = None, stream=None, want_flags: bool = False):
        """Batched cell_geometry + bilinear_kernel on device tensors (torch, cuda).
        verts: (n, 4, 3) float64 private vertices, or the (n_verts, 3) table when `cells`
        (n, 4) int32 is given. Returns out (n, n_phi, n_phi) [and the FP flag mask]."""
        import torch
        n = int(cells.shape[0]) if cells is not None else int(verts.shape[0])
        n2 = self.n_phi * self.n_phi
        pitch = out_pitch or n2
        dt = torch.float64 if self.path == 2 else torch.float32
        if out is None:
            out = torch.empty((n, pitch), dtype=dt, device=verts.device)
        stride = 0 if coef is None else int(coef.shape[-1]) if coef.dim() > 1 else int(coef.numel() // max(n, 1))
        fl = C.c_uint32(0)
        check(lib().mpfem_b200_cell_matrices(self._h, _ptr(verts), _ptr(cells), n, int(coef_kind),
                                             _ptr(coef), stride, _ptr(out), pitch,
                                             _stream_handle(stream),
                                             C.byref(fl) if want_flags else None))
        res = out[:, :n2].reshape(n, self.n_phi, self.n_phi) if pitch == n2 else out
        return (res, fl.value) if want_flags else res

    def cell_matrices_host(self, verts: np.ndarray, cells: np.ndarray | None = None,
                           coef_kind: int = CoefKind.one, coef: np.ndarray | None = None,
                           out: np.ndarray | None = None, stream=None, want_flags: bool = False):
        """Same on host (numpy) buffers: H2D, compute, D2H inside the call."""
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        n = cells.shape[0] if cells is not None else verts.shape[0]
        n_verts = verts.reshape(-1, 3).shape[0] if cells is not None else 0
        if cells is not None:
            cells = np.ascontiguousarray(cells, dtype=np.int32)
        stride = 0
        if coef is not None:
            coef = np.ascontiguousarray(coef, dtype=np.float64).reshape(n, -1)
            stride = coef.shape[1]
        n2 = self.n_phi * self.n_phi
        if out is None:
            out = np.empty((n, self.n_phi, self.n_phi), dtype=self.out_dtype)
        fl = C.c_uint32(0)
        check(lib().mpfem_b200_cell_matrices_host(self._h, _ptr(verts), n_verts, _ptr(cells), n,
                                                  int(coef_kind), _ptr(coef), stride, _ptr(out), n2,
                                                  _stream_handle(stream),
                                                  C.byref(fl) if want_flags else None))
        return (out, fl.value) if want_flags else out

    def scaled_weights(self, verts, cells=None, coef_kind: int = CoefKind.one, coef=None,
                       stream=None):
        """Device W operand (n, K) as fp64 carriers; parity/debug entry."""
        import torch
        n = int(cells.shape[0]) if cells is not None else int(verts.shape[0])
        out = torch.empty((n, self.k), dtype=torch.float64, device=verts.device)
        stride = 0 if coef is None else int(coef.shape[-1])
        fl = C.c_uint32(0)
        check(lib().mpfem_b200_scaled_weights(self._h, _ptr(verts), _ptr(cells), n, int(coef_kind),
                                              _ptr(coef), stride, _ptr(out), _stream_handle(stream),
                                              C.byref(fl)))
        return out, fl.value

    def action(self, verts, w, cells=None, coef_kind: int = CoefKind.one, coef=None, out=None,
               stream=None, want_flags: bool = False):
        """Batched action_kernel (Algorithm 2) on device tensors: w (n, n_phi) float64 FE
        coefficients per cell -> v (n, n_phi), row c = the reference's column c. Bitwise the
        reference's result in every mode. A 1-D coef (one nodal z for the whole batch, as the
        reference's action_kernel takes it) is shared by all cells."""
        import torch
        n = int(cells.shape[0]) if cells is not None else int(verts.shape[0])
        if w.dim() != 2 or w.shape[0] != n:
            raise ConfigError("action batch needs one coefficient vector per cell")
        dt = torch.float64 if self.config.u_q == Fmt.fp64 else torch.float32
        if out is None:
            out = torch.empty((n, self.n_phi), dtype=dt, device=w.device)
        # a 1-D coef is one vector shared by the batch (stride 0), as the reference's z
        stride = 0 if coef is None or coef.dim() == 1 else int(coef.stride(0))
        fl = C.c_uint32(0)
        check(lib().mpfem_b200_action(self._h, _ptr(verts), _ptr(cells), n, int(coef_kind),
                                      _ptr(coef), stride, _ptr(w), int(w.stride(0)), _ptr(out),
                                      int(out.stride(0)), _stream_handle(stream),
                                      C.byref(fl) if want_flags else None))
        return (out, fl.value) if want_flags else out

    def action_host(self, verts: np.ndarray, w: np.ndarray, cells: np.ndarray | None = None,
                    coef_kind: int = CoefKind.one, coef: np.ndarray | None = None, stream=None,
                    want_flags: bool = False):
        """Same on host (numpy) buffers: H2D, compute, D2H inside the call."""
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        n = cells.shape[0] if cells is not None else verts.shape[0]
        n_verts = verts.reshape(-1, 3).shape[0] if cells is not None else 0
        if cells is not None:
            cells = np.ascontiguousarray(cells, dtype=np.int32)
        w = np.ascontiguousarray(w, dtype=np.float64).reshape(n, -1)
        stride = 0
        if coef is not None:
            coef = np.ascontiguousarray(coef, dtype=np.float64).reshape(n, -1)
            stride = coef.shape[1]
        out = np.empty((n, self.n_phi), dtype=np.float64 if self.config.u_q == Fmt.fp64 else np.float32)
        fl = C.c_uint32(0)
        check(lib().mpfem_b200_action_host(self._h, _ptr(verts), n_verts, _ptr(cells), n,
                                           int(coef_kind), _ptr(coef), stride, _ptr(w), w.shape[1],
                                           _ptr(out), self.n_phi, _stream_handle(stream),
                                           C.byref(fl) if want_flags else None))
        return (out, fl.value) if want_flags else out

    def cell_bounds(self, verts, cells=None, coef_kind: int = CoefKind.one, coef=None,
                    want_a64: bool = False, stream=None):
        """kernel_bounds (bounds.cpp:29-281, bilinear part) for every cell on the GPU:
        (n, 4) float64 {bound_a, kappa_q, kappa_p, kappa_g} [and the exact A (n, n_phi, n_phi)]."""
        import torch
        n = int(cells.shape[0]) if cells is not None else int(verts.shape[0])
        out = torch.empty((n, 4), dtype=torch.float64, device=verts.device)
        a64 = torch.empty((n, self.n_phi, self.n_phi), dtype=torch.float64, device=verts.device) if want_a64 else None
        stride = 0 if coef is None else int(coef.shape[-1])
        check(lib().mpfem_b200_cell_bounds(self._h, _ptr(verts), _ptr(cells), n, int(coef_kind),
                                           _ptr(coef), stride, _ptr(out), _ptr(a64),
                                           _stream_handle(stream)))
        return (out, a64) if want_a64 else out

    def action_bounds(self, verts, w, cells=None, coef_kind: int = CoefKind.one, coef=None,
                      want_v64: bool = False, stream=None):
        """kernel_bounds' action part for every cell on the GPU: (n, 4) {bound_v, kappa_q,
        kappa_p, kappa_g} [and the exact v (n, n_phi)]."""
        import torch
        n = int(cells.shape[0]) if cells is not None else int(verts.shape[0])
        out = torch.empty((n, 4), dtype=torch.float64, device=verts.device)
        v64 = torch.empty((n, self.n_phi), dtype=torch.float64, device=verts.device) if want_v64 else None
        stride = 0 if coef is None else int(coef.shape[-1])
        check(lib().mpfem_b200_action_bounds(self._h, _ptr(verts), _ptr(cells), n, int(coef_kind),
                                             _ptr(coef), stride, _ptr(w), int(w.stride(0)), _ptr(out),
                                             _ptr(v64), _stream_handle(stream)))
        return (out, v64) if want_v64 else out

    def last_launch_count(self) -> int:
        return lib().mpfem_b200_last_launch_count(self._h)

    def set_timing(self, enable: bool) -> None:
        check(lib().mpfem_b200_set_timing(self._h, int(enable)))

    def last_timings(self) -> list[float]:
        """Durations (ms) of K1 and K2 of the last call, from CUDA events on its stream."""
        buf = (C.c_float * 8)()
        n = lib().mpfem_b200_last_timings(self._h, buf, 8)
        if n < 0:
            check(-n)
        return [buf[i] for i in range(n)]


def make_setup(p: int, config: KernelConfig, cell_kind: int = 0, dim: int = 3) -> KernelSetup:
    """make_setup (kernels.hpp:60-62) for affine tetrahedra (bilinear or action mode)."""
    return KernelSetup(p, config, cell_kind, dim)


def bilinear_kernel(setup: KernelSetup, verts, cells=None, coef_kind: int = CoefKind.one,
                    coef=None, **kw):
    """Batched bilinear_kernel (kernels.hpp:85-86): one n_phi x n_phi matrix per cell."""
    if setup.config.mode != ModeKind.bilinear:
        raise ConfigError("configuration is not a bilinear-mode config")
    return setup.cell_matrices(verts, cells, coef_kind, coef, **kw)


def action_kernel(setup: KernelSetup, verts, w, cells=None, coef_kind: int = CoefKind.one,
                  coef=None, **kw):
    """Batched action_kernel (kernels.hpp:90-92): v (n, n_phi), bitwise the reference's."""
    if setup.config.mode != ModeKind.action:
        raise ConfigError("configuration is not an action-mode config")
    return setup.action(verts, w, cells, coef_kind, coef, **kw)


def gen_tets(kind: int, seed: int, n: int):
    """Seeded synthetic tets (BASELINE configs 0-3) on the host: (verts (n,4,3), coef (n,4))."""
    verts = np.zeros((n, 4, 3))
    coef = np.zeros((n, 4))
    check(lib().mpfem_b200_gen_tets(int(kind), int(seed), int(n), _ptr(verts), _ptr(coef)))
    return verts, coef


def structured_tet_mesh(nx: int, ny: int, nz: int, extent: float = 1.0, jitter: float = 0.15,
                        seed: int = 1):
    """structured_tet_mesh (mesh.hpp:38-39 defaults): (vertices (nv,3), cells (nc,4) int32)."""
    verts = np.zeros(((nx + 1) * (ny + 1) * (nz + 1), 3))
    cells = np.zeros((6 * nx * ny * nz, 4), dtype=np.int32)
    check(lib().mpfem_b200_structured_tet_mesh(nx, ny, nz, float(extent), float(jitter), int(seed),
                                               _ptr(verts), _ptr(cells)))
    return verts, cells
