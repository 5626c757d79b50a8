"""Global assembly on the device: dof map, CSR sparsity, scatter-add.

Host mirror of the reference's mesh/assembly interface (mesh.hpp:58-68 DofMap /
build_dofmap, assembly.hpp:13-34 SparseCoo / assemble_matrix) over the C-ABI. Arrays are
torch CUDA tensors; the CSR (row_ptr, col_idx, values) holds exactly the reference COO
entries in (row, col) order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import ConfigError, _ptr, _stream_handle, check, lib, nphi

FP32, FP64 = 2, 3
ATOMIC, DETERMINISTIC = 0, 1


@dataclass
class DofMap:  # mesh.hpp:58-65
    n_dofs: int
    n_local: int
    cell_dofs: "object"  # torch.int32 (n_cells, n_local) on device
    max_multiplicity: int

    @property
    def n_cells(self) -> int:
        return int(self.cell_dofs.shape[0])


@dataclass
class CsrPattern:
    n_rows: int
    row_ptr: "object"  # int64 (n_rows + 1)
    col_idx: "object"  # int32 (nnz)
    inc_ptr: "object"  # int64 (n_rows + 1): dof -> incident (cell, local) pairs
    inc: "object"      # int64 (n_cells * n_local), cell * n_local + local, ascending
    pos_map: "object" = None  # int32 (n_cells * n_local^2): CSR position of each local entry
    seg_ptr: "object" = None  # int32 view of uint32 (nnz + 1): contribution segments per CSR entry
    perm: "object" = None     # int32 view of uint32 (n_cells * n_local^2): reference order
    pull_pos: "object" = None  # uint16 (n_cells * n_local^2 + 8): positions in row-pull order

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())


def build_dofmap(p: int, cells, n_verts: int, stream=None) -> DofMap:
    """build_dofmap(mesh, basis(p), continuous) (mesh.cpp:204-298) for a tet mesh given by
    its cell->vertex table `cells` (n, 4) int32 on the device."""
    import torch
    if cells.dtype != torch.int32 or not cells.is_cuda:
        raise ConfigError("cells must be an int32 CUDA tensor")
    n = int(cells.shape[0])
    n_loc = nphi(p)
    cd = torch.empty((n, n_loc), dtype=torch.int32, device=cells.device)
    nd, mm = C.c_int32(0), C.c_int32(0)
    check(lib().mpfem_b200_dofmap(p, _ptr(cells), n, int(n_verts), _ptr(cd), C.byref(nd),
                                  C.byref(mm), _stream_handle(stream)))
    return DofMap(nd.value, n_loc, cd, mm.value)


def incidence(dm: DofMap, stream=None):
    import torch
    dev = dm.cell_dofs.device
    inc_ptr = torch.empty(dm.n_dofs + 1, dtype=torch.int64, device=dev)
    inc = torch.empty(dm.n_cells * dm.n_local, dtype=torch.int64, device=dev)
    check(lib().mpfem_b200_incidence(_ptr(dm.cell_dofs), dm.n_cells, dm.n_local, dm.n_dofs,
                                     _ptr(inc_ptr), _ptr(inc), _stream_handle(stream)))
    return inc_ptr, inc


def csr_pattern(dm: DofMap, stream=None, plan: bool = True, deterministic_plan: bool = False,
                pull_plan: bool = True, pos_map: bool = True) -> CsrPattern:
    """The reference COO key set (assembly.cpp:67-86) as CSR, plus the incidence lists and
    (plan=True) the scatter plan used by assemble_matrix: pos_map, and with
    deterministic_plan=True also seg_ptr/perm for the segment-gather kernel (the default
    deterministic path, row pull, does not need them). pull_plan adds pull_pos, the row-pull
    kernel's own uint16 position stream (half of pos_map's bytes, read sequentially);
    pos_map=False leaves out the int32 pos_map that the atomic and fused scatters use."""
    import torch
    dev = dm.cell_dofs.device
    row_ptr = torch.empty(dm.n_dofs + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64(0)
    sh = _stream_handle(stream)
    check(lib().mpfem_b200_csr_pattern(_ptr(dm.cell_dofs), dm.n_cells, dm.n_local, dm.n_dofs,
                                       _ptr(row_ptr), None, C.byref(nnz), sh))
    col_idx = torch.empty(nnz.value, dtype=torch.int32, device=dev)
    check(lib().mpfem_b200_csr_pattern(_ptr(dm.cell_dofs), dm.n_cells, dm.n_local, dm.n_dofs,
                                       _ptr(row_ptr), _ptr(col_idx), C.byref(nnz), sh))
    inc_ptr, inc = incidence(dm, stream)
    pat = CsrPattern(dm.n_dofs, row_ptr, col_idx, inc_ptr, inc)
    if plan:
        nk = dm.n_cells * dm.n_local * dm.n_local
        if pos_map or deterministic_plan or not pull_plan:
            pat.pos_map = torch.empty(nk, dtype=torch.int32, device=dev)
        if deterministic_plan:
            pat.seg_ptr = torch.empty(nnz.value + 1, dtype=torch.int32, device=dev)
            pat.perm = torch.empty(nk, dtype=torch.int32, device=dev)
        if pull_plan:
            pat.pull_pos = torch.empty(nk + 8, dtype=torch.uint16, device=dev)

        def build():
            check(lib().mpfem_b200_scatter_plan_pull(_ptr(dm.cell_dofs), None, dm.n_cells, dm.n_local,
                                                     dm.n_dofs, _ptr(row_ptr), _ptr(col_idx),
                                                     _ptr(pat.pos_map), _ptr(pat.seg_ptr),
                                                     _ptr(pat.perm), _ptr(pat.pull_pos), sh))
        try:
            build()
        except ConfigError:
            # rows beyond pull_pos's uint16 range (high p): the row-pull kernel reads pos_map
            if pat.pull_pos is None:
                raise
            pat.pull_pos = None
            if pat.pos_map is None:
                pat.pos_map = torch.empty(nk, dtype=torch.int32, device=dev)
            build()
    return pat


def assemble_matrix(local, dm: DofMap, pat: CsrPattern, fmt: int = FP64,
                    mode: int = DETERMINISTIC, cell_begin: int = 0, cell_end: int | None = None,
                    rows=None, accumulate: bool = False, values=None, stream=None,
                    pull: bool | None = None):
    """assemble_matrix (assembly.cpp:41-88) into CSR values at fmt (fp32/fp64).

    `local` holds the local matrices of cells [cell_begin, cell_end), (n, n_loc, n_loc)
    fp32 or fp64. Deterministic mode reproduces the reference's ascending-cell sequential
    sum bitwise; atomic mode is order-free (within gamma_{m+1} of the exact sum).
    Deterministic mode runs the row-pull kernel (incidence lists + pos_map: rows replay their
    incident local rows in ascending cell order from shared memory). Patterns built with
    deterministic_plan=True carry seg_ptr/perm (13 GB at config-4 P3) and use the block-staged
    segment gather instead unless pull=True -- the same bits, about 1.5x slower at config 4."""
    import torch
    if cell_end is None:
        cell_end = cell_begin + int(local.shape[0])
    if local.dtype == torch.float32:
        lf = FP32
    elif local.dtype == torch.float64:
        lf = FP64
    else:
        raise ConfigError("local matrices must be fp32 or fp64")
    if values is None:
        values = torch.empty(pat.nnz, dtype=torch.float32 if fmt == FP32 else torch.float64,
                             device=local.device)
    n_rows = 0 if rows is None else int(rows.numel())
    if pat.pos_map is None and pat.pull_pos is None:
        raise ConfigError("assemble_matrix needs a pattern built with plan=True")
    if pull is None:
        pull = pat.seg_ptr is None
    if pat.pos_map is None and not (mode == DETERMINISTIC and pull):
        raise ConfigError("this assembly mode needs a pattern built with pos_map=True")
    if mode == DETERMINISTIC and pull:
        # row-pull: incidence lists + pos_map, no seg_ptr/perm plan needed
        check(lib().mpfem_b200_assemble_pull(_ptr(local), lf, int(cell_begin), int(cell_end),
                                             dm.n_local, _ptr(pat.row_ptr), dm.n_dofs,
                                             _ptr(pat.inc_ptr), _ptr(pat.inc), _ptr(pat.pos_map),
                                             _ptr(pat.pull_pos), _ptr(values), int(fmt),
                                             int(accumulate), _ptr(rows), n_rows,
                                             _stream_handle(stream)))
        return values
    check(lib().mpfem_b200_assemble(_ptr(local), lf, int(cell_begin), int(cell_end), dm.n_local,
                                    _ptr(pat.row_ptr), dm.n_dofs, _ptr(pat.pos_map),
                                    _ptr(pat.seg_ptr), _ptr(pat.perm), _ptr(values), int(fmt),
                                    int(mode), int(accumulate), _ptr(rows), n_rows,
                                    _stream_handle(stream)))
    return values


def assemble_cells(setup, verts, cells, dm: DofMap, pat: CsrPattern, fmt: int = FP64,
                   coef_kind: int = 0, coef=None, cell_begin: int = 0, accumulate: bool = False,
                   values=None, stream=None, want_flags: bool = False):
    """Cell kernels fused with the atomic CSR scatter (run_assemble's bilinear_kernel ->
    assemble_matrix loop, mpfem_cli.cpp:322-332, in the order-free atomic mode): adds the
    local matrices of `cells` (global cells cell_begin .. cell_begin + len(cells)) into the
    CSR values. On the tcgen05 path K2 adds straight from TMEM, so the local matrices never
    reach HBM. Values are within gamma_{m+1}(fmt) * sum|contrib| of the exact sum."""
    import torch
    if pat.pos_map is None:
        raise ConfigError("assemble_cells needs a pattern built with plan=True")
    n = int(cells.shape[0])
    per = dm.n_local * dm.n_local
    if values is None:
        values = torch.zeros(pat.nnz, dtype=torch.float32 if fmt == FP32 else torch.float64,
                             device=cells.device)
    elif not accumulate:
        values.zero_()
    stride = 0 if coef is None else int(coef.shape[-1]) if coef.dim() > 1 else 0
    fl = C.c_uint32(0)
    pm = pat.pos_map[cell_begin * per:(cell_begin + n) * per]
    check(lib().mpfem_b200_cell_matrices_scatter(setup._h, _ptr(verts), _ptr(cells), n, int(coef_kind),
                                                 _ptr(coef), stride, _ptr(pm), _ptr(values), int(fmt),
                                                 _stream_handle(stream),
                                                 C.byref(fl) if want_flags else None))
    return (values, fl.value) if want_flags else values


class CudaPartitionBackend:
    """The device operations of the partitioned multi-GPU assembly (distributed.py) on the
    C-ABI: first-encounter dof maps of cell ranges, the layer table / globalisation of the
    numbering, local-row / global-column CSR patterns with their scatter plan, CSR position
    lookup, and the rows-restricted deterministic scatter."""

    def dofmap(self, p: int, cells, n_verts: int):
        dm = build_dofmap(p, cells, n_verts)
        return dm.cell_dofs, dm.n_dofs

    def table(self, key, val, n_table: int):
        import torch
        t = torch.full((max(n_table, 1),), -1, dtype=torch.int32, device=key.device)
        check(lib().mpfem_b200_dofmap_table(_ptr(key), _ptr(val), int(key.numel()), _ptr(t), _stream_handle(None)))
        return t[:n_table]

    def globalize(self, local, table, n_table: int, offset: int):
        import torch
        out = torch.empty_like(local)
        tb = table if table is not None and table.numel() else torch.zeros(1, dtype=torch.int32, device=local.device)
        check(lib().mpfem_b200_dofmap_globalize(_ptr(local), int(local.numel()), _ptr(tb), int(n_table),
                                                int(offset), _ptr(out), _stream_handle(None)))
        return out

    def pattern(self, row_dofs, col_dofs, n_rows: int):
        import torch
        dev = row_dofs.device
        n, n_loc = int(row_dofs.shape[0]), int(row_dofs.shape[1])
        row_ptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
        nnz = C.c_int64(0)
        sh = _stream_handle(None)
        check(lib().mpfem_b200_csr_pattern_cols(_ptr(row_dofs), _ptr(col_dofs), n, n_loc, n_rows,
                                                _ptr(row_ptr), None, C.byref(nnz), sh))
        col_idx = torch.empty(nnz.value, dtype=torch.int32, device=dev)
        check(lib().mpfem_b200_csr_pattern_cols(_ptr(row_dofs), _ptr(col_dofs), n, n_loc, n_rows,
                                                _ptr(row_ptr), _ptr(col_idx), C.byref(nnz), sh))
        inc_ptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
        inc = torch.empty(n * n_loc, dtype=torch.int64, device=dev)
        check(lib().mpfem_b200_incidence(_ptr(row_dofs), n, n_loc, n_rows, _ptr(inc_ptr), _ptr(inc), sh))
        pat = CsrPattern(n_rows, row_ptr, col_idx, inc_ptr, inc)
        nk = n * n_loc * n_loc
        pat.pos_map = torch.empty(nk, dtype=torch.int32, device=dev)
        pat.pull_pos = torch.empty(nk + 8, dtype=torch.uint16, device=dev)
        try:
            check(lib().mpfem_b200_scatter_plan_pull(_ptr(row_dofs), _ptr(col_dofs), n, n_loc, n_rows,
                                                     _ptr(row_ptr), _ptr(col_idx), _ptr(pat.pos_map),
                                                     None, None, _ptr(pat.pull_pos), sh))
        except ConfigError:  # rows beyond pull_pos's uint16 range: pos_map only
            pat.pull_pos = None
            check(lib().mpfem_b200_scatter_plan_pull(_ptr(row_dofs), _ptr(col_dofs), n, n_loc, n_rows,
                                                     _ptr(row_ptr), _ptr(col_idx), _ptr(pat.pos_map),
                                                     None, None, None, sh))
        pat.n_local = n_loc
        return pat

    def find(self, pat, rows, cols):
        import torch
        pos = torch.empty(int(rows.numel()), dtype=torch.int64, device=rows.device)
        check(lib().mpfem_b200_csr_find(_ptr(pat.row_ptr), _ptr(pat.col_idx), _ptr(rows), _ptr(cols),
                                        int(rows.numel()), _ptr(pos), _stream_handle(None)))
        return pos

    def assemble_rows(self, local, pat, fmt, cell_begin, cell_end, rows, accumulate, values):
        if rows is None or rows.numel() == 0:
            return values
        lf = FP32 if local.dtype.itemsize == 4 else FP64
        check(lib().mpfem_b200_assemble_pull(_ptr(local), lf, int(cell_begin), int(cell_end), pat.n_local,
                                             _ptr(pat.row_ptr), pat.n_rows, _ptr(pat.inc_ptr),
                                             _ptr(pat.inc), _ptr(pat.pos_map), _ptr(pat.pull_pos),
                                             _ptr(values), int(fmt), int(accumulate), _ptr(rows),
                                             int(rows.numel()),
                                             _stream_handle(None)))
        return values
