"""CPU stand-in for the assembly backend (TEST INFRASTRUCTURE): the dof map and pattern
from the oracle (the reference algorithm), and a direct restatement of the deterministic
row-centric scatter (ascending-cell sequential sum per entry, assembly.cpp:50-67) on torch
CPU tensors, so the multi-rank host logic of paper_2410_12614_b200.distributed runs under
gloo without a GPU."""
from dataclasses import dataclass

import numpy as np
import torch

from oracle_lib import Oracle, nphi


@dataclass
class DM:
    n_dofs: int
    n_local: int
    cell_dofs: torch.Tensor
    max_multiplicity: int

    @property
    def n_cells(self):
        return int(self.cell_dofs.shape[0])


@dataclass
class Pat:
    n_rows: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    inc_ptr: torch.Tensor
    inc: torch.Tensor

    @property
    def nnz(self):
        return int(self.col_idx.numel())


class CpuBackend:
    def __init__(self):
        self.O = Oracle()

    def build(self, p, verts, cells):
        cd, nd, mm = self.O.build_dofmap(p, verts, cells)
        dm = DM(nd, nphi(p), torch.from_numpy(cd), mm)
        n_loc = nphi(p)
        flat = cd.reshape(-1)
        order = np.argsort(flat, kind="stable")
        counts = np.bincount(flat, minlength=nd)
        inc_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        rows, cols = [], []
        for r in range(nd):
            cs = set()
            for pk in order[inc_ptr[r]:inc_ptr[r + 1]]:
                cs.update(cd[pk // n_loc].tolist())
            cs = sorted(cs)
            rows.append(len(cs))
            cols.extend(cs)
        row_ptr = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
        pat = Pat(nd, torch.from_numpy(row_ptr), torch.from_numpy(np.array(cols, dtype=np.int32)),
                  torch.from_numpy(inc_ptr), torch.from_numpy(order.astype(np.int64)))
        return dm, pat

    def assemble_matrix(self, local, dm, pat, fmt, mode, cell_begin, cell_end, rows=None,
                        accumulate=False, values=None):
        n_loc = dm.n_local
        cd = dm.cell_dofs.numpy()
        rp = pat.row_ptr.numpy()
        ci = pat.col_idx.numpy()
        ip = pat.inc_ptr.numpy()
        inc = pat.inc.numpy()
        dt = np.float32 if fmt == 2 else np.float64
        loc = local.numpy()
        vals = values.numpy()  # shares memory with the torch tensor
        rr = range(dm.n_dofs) if rows is None else rows.numpy().tolist()
        for r in rr:
            b, e = rp[r], rp[r + 1]
            if not accumulate:
                vals[b:e] = dt(-0.0)
            for pk in inc[ip[r]:ip[r + 1]]:
                c, i = divmod(int(pk), n_loc)
                if c < cell_begin or c >= cell_end:
                    continue
                for j in range(n_loc):
                    x = b + np.searchsorted(ci[b:e], cd[c, j])
                    vals[x] = dt(vals[x] + dt(loc[c - cell_begin, i, j]))
        return values
