"""CPU stand-in for the partitioned assembly backend (TEST INFRASTRUCTURE): the same operations
as paper_2410_12614_b200.assembly.CudaPartitionBackend restated in numpy on torch CPU tensors
-- dof maps from the oracle (the reference algorithm, mesh.cpp:204-298), CSR patterns by
explicit row unions, the deterministic row-centric scatter as the ascending-cell sequential
sum per entry (assembly.cpp:50-67) -- so the multi-rank host logic of
paper_2410_12614_b200.distributed runs under gloo without a GPU."""
from dataclasses import dataclass

import numpy as np
import torch

from oracle_lib import Oracle


@dataclass
class Pat:
    n_rows: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    inc_ptr: torch.Tensor
    inc: torch.Tensor
    col_dofs: np.ndarray
    n_local: int

    @property
    def nnz(self):
        return int(self.col_idx.numel())


class CpuPartitionBackend:
    def __init__(self, verts):
        self.O = Oracle()
        self.verts = verts

    def dofmap(self, p, cells, n_verts):
        cd, nd, _ = self.O.build_dofmap(p, self.verts, cells.numpy())
        return torch.from_numpy(cd.astype(np.int32)), nd

    def table(self, key, val, n_table):
        t = np.full(max(n_table, 1), -1, dtype=np.int32)
        t[key.numpy().astype(np.int64)] = val.numpy()
        return torch.from_numpy(t[:n_table])

    def globalize(self, local, table, n_table, offset):
        loc = local.numpy()
        tab = table.numpy()
        out = np.where(loc < n_table, tab[np.minimum(loc, max(n_table - 1, 0))] if n_table else 0,
                       offset + loc - n_table)
        return torch.from_numpy(out.astype(np.int32))

    def pattern(self, row_dofs, col_dofs, n_rows):
        rd = row_dofs.numpy()
        cd = col_dofs.numpy()
        n_loc = rd.shape[1]
        flat = rd.reshape(-1)
        order = np.argsort(flat, kind="stable")
        counts = np.bincount(flat, minlength=n_rows)
        inc_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        lens, cols = [], []
        for r in range(n_rows):
            cs = sorted({int(x) for pk in order[inc_ptr[r]:inc_ptr[r + 1]] for x in cd[pk // n_loc]})
            lens.append(len(cs))
            cols.extend(cs)
        row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        return Pat(n_rows, torch.from_numpy(row_ptr), torch.from_numpy(np.array(cols, dtype=np.int32)),
                   torch.from_numpy(inc_ptr), torch.from_numpy(order.astype(np.int64)), cd, n_loc)

    def find(self, pat, rows, cols):
        rp = pat.row_ptr.numpy()
        ci = pat.col_idx.numpy()
        out = np.empty(rows.numel(), dtype=np.int64)
        for t, (r, c) in enumerate(zip(rows.numpy(), cols.numpy())):
            b, e = rp[r], rp[r + 1]
            x = b + np.searchsorted(ci[b:e], c)
            out[t] = x if x < e and ci[x] == c else -1
        return torch.from_numpy(out)

    def assemble_rows(self, local, pat, fmt, cell_begin, cell_end, rows, accumulate, values):
        if rows is None or rows.numel() == 0:
            return values
        n_loc = pat.n_local
        rp = pat.row_ptr.numpy()
        ci = pat.col_idx.numpy()
        ip = pat.inc_ptr.numpy()
        inc = pat.inc.numpy()
        dt = np.float32 if fmt == 2 else np.float64
        loc = local.numpy()
        vals = values.numpy()  # shares memory with the torch tensor
        for r in rows.numpy().tolist():
            b, e = rp[r], rp[r + 1]
            if not accumulate:
                vals[b:e] = dt(-0.0)
            for pk in inc[ip[r]:ip[r + 1]]:
                c, i = divmod(int(pk), n_loc)
                if c < cell_begin or c >= cell_end:
                    continue
                for j in range(n_loc):
                    x = b + np.searchsorted(ci[b:e], pat.col_dofs[c, j])
                    vals[x] = dt(vals[x] + dt(loc[c - cell_begin, i, j]))
        return values
