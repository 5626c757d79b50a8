"""Multi-GPU assembly over z-slabs, one process per GPU.

Cells of a structured tet mesh are z-major (mesh.cpp:102-112), so a contiguous range of
hex layers is a contiguous range of cells. Rank r owns cell range [cb, ce) and every
global row (dof) whose highest incident cell lies in its range. A row whose incident
cells straddle the slab boundary (the interface plane) is started by rank r - 1, which
sums its own contributions in ascending cell order and sends those prefix partial sums to
rank r; rank r continues the same sequential sum with its cells. The result is therefore
the reference's single ascending-cell sum (assembly.cpp:50-67) bit for bit, on any number
of ranks. The only collective on the data path is that one neighbour exchange
(send to r + 1, receive from r - 1), issued as one batched P2P group (NCCL on GPUs, gloo
in the CPU tests).

The dof numbering itself is replicated: each rank builds the global dof map, pattern and
incidence on its own device (integer work, milliseconds at 96^3), which keeps the
first-encounter numbering global without an extra collective.

`backend` supplies build_dofmap / csr_pattern / assemble_matrix with the signatures of
paper_2410_12614_b200.assembly (the CUDA product); tests pass a CPU stand-in to exercise
this host logic under gloo.
"""
from __future__ import annotations

from dataclasses import dataclass


def slab_cell_range(rank: int, world: int, n_layers: int, cells_per_layer: int):
    """Contiguous hex layers per rank (remainder spread over the first ranks)."""
    base, extra = divmod(n_layers, world)
    l0 = rank * base + min(rank, extra)
    l1 = l0 + base + (1 if rank < extra else 0)
    return l0 * cells_per_layer, l1 * cells_per_layer


@dataclass
class SlabPlan:
    rank: int
    world: int
    cell_begin: int
    cell_end: int
    owned_rows: "object"   # int32 rows this rank finalises
    recv_rows: "object"    # int32 owned rows that continue rank-1's partial sums
    fresh_rows: "object"   # int32 owned rows that start here
    send_rows: "object"    # int32 rows started here and finished by rank+1
    recv_index: "object"   # int64 value positions of recv_rows (packed order)
    send_index: "object"   # int64 value positions of send_rows (packed order)


def _segments(row_ptr, rows):
    """Concatenated CSR value positions of `rows` (in row order)."""
    import torch
    rows = rows.to(torch.int64)
    starts = row_ptr[rows]
    lens = row_ptr[rows + 1] - starts
    if rows.numel() == 0:
        return torch.empty(0, dtype=torch.int64, device=row_ptr.device)
    offs = torch.repeat_interleave(starts - torch.cumsum(lens, 0) + lens, lens)
    return offs + torch.arange(int(lens.sum()), device=row_ptr.device, dtype=torch.int64)


def plan_slabs(dm, pat, rank: int, world: int, cell_begin: int, cell_end: int) -> SlabPlan:
    import torch
    n_loc = dm.n_local
    inc_ptr, inc = pat.inc_ptr, pat.inc
    first_cell = inc[inc_ptr[:-1]] // n_loc
    last_cell = inc[inc_ptr[1:] - 1] // n_loc
    owned = (last_cell >= cell_begin) & (last_cell < cell_end)
    starts_here = (first_cell >= cell_begin) & (first_cell < cell_end)
    rows = torch.arange(dm.n_dofs, device=inc.device, dtype=torch.int32)
    recv = owned & (first_cell < cell_begin)
    send = starts_here & (last_cell >= cell_end)
    owned_rows = rows[owned]
    recv_rows = rows[recv]
    fresh_rows = rows[owned & ~recv]
    send_rows = rows[send]
    return SlabPlan(rank, world, cell_begin, cell_end, owned_rows, recv_rows, fresh_rows, send_rows,
                    _segments(pat.row_ptr, recv_rows), _segments(pat.row_ptr, send_rows))


def check_adjacent(dm, pat, ranges) -> None:
    """Every row's incident cells must lie in at most two adjacent slabs."""
    import torch
    n_loc = dm.n_local
    bounds = torch.tensor([r[1] for r in ranges], device=pat.inc.device)
    first = torch.bucketize(pat.inc[pat.inc_ptr[:-1]] // n_loc, bounds, right=True)
    last = torch.bucketize(pat.inc[pat.inc_ptr[1:] - 1] // n_loc, bounds, right=True)
    if int((last - first).max()) > 1:
        raise ValueError("slabs thinner than one cell layer: a row spans more than two ranks")


def assemble_slab(backend, local, dm, pat, plan: SlabPlan, fmt: int, group=None, values=None):
    """Deterministic assembly of this rank's owned rows. `local` holds the local matrices of
    cells [plan.cell_begin, plan.cell_end). Returns the full-length values tensor (pass
    `values` to reuse one), valid on plan.owned_rows' segments."""
    import torch
    import torch.distributed as dist
    dtype = torch.float32 if fmt == 2 else torch.float64
    if values is None:
        values = torch.empty(pat.nnz, dtype=dtype, device=local.device)
    cb, ce = plan.cell_begin, plan.cell_end
    # 1. prefix partial sums of the rows the next rank finishes (our cells only)
    if plan.send_rows.numel():
        backend.assemble_matrix(local, dm, pat, fmt, 1, cb, ce, rows=plan.send_rows,
                                accumulate=False, values=values)
    send_buf = values[plan.send_index].contiguous()
    recv_buf = torch.empty(int(plan.recv_index.numel()), dtype=dtype, device=local.device)
    # 2. the single neighbour exchange (r -> r+1), batched (NCCL: device buffers over
    #    NVLink; gloo: staged through host memory)
    if plan.world > 1:
        host = dist.get_backend(group) == "gloo" and send_buf.is_cuda
        sb = send_buf.cpu() if host else send_buf
        rb = torch.empty(recv_buf.shape, dtype=dtype) if host else recv_buf
        ops = []
        if plan.rank + 1 < plan.world:
            ops.append(dist.P2POp(dist.isend, sb, plan.rank + 1, group))
        if plan.rank > 0:
            ops.append(dist.P2POp(dist.irecv, rb, plan.rank - 1, group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if host:
            recv_buf.copy_(rb)
    # 3. continue the received sums, start the fresh rows
    if plan.recv_rows.numel():
        values[plan.recv_index] = recv_buf
        backend.assemble_matrix(local, dm, pat, fmt, 1, cb, ce, rows=plan.recv_rows,
                                accumulate=True, values=values)
    if plan.fresh_rows.numel():
        backend.assemble_matrix(local, dm, pat, fmt, 1, cb, ce, rows=plan.fresh_rows,
                                accumulate=False, values=values)
    return values
