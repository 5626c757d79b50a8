"""Multi-GPU assembly over z-slabs, one process per GPU, partitioned.

Cells of a structured tet mesh are z-major (mesh.cpp:102-112), so a contiguous range of hex
layers is a contiguous range of cells. Rank r owns the cells [cb, ce) and holds one extra
layer below them (the halo, [cb - cells_per_layer, cb), rank 0 none) -- nothing else of the
mesh's numbering, pattern or values: per-rank memory shrinks as 1/P.

Numbering (first-encounter, mesh.cpp:247-293, made global without replicating it):
  * the rank numbers the nodes of halo + own cells in first-encounter order; since the halo
    comes first, the halo's nodes take local ids 0 .. n_halo - 1, exactly the first-encounter
    numbering of that single layer, which the lower rank (who owns the layer) computes the
    same way;
  * the nodes first met in the own cells are this rank's new dofs (n_new); an all-gather of
    n_new gives every rank its offset (exclusive scan), so new node ids are
    offset + local - n_halo -- exactly their global first-encounter ids, because no lower cell
    contains them;
  * the halo nodes' global ids arrive from the lower rank as a table (layer-local id -> global
    id) over its top layer; with at least two layers per rank that layer holds only the lower
    rank's new dofs, so no rank waits on a chain of exchanges.

Rows: local ids (halo + own nodes); columns: global ids, so every row's columns sort exactly
as the reference COO's (assembly.cpp:67-86). A row is owned by the rank of its highest incident
cell: the top-plane rows of a rank (shared with the next rank's cells) are started here and
finished by rank r + 1; the bottom-plane rows continue the lower rank's sums.

Assembly (deterministic, the reference's ascending-cell sequential sum, assembly.cpp:50-67):
the rank sums its own cells' contributions to the rows the next rank finishes and sends those
prefix partial sums up (one batched P2P exchange, NCCL over NVLink on GPUs, gloo in the CPU
tests); it seeds its bottom-plane rows with the received sums and continues them with its own
cells. Every owned row is therefore the reference's sum bit for bit on any number of ranks.

`backend` supplies the device operations (assembly.CudaPartitionBackend on GPUs; the tests
pass a CPU restatement to run this host logic under gloo without a GPU).
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
class Partition:
    rank: int
    world: int
    cell_begin: int        # own cells [cell_begin, cell_end) (global cell ids)
    cell_end: int
    halo_begin: int        # first cell of the halo layer (== cell_begin on rank 0)
    n_halo: int            # nodes of the halo layer: local ids 0 .. n_halo - 1
    n_local: int           # local rows (halo + own nodes)
    offset: int            # global id of this rank's first new node
    n_dofs: int            # global number of dofs
    cell_dofs: "object"    # (ce - hb, n_loc) local ids
    cell_dofs_global: "object"  # (ce - hb, n_loc) global ids
    row_global: "object"   # (n_local,) global id of every local row
    pat: "object"          # local-row / global-column CSR with its scatter plan
    owned_rows: "object"   # int32 local rows this rank finalises (recv + fresh)
    recv_rows: "object"    # owned rows that continue the lower rank's partial sums
    fresh_rows: "object"   # owned rows that start here
    send_rows: "object"    # rows started here and finished by the next rank (layer-id order)
    send_pos: "object"     # int64 CSR positions of the send rows' entries (concatenated)
    recv_pos: "object"     # int64 CSR positions the received entries go to
    recv_seg: "object"     # int64 every CSR position of the recv rows

    @property
    def own_local_cells(self):
        """Own cells in the rank's local cell indexing (halo first)."""
        return self.cell_begin - self.halo_begin, self.cell_end - self.halo_begin


def _host_comm(group, t):
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo" and t.is_cuda


def _exchange(sends, recvs, group):
    """One batched P2P group: sends = [(tensor, peer)], recvs = [(tensor, peer)] (device
    tensors; staged through host memory for gloo)."""
    import torch.distributed as dist
    ops, back = [], []
    for t, peer in sends:
        ops.append(dist.P2POp(dist.isend, t.cpu() if _host_comm(group, t) else t, peer, group))
    for t, peer in recvs:
        if _host_comm(group, t):
            h = t.new_empty(t.shape, device="cpu")
            back.append((h, t))
            ops.append(dist.P2POp(dist.irecv, h, peer, group))
        else:
            ops.append(dist.P2POp(dist.irecv, t, peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for h, t in back:
        t.copy_(h)


def _segments(row_ptr, rows):
    """Concatenated CSR value positions of `rows` (in the order given)."""
    import torch
    rows = rows.to(torch.int64)
    if rows.numel() == 0:
        return torch.empty(0, dtype=torch.int64, device=row_ptr.device)
    starts = row_ptr[rows]
    lens = row_ptr[rows + 1] - starts
    offs = torch.repeat_interleave(starts - torch.cumsum(lens, 0) + lens, lens)
    return offs + torch.arange(int(lens.sum()), device=row_ptr.device, dtype=torch.int64)


def build_partition(backend, p: int, cells, n_verts: int, rank: int, world: int, n_layers: int,
                    cells_per_layer: int, group=None) -> Partition:
    """Per-rank dof numbering, pattern and exchange plan of the z-slab partition. `cells` is
    the mesh's (n_cells, 4) int32 cell table on the rank's device (only the rank's slab and
    its halo layer are read)."""
    import torch
    import torch.distributed as dist
    from . import ConfigError
    if world > 1 and n_layers < 2 * world:
        raise ConfigError("z-slab assembly needs at least two hex layers per rank")
    dev = cells.device
    cb, ce = slab_cell_range(rank, world, n_layers, cells_per_layer)
    hb = cb - cells_per_layer if rank > 0 else cb
    # 1. local first-encounter numbering of halo + own cells; the halo layer alone
    cd_loc, n_ext = backend.dofmap(p, cells[hb:ce].contiguous(), n_verts)
    n_halo = backend.dofmap(p, cells[hb:cb].contiguous(), n_verts)[1] if rank > 0 else 0
    n_new = n_ext - n_halo
    # 2. global offsets (all-gather of the new-dof counts)
    if world > 1:
        cnt = torch.tensor([n_new], dtype=torch.int64, device="cpu" if dist.get_backend(group) == "gloo" else dev)
        allc = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(allc, cnt, group=group)
        counts = [int(c.item()) for c in allc]
    else:
        counts = [n_new]
    offset = sum(counts[:rank])
    n_dofs = sum(counts)
    n_loc = int(cd_loc.shape[1])
    # 3. the top layer's table (layer-local id -> global id) goes up, the halo's comes down
    top_cd = None
    send_table = None
    if rank + 1 < world:
        top0 = ce - cells_per_layer
        top_cd, n_top = backend.dofmap(p, cells[top0:ce].contiguous(), n_verts)
        top_glob = cd_loc[top0 - hb:ce - hb].reshape(-1) - n_halo + offset  # new dofs only
        send_table = backend.table(top_cd.reshape(-1), top_glob.to(torch.int32), n_top)
    recv_table = torch.zeros(max(n_halo, 1), dtype=torch.int32, device=dev)[:n_halo]
    if world > 1:
        _exchange([(send_table, rank + 1)] if send_table is not None else [],
                  [(recv_table, rank - 1)] if rank > 0 else [], group)
    cd_glob = backend.globalize(cd_loc.reshape(-1), recv_table, n_halo, offset).reshape(cd_loc.shape)
    row_global = torch.empty(n_ext, dtype=torch.int32, device=dev)
    row_global[cd_loc.reshape(-1).to(torch.int64)] = cd_glob.reshape(-1)
    # 4. local-row / global-column pattern and plan over halo + own cells
    pat = backend.pattern(cd_loc, cd_glob, n_ext)
    first_cell = pat.inc[pat.inc_ptr[:-1]] // n_loc
    last_cell = pat.inc[pat.inc_ptr[1:] - 1] // n_loc
    own0 = cb - hb
    touched = last_cell >= own0
    recv = touched & (first_cell < own0)
    rows = torch.arange(n_ext, device=dev, dtype=torch.int32)
    recv_rows = rows[recv]  # local ids < n_halo == the lower rank's top-layer ids
    # 5. which of our top-layer rows does the next rank finish? (it sends its recv rows as
    #    top-layer ids); and their columns go up once, so the next rank can place our sums
    send_rows = torch.empty(0, dtype=torch.int32, device=dev)
    send_pos = torch.empty(0, dtype=torch.int64, device=dev)
    recv_pos = torch.empty(0, dtype=torch.int64, device=dev)
    if world > 1:
        n_recv_rows = torch.tensor([int(recv_rows.numel())], dtype=torch.int64, device=dev)
        n_send_rows = torch.zeros(1, dtype=torch.int64, device=dev)
        _exchange([(n_recv_rows, rank - 1)] if rank > 0 else [],
                  [(n_send_rows, rank + 1)] if rank + 1 < world else [], group)
        send_ids = torch.empty(int(n_send_rows.item()), dtype=torch.int32, device=dev)
        _exchange([(recv_rows.contiguous(), rank - 1)] if rank > 0 else [],
                  [(send_ids, rank + 1)] if rank + 1 < world else [], group)
        if rank + 1 < world:
            top0 = ce - cells_per_layer
            layer_to_local = backend.table(top_cd.reshape(-1), cd_loc[top0 - hb:ce - hb].reshape(-1), n_top)
            send_rows = layer_to_local[send_ids.to(torch.int64)]
            send_pos = _segments(pat.row_ptr, send_rows)
        # the columns of the send rows (global ids), with per-row counts
        send_lens = (pat.row_ptr[send_rows.to(torch.int64) + 1] - pat.row_ptr[send_rows.to(torch.int64)]) \
            if send_rows.numel() else torch.empty(0, dtype=torch.int64, device=dev)
        recv_lens = torch.empty(int(recv_rows.numel()), dtype=torch.int64, device=dev)
        _exchange([(send_lens.contiguous(), rank + 1)] if rank + 1 < world else [],
                  [(recv_lens, rank - 1)] if rank > 0 else [], group)
        send_cols = pat.col_idx[send_pos] if send_pos.numel() else torch.empty(0, dtype=torch.int32, device=dev)
        recv_cols = torch.empty(int(recv_lens.sum().item()) if recv_lens.numel() else 0, dtype=torch.int32, device=dev)
        _exchange([(send_cols.contiguous(), rank + 1)] if rank + 1 < world else [],
                  [(recv_cols, rank - 1)] if rank > 0 else [], group)
        if recv_rows.numel():
            rr = torch.repeat_interleave(recv_rows, recv_lens)
            recv_pos = backend.find(pat, rr.contiguous(), recv_cols)
            if bool((recv_pos < 0).any()):
                raise RuntimeError("interface columns missing from the receiving rank's pattern")
    send_mask = torch.zeros(n_ext, dtype=torch.bool, device=dev)
    if send_rows.numel():
        send_mask[send_rows.to(torch.int64)] = True
    fresh = touched & ~recv & ~send_mask
    fresh_rows = rows[fresh]
    owned_rows = rows[touched & ~send_mask]
    return Partition(rank, world, cb, ce, hb, n_halo, n_ext, offset, n_dofs, cd_loc, cd_glob,
                     row_global, pat, owned_rows, recv_rows, fresh_rows, send_rows, send_pos,
                     recv_pos, _segments(pat.row_ptr, recv_rows))


def assemble_partition(backend, part: Partition, local, fmt: int, group=None, values=None):
    """Deterministic assembly of the rank's owned rows. `local` holds the local matrices of the
    own cells [cell_begin, cell_end). Returns the rank's local CSR values (valid on the owned
    rows' segments; row i is global row part.row_global[i])."""
    import torch
    dtype = torch.float32 if fmt == 2 else torch.float64
    if values is None:
        values = torch.empty(part.pat.nnz, dtype=dtype, device=local.device)
    c0, c1 = part.own_local_cells
    # 1. prefix partial sums of the rows the next rank finishes (own cells only)
    backend.assemble_rows(local, part.pat, fmt, c0, c1, part.send_rows, False, values)
    send_buf = values[part.send_pos].contiguous()
    recv_buf = torch.empty(int(part.recv_pos.numel()), dtype=dtype, device=local.device)
    # 2. the single neighbour exchange (r -> r + 1)
    if part.world > 1:
        _exchange([(send_buf, part.rank + 1)] if part.rank + 1 < part.world else [],
                  [(recv_buf, part.rank - 1)] if part.rank > 0 else [], group)
    # 3. seed the bottom-plane rows with the received sums (entries the lower rank did not
    #    touch start empty: -0.0 leaves the first own contribution exact) and continue them
    if part.recv_rows.numel():
        values[part.recv_seg] = -0.0
        values[part.recv_pos] = recv_buf
        backend.assemble_rows(local, part.pat, fmt, c0, c1, part.recv_rows, True, values)
    backend.assemble_rows(local, part.pat, fmt, c0, c1, part.fresh_rows, False, values)
    return values
