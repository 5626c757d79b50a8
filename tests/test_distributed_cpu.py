"""World-size-2 and -3 gloo runs of the z-slab assembly host logic on CPU:
every rank's owned rows must equal the single-process reference assembly bitwise, and
every row must be owned by exactly one rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2410_12614_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, nz, fmt, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from cpu_backend import CpuBackend
    from oracle_lib import Oracle, nphi
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()
    nx, ny = 3, 2
    verts, cells = O.structured_tet_mesh(nx, ny, nz, 1.0, 0.15, 17)
    be = CpuBackend()
    dm, pat = be.build(p, verts, cells)
    cpl = 6 * nx * ny
    ranges = [D.slab_cell_range(r, world, nz, cpl) for r in range(world)]
    D.check_adjacent(dm, pat, ranges)
    cb, ce = ranges[rank]
    rng = np.random.default_rng(123)
    all_loc = rng.uniform(-1, 1, size=(cells.shape[0], nphi(p), nphi(p))).astype(np.float32)
    local = torch.from_numpy(all_loc[cb:ce].copy())
    plan = D.plan_slabs(dm, pat, rank, world, cb, ce)
    vals = D.assemble_slab(be, local, dm, pat, plan, fmt)
    out_q.put((rank, plan.owned_rows.numpy().copy(), vals.numpy().copy(),
               pat.row_ptr.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nz,p,fmt", [(2, 4, 2, 2), (2, 2, 1, 3), (3, 6, 2, 3)])
def test_slab_assembly_matches_reference(oracle, world, nz, p, fmt):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, nz, fmt, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    verts, cells = oracle.structured_tet_mesh(3, 2, nz, 1.0, 0.15, 17)
    cd, nd, _ = oracle.build_dofmap(p, verts, cells)
    from oracle_lib import nphi
    rng = np.random.default_rng(123)
    all_loc = rng.uniform(-1, 1, size=(cells.shape[0], nphi(p), nphi(p))).astype(np.float32)
    _, _, ref, _ = oracle.assemble_matrix(cd, nd, all_loc.astype(np.float64), fmt)
    seen = np.zeros(nd, dtype=int)
    for rank, owned, vals, rp in sorted(results, key=lambda t: t[0]):
        seen[owned] += 1
        for r in owned:
            got = vals[rp[r]:rp[r + 1]].astype(np.float64)
            assert np.array_equal(got.view(np.uint64), ref[rp[r]:rp[r + 1]].view(np.uint64)), (rank, r)
    assert np.all(seen == 1)
