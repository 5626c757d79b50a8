"""World-size-2 and -3 gloo runs of the partitioned z-slab assembly on CPU with the
numpy backend (tests/cpu_backend.py): the per-rank first-encounter numbering made global by one
all-gather must equal the reference dof map, every owned row must equal the single-process
reference assembly bitwise (columns and values), every row must be owned by exactly one rank,
and each rank holds only its slab plus one halo layer."""
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

from dist_worker import worker
from oracle_lib import nphi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def run_world(world, p, dims, fmt, use_cuda):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, p, dims, fmt, use_cuda, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for r in results:
        assert r[1] != "error", r[2]
    for pr in procs:
        assert pr.exitcode == 0
    return sorted(results, key=lambda t: t[0])


def check_against_reference(oracle, results, p, dims, fmt):
    nx, ny, nz = dims
    verts, cells = oracle.structured_tet_mesh(nx, ny, nz, 1.0, 0.15, 17)
    cd, nd, _ = oracle.build_dofmap(p, verts, cells)
    rng = np.random.default_rng(123)
    all_loc = rng.uniform(-1, 1, size=(cells.shape[0], nphi(p), nphi(p))).astype(np.float32)
    rows, cols, vals, _ = oracle.assemble_matrix(cd, nd, all_loc.astype(np.float64), fmt)
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=nd))])
    seen = np.zeros(nd, dtype=int)
    for rank, n_dofs, owned, nnz_local, n_cells_local in results:
        assert n_dofs == nd
        for g, (c, v) in owned.items():
            seen[g] += 1
            assert np.array_equal(c, cols[rp[g]:rp[g + 1]]), (rank, g)
            assert np.array_equal(v.view(np.uint64), vals[rp[g]:rp[g + 1]].view(np.uint64)), (rank, g)
        # partitioned, not replicated: slab + one halo layer
        assert n_cells_local <= cells.shape[0] // len(results) + 2 * 6 * nx * ny
    assert np.all(seen == 1)


@pytest.mark.parametrize("world,dims,p,fmt", [(2, (2, 2, 4), 2, 2), (2, (2, 1, 4), 1, 3), (3, (2, 2, 6), 2, 3)])
def test_partitioned_slab_assembly_matches_reference(oracle, world, dims, p, fmt):
    res = run_world(world, p, dims, fmt, use_cuda=False)
    check_against_reference(oracle, res, p, dims, fmt)
