"""Worker of the multi-rank z-slab assembly tests (test_distributed_cpu.py on gloo/CPU with the
numpy backend, test_gpu_distributed.py on gloo with the CUDA backend, ranks sharing cuda:0).
TEST INFRASTRUCTURE."""
import os
import sys

import numpy as np


def worker(rank, world, port, p, dims, fmt, use_cuda, out_q):
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from oracle_lib import Oracle, nphi
    from paper_2410_12614_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = dims
        verts, cells = Oracle().structured_tet_mesh(nx, ny, nz, 1.0, 0.15, 17)
        if use_cuda:
            from paper_2410_12614_b200 import assembly as am
            backend = am.CudaPartitionBackend()
            cells_t = torch.from_numpy(cells).cuda()
        else:
            from cpu_backend import CpuPartitionBackend
            backend = CpuPartitionBackend(verts)
            cells_t = torch.from_numpy(cells)
        part = D.build_partition(backend, p, cells_t, verts.shape[0], rank, world, nz, 6 * nx * ny)
        rng = np.random.default_rng(123)
        all_loc = rng.uniform(-1, 1, size=(cells.shape[0], nphi(p), nphi(p))).astype(np.float32)
        local = torch.from_numpy(all_loc[part.cell_begin:part.cell_end].copy())
        if use_cuda:
            local = local.cuda()
        vals = D.assemble_partition(backend, part, local, fmt)
        rp = part.pat.row_ptr.cpu().numpy()
        ci = part.pat.col_idx.cpu().numpy()
        vv = vals.double().cpu().numpy()
        rg = part.row_global.cpu().numpy()
        rows = {}
        for r in part.owned_rows.cpu().numpy().tolist():
            rows[int(rg[r])] = (ci[rp[r]:rp[r + 1]].copy(), vv[rp[r]:rp[r + 1]].copy())
        out_q.put((rank, part.n_dofs, rows, int(part.pat.nnz), int(part.cell_end - part.halo_begin)))
        dist.barrier()
    except Exception as e:  # report instead of hanging the parent
        import traceback
        out_q.put((rank, "error", traceback.format_exc(), 0, 0))
    finally:
        dist.destroy_process_group()
