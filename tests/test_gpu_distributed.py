"""The partitioned z-slab assembly with the CUDA backend: 2 and 3 ranks on gloo,
all on cuda:0 (this pool has one GPU per box; the ranks do not wait on each other's kernels,
only on the host-staged P2P exchange). Every owned row of every rank -- dof numbering,
columns, values -- must equal the single-process reference assembly (oracle, pinned to the
compiled reference) bit for bit; the path exercised is the product's: per-rank dof maps,
the layer table, local-row / global-column CSR + scatter plan, rows-restricted deterministic
assembly (assemble_seg_rows_kernel) continuing the received partial sums."""
import pytest

pytestmark = pytest.mark.gpu

from test_distributed_cpu import check_against_reference, run_world  # noqa: E402


@pytest.mark.parametrize("world,dims,p,fmt", [(2, (3, 2, 4), 2, 2), (2, (2, 2, 4), 3, 3), (3, (3, 3, 6), 2, 3),
                                              (3, (2, 2, 6), 1, 2)])
def test_partitioned_cuda_assembly_matches_reference(oracle, world, dims, p, fmt):
    res = run_world(world, p, dims, fmt, use_cuda=True)
    check_against_reference(oracle, res, p, dims, fmt)
