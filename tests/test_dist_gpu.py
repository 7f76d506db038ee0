"""The partitioned path end to end on the GPU: R ranks, one process each, sharing
the one B200 of the test box (gloo: buffers staged through host memory -- the kernels, exchanges
and numbers are those of the NCCL run).  Each rank checks its tags, map, coarse rows (owned and
halo columns) and the distributed PCG against the oracle run on the global mesh with
segments = rank bounds (reading R24)."""
import os

import pytest
import torch.multiprocessing as mp

from test_dist_host import free_port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,R,thr,kind", [(10, 2, 32, "twist"), (8, 3, 32, "random"), (8, 2, 5, "random"),
                                          (6, 4, 10 ** 9, "random"), (14, 2, 32, "twist"),
                                          (6, 3, 32, "c4"), (6, 2, 5, "c4"), (12, 3, 32, "thin"),
                                          (12, 4, 5, "thin")])
def test_distributed_step_matches_segmented_oracle(gpu, tmp_path, n, R, thr, kind):
    from dist_worker import gpu_worker
    mp.start_processes(gpu_worker, args=(R, free_port(), str(tmp_path), n, thr, kind), nprocs=R,
                       start_method="spawn")
    errs = [f.read_text() for f in tmp_path.glob("err*")]
    assert not errs, errs
    assert sorted(os.listdir(tmp_path)) == [f"ok{r}" for r in range(R)]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("R", [2, 3])
def test_singular_block_on_one_rank_stops_every_rank(gpu, tmp_path, R):
    """the singular flag travels with the setup sums (red[3]), so every rank
    returns ESINGULAR instead of the other ranks waiting in the next all-reduce."""
    from dist_worker import singular_worker
    mp.start_processes(singular_worker, args=(R, free_port(), str(tmp_path)), nprocs=R, start_method="spawn")
    errs = [f.read_text() for f in tmp_path.glob("err*")]
    assert not errs, errs
    assert [(tmp_path / f"ok{r}").read_text() for r in range(R)] == ["AGIPC_ESINGULAR"] * R
