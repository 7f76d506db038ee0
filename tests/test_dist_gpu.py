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
                                          (6, 3, 32, "c4"), (6, 2, 5, "c4")])
def test_distributed_step_matches_segmented_oracle(gpu, tmp_path, n, R, thr, kind):
    from dist_worker import gpu_worker
    mp.start_processes(gpu_worker, args=(R, free_port(), str(tmp_path), n, thr, kind), nprocs=R,
                       start_method="spawn")
    errs = [f.read_text() for f in tmp_path.glob("err*")]
    assert not errs, errs
    assert sorted(os.listdir(tmp_path)) == [f"ok{r}" for r in range(R)]
