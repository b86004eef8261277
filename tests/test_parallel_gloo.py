"""Multi-process (gloo, world_size 2, CPU) tests of the view-parallel driver: partition,
flat-buffer layout, bucketed all-reduce, and equivalence of the P-rank step with a
single-process accumulation over all views (SURVEY.md §8(e) correctness criterion)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_01467_b200.parallel import FlatGrads, view_parallel_step, views_for_rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_views_for_rank_partition():
    for n_views in (1, 7, 200):
        for ws in (1, 2, 3, 8):
            owned = sorted(v for r in range(ws) for v in views_for_rank(n_views, ws, r))
            assert owned == list(range(n_views))
    with pytest.raises(ValueError):
        views_for_rank(10, 2, 2)


def test_flat_grads_layout():
    g = FlatGrads.allocate(5, 16, "cpu")
    assert g.flat.numel() == 59 * 5
    g.sh[4, 3, 2] = 7.0   # Gaussian 4, coefficient 3, channel 2 of sh[n][K][3]
    g.means[1, 0] = 3.0   # Gaussian 1, x of means[n][3]
    assert g.flat[1 * 3 + 0].item() == 3.0
    off = (3 + 3 + 4 + 1) * 5 + 4 * 48 + 3 * 3 + 2
    assert g.flat[off].item() == 7.0
    g.zero_()
    assert g.flat.abs().sum().item() == 0


def _fake_view_grads(camera_id, n):
    """Deterministic stand-in for one view's fwd+bwd (the CUDA path is not on CPU)."""
    rng = np.random.default_rng(1000 + camera_id)
    return torch.as_tensor(rng.normal(size=59 * n).astype(np.float32))


def _worker(rank, ws, port, n, n_views, bucket, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    grads = FlatGrads.allocate(n, 16, "cpu")

    def render_view(cam, gr):
        gr.flat += _fake_view_grads(cam, n)

    cams = list(range(n_views))
    done = view_parallel_step(render_view, cams, grads, views_for_rank(n_views, ws, rank), bucket_bytes=bucket)
    out[rank] = (done, grads.flat.clone())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("bucket", [0, 1000])
def test_two_rank_step_equals_single_process_sum(bucket):
    n, n_views, ws = 37, 9, 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(ws, port, n, n_views, bucket, out), nprocs=ws, join=True)
    ref = sum(_fake_view_grads(v, n).double() for v in range(n_views))
    assert out[0][0] + out[1][0] == n_views
    for r in range(ws):
        # only the summation order differs from the single-process accumulation
        assert torch.allclose(out[r][1].double(), ref, rtol=1e-6, atol=1e-5)
    # replicas are bitwise identical after the all-reduce
    assert torch.equal(out[0][1], out[1][1])
