"""View-parallel multi-GPU driver.

Views are independent units: rank r of P takes views {v : v mod P = r}; the Gaussians are
replicated on every rank. Each rank accumulates (+=) the gradients of its views into ONE
flat fp32 buffer (59·N floats at SH degree 3, laid out as the rd_grads arrays), then the
only exchange step of the path runs: an all-reduce (sum) of that buffer — NCCL over
NVLink/NVSwitch on GPUs, gloo on CPU for the tests. All-reduce results are bitwise identical
on every rank, so replicas that apply the same optimizer step stay identical.

Host logic only; every device computation is a C-ABI call of librade.so (via `rade`).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def views_for_rank(n_views: int, world_size: int, rank: int) -> list:
    """Round-robin view partition: every view is owned by exactly one rank."""
    if world_size <= 0 or not 0 <= rank < world_size:
        raise ValueError("bad world_size / rank")
    return [v for v in range(n_views) if v % world_size == rank]


@dataclass
class FlatGrads:
    """One contiguous fp32 buffer and the five rd_grads views into it."""
    flat: torch.Tensor
    means: torch.Tensor
    scales: torch.Tensor
    rotations: torch.Tensor
    opacities: torch.Tensor
    sh: torch.Tensor

    @staticmethod
    def allocate(n: int, sh_coeffs: int = 16, device="cuda") -> "FlatGrads":
        shapes = ((n, 3), (n, 3), (n, 4), (n,), (n, sh_coeffs, 3))
        total = sum(int(torch.Size(s).numel()) for s in shapes)
        flat = torch.zeros(total, dtype=torch.float32, device=device)
        parts, o = [], 0
        for s in shapes:
            c = int(torch.Size(s).numel())
            parts.append(flat[o:o + c].view(*s))
            o += c
        return FlatGrads(flat, *parts)

    def zero_(self):
        self.flat.zero_()
        return self

    def zero_geometry_(self):
        """Zeroes all but the SH gradients (the segments before them): the step's SH rows are then
        SET by rd_preprocess_bwd_views_ex(..., RD_K5_SET_SH)."""
        self.flat[: self.flat.numel() - self.sh.numel()].zero_()
        return self

    def as_gaussians(self):
        from .rade import Gaussians
        return Gaussians(self.means, self.scales, self.rotations, self.opacities, self.sh)

    def allreduce(self, group=None, bucket_bytes: int = 0, async_op: bool = False):
        """Sum over ranks in place. bucket_bytes > 0 splits the buffer into buckets issued
        back to back (lets the collective start on early buckets); 0 = one call."""
        if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
            return []
        if bucket_bytes <= 0:
            h = dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
            return [h] if async_op else []
        step = max(1, bucket_bytes // 4)
        handles = []
        for o in range(0, self.flat.numel(), step):
            handles.append(dist.all_reduce(self.flat[o:o + step], op=dist.ReduceOp.SUM, group=group,
                                           async_op=True))
        if async_op:
            return handles
        for h in handles:
            h.wait()
        return []


def view_parallel_step(render_view, cameras, grads: FlatGrads, views, group=None, bucket_bytes: int = 0):
    """One data-parallel step: this rank runs `render_view(camera, grads)` (forward, loss,
    backward accumulating into grads) for each of its views, then all-reduces the grads.
    Returns the number of views this rank processed."""
    grads.zero_()
    for v in views:
        render_view(cameras[v], grads)
    grads.allreduce(group, bucket_bytes)
    return len(views)
