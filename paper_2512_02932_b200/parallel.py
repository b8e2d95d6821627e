"""Camera-sharded multi-view training step.

Views of a replicated scene are independent, so one process per GPU renders
and back-propagates its own shard of the cameras and the per-Gaussian flat
gradient buffer is summed across ranks with one all-reduce per step (NCCL
over NVLink on a B200 box; gloo in the CPU tests).  The buffer is the C ABI's
field-major ParamGrads layout (center | log_scale | rotation | opacity | sh),
one contiguous tensor, so the reduction is a single collective.

The render / backward / loss callables are injectable: the product path uses
the CUDA rasterizer (``default_view_grad``); the CPU tests drive the same
sharding and reduction logic with the oracle.
"""

import math

__all__ = ["shard_views", "allreduce_grads", "replica_checksum", "MultiViewStep",
           "default_view_grad"]


def shard_views(n_views, rank, world):
    """Contiguous, balanced block of view indices for ``rank`` (every view
    exactly once across ranks; sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world %r/%r" % (rank, world))
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def allreduce_grads(buf, group=None):
    """Sum the flat gradient buffer over all ranks (no-op for world size 1)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def replica_checksum(tensors, group=None):
    """True iff every rank holds bit-identical replicas (cheap sum-of-bits
    fingerprint, all-reduced MIN vs MAX).  Exchange passes are deterministic,
    so replicas never need a parameter broadcast -- this asserts it."""
    import torch
    import torch.distributed as dist
    acc = 0
    for t in tensors:
        b = t.detach().contiguous().view(torch.uint8).to(torch.int64)
        acc = acc + int(b.sum().item()) * 1000003 + b.numel()
    if not (dist.is_available() and dist.is_initialized()):
        return True
    dev = tensors[0].device if tensors[0].is_cuda else "cpu"
    lo = torch.tensor([acc], dtype=torch.int64, device=dev)
    hi = lo.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return int(lo.item()) == int(hi.item())


def default_view_grad(scene, camera, settings, loss_grad, out_buf):
    """Render one view on the GPU, back-propagate ``loss_grad(color)`` and
    add the field-major gradient into ``out_buf`` (float32, n*P)."""
    from . import grad, raster
    imgs, frame = raster.rasterize(scene, camera, settings)
    pg = loss_grad(imgs["color"])
    if pg.dim() == 3:
        pg = pg.unsqueeze(0)
    g, _ = grad.backward_device(frame, pg.float().contiguous())
    out_buf += g.sum(dim=0)
    return imgs


class MultiViewStep:
    """One data-parallel step over a batch of views.

    ``view_grad(scene, camera, settings, loss_grad, out_buf)`` accumulates one
    view's gradient into ``out_buf``; ``loss_grad(view_index, color)`` returns
    the upstream pixel gradient of that view's loss.
    """

    def __init__(self, scene, cameras, settings, n_params, device=None, group=None,
                 view_grad=None):
        import torch
        import torch.distributed as dist
        self.scene = scene
        self.cameras = list(cameras)
        self.settings = settings
        self.group = group
        self.view_grad = view_grad or default_view_grad
        ready = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if ready else 0
        self.world = dist.get_world_size(group) if ready else 1
        self.views = shard_views(len(self.cameras), self.rank, self.world)
        self.buf = torch.zeros(n_params, dtype=torch.float32, device=device)

    def step(self, loss_grad):
        """Returns the summed (all-ranks) flat gradient buffer."""
        self.buf.zero_()
        for v in self.views:
            self.view_grad(self.scene, self.cameras[v], self.settings,
                           lambda color, v=v: loss_grad(v, color), self.buf)
        return allreduce_grads(self.buf, self.group)

    @property
    def views_per_rank(self):
        return math.ceil(len(self.cameras) / self.world)
