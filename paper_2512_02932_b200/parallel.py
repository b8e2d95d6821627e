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
import os

__all__ = ["shard_views", "allreduce_grads", "replica_checksum", "MultiViewStep",
           "default_view_grad", "field_slices", "bucket_bounds", "bucketed_allreduce",
           "view_batch_grads"]


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


def field_slices(buf, n, sh_bases, g0, g1):
    """The five slices of a flat field-major gradient buffer (center | log_scale
    | rotation | opacity | sh, include/hgs.h) that hold Gaussians [g0, g1)."""
    B3 = 3 * sh_bases
    out = []
    off = 0
    for width in (3, 3, 4, 1, B3):
        out.append(buf[off + width * g0: off + width * g1])
        off += width * n
    return out


def bucket_bounds(n, buckets):
    """[g0, g1) Gaussian ranges of ``buckets`` near-equal buckets (multiples of
    32, the chain rule's warp step)."""
    step = -(-max(n, 1) // max(buckets, 1))
    step = -(-step // 32) * 32
    return [(g0, min(g0 + step, n)) for g0 in range(0, n, step)]


def bucketed_allreduce(out, n, sh_bases, buckets, write_bucket, group=None):
    """Fill and all-reduce a flat field-major gradient buffer bucket by bucket:
    ``write_bucket(g0, g1)`` enqueues the writes of Gaussians [g0, g1) (on the
    GPU: the chain rule over that range), then that bucket's five field slices
    are all-reduced asynchronously while the next bucket is written.  Waits
    for every collective before returning (the caller's stream then orders
    after them)."""
    import torch.distributed as dist
    works = []
    for g0, g1 in bucket_bounds(n, buckets):
        write_bucket(g0, g1)
        works += [dist.all_reduce(sl, op=dist.ReduceOp.SUM, group=group, async_op=True)
                  for sl in field_slices(out, n, sh_bases, g0, g1)]
    for w in works:
        w.wait()
    return out


def view_batch_grads(scene, cameras, settings, pixel_grads_of, out, scratch=None, touched=None,
                     flags=0, buckets=4, group=None, events=None, fwd_events=None, outputs=None,
                     ext_grads=(None, None, None), pipeline=None):
    """One data-parallel step's gradient over this rank's views, all-reduced.

    Every view's gradient is added into ``out`` (flat float32 n*P, KG = 1) by
    the chain rule itself (HGS_FLAG_ACCUMULATE; the first view overwrites).
    For the last view the chain rule runs in ``buckets`` Gaussian ranges and
    each range's five field slices are all-reduced asynchronously as soon as
    it is written, so the collective overlaps the remaining chain rule
    (NCCL runs on its own stream, ordered after the work already enqueued).
    ``pixel_grads_of(j, images)`` returns view j's (1, H, W, 3) upstream
    gradient.  ``fwd_events`` / ``events`` (5 / 3 torch.cuda.Event) time the
    last view's forward / backward stages; ``outputs`` are reused image
    buffers; ``ext_grads`` = (depth, normal, alpha) upstream gradients of the
    extension images (same for every view; each nullable).  ``pipeline``
    (0 / 1 / 2, default ``HGS_VIEW_PIPELINE`` or 1): view j + 1's forward
    is enqueued on a second stream while view j back-propagates (see
    ``_view_batch_pipelined``, the default; ``pipeline=2`` also moves each
    view's chain rule to a third stream).  Returns the last frame."""
    import torch.distributed as dist

    from . import grad, raster
    ready = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if ready else 1
    import torch
    n, B = scene.count, scene.sh_bases
    acc = out.view(1, -1)
    frame = None
    if not cameras:
        out.zero_()
    # Every view renders into one frame buffer with no host round trip
    # (HGS_FLAG_ASYNC): the views queue back to back on the stream.  Each
    # view's status / M / K word (the first 16 bytes of the frame) is copied
    # to pinned memory; a view that outgrew the pair capacity composited
    # nothing and back-propagated zeros, so it is simply redone synchronously
    # (accumulating) once the step's work has drained.
    dev = scene.device
    if cameras and any((int(c.width), int(c.height)) != (int(cameras[0].width), int(cameras[0].height))
                       for c in cameras):
        from .errors import ConfigError
        raise ConfigError("view_batch_grads: every camera of a batch must have the same image size")
    fbuf = torch.empty(raster.frame_bytes(n, int(cameras[0].width), int(cameras[0].height)),
                       dtype=torch.uint8, device=dev) if cameras else None
    heads = torch.empty((len(cameras), 16), dtype=torch.uint8, pin_memory=True) if cameras else None

    def view(j, cam, last, async_):
        imgs, fr = raster.rasterize(scene, cam, settings, flags, outputs=outputs,
                                    events=fwd_events if last else None, async_=async_,
                                    frame_buf=fbuf if async_ else None)
        if async_:
            heads[j].copy_(fbuf[:16], non_blocking=True)
        return imgs, fr

    pipe = _PIPELINE if pipeline is None else pipeline
    if pipe and len(cameras) >= 2:
        return _view_batch_pipelined(scene, cameras, settings, pixel_grads_of, out, acc, scratch,
                                     touched, flags, buckets, group, events, fwd_events, outputs,
                                     ext_grads, fbuf, heads, view, world, pipe)
    for j, cam in enumerate(cameras):
        last = j == len(cameras) - 1
        imgs, frame = view(j, cam, last, True)
        pg = pixel_grads_of(j, imgs)
        if not last or world == 1:
            grad.backward_device(frame, pg, *ext_grads, grads_out=acc, touched_out=touched,
                                 scratch=scratch, accumulate=j > 0, events=events if last else None)
            continue
        grad.backward_device(frame, pg, *ext_grads, grads_out=acc, touched_out=touched,
                             scratch=scratch, replay_only=True, events=events)
        if _redo_failed(cameras, heads, view, pixel_grads_of, ext_grads, acc, touched, scratch,
                        last_excluded=True):
            frame = view(j, cam, True, False)[1]  # the last view again, synchronously
            grad.backward_device(frame, pg, *ext_grads, grads_out=acc, touched_out=touched,
                                 scratch=scratch, replay_only=True)
        bucketed_allreduce(out, n, B, buckets,
                           lambda g0, g1: grad.chain_range(frame, g0, g1, acc, accumulate=True),
                           group=group)
        return frame
    if cameras:
        _redo_failed(cameras, heads, view, pixel_grads_of, ext_grads, acc, touched, scratch)
    if world > 1:  # no views on this rank: contribute zeros
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return frame


_PIPELINE = int(os.environ.get("HGS_VIEW_PIPELINE", "1"))  # 0 off, 1 two streams, 2 three
_PIPE_PRIO = os.environ.get("HGS_PIPE_PRIO", "none")  # which stream gets the higher priority
_pipe_streams = {}  # device index -> (forward stream, backward stream)


def _streams(dev):
    import torch
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _pipe_streams:
        lo, hi = torch.cuda.Stream.priority_range()  # (0, -N): lower number = higher priority
        pf = hi if _PIPE_PRIO == "fwd" else 0
        pb = hi if _PIPE_PRIO == "bwd" else 0
        _pipe_streams[idx] = (torch.cuda.Stream(device=idx, priority=pf),
                              torch.cuda.Stream(device=idx, priority=pb))
    return _pipe_streams[idx]


_chain_streams = {}


def _chain_stream(dev):
    import torch
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _chain_streams:
        _chain_streams[idx] = torch.cuda.Stream(device=idx)
    return _chain_streams[idx]


def _view_batch_pipelined(scene, cameras, settings, pixel_grads_of, out, acc, scratch, touched,
                          flags, buckets, group, events, fwd_events, outputs, ext_grads, fbuf,
                          heads, view, world, pipe):
    """Views of one batch are independent given the scene, so the forward of
    view j + 1 need not wait for the backward of view j: forwards queue on
    one stream, backwards on another (the higher-priority one), and the
    latency-bound front end of the next view (depth sort, float64
    preprocess, binning) fills the SM slots the current view's compositors
    leave.  Two frame buffers and two image sets alternate (the last view
    gets the caller's ``outputs``); the forward into a buffer waits for the backward of view j - 2 (its last
    reader), every backward waits for its own forward, and the backwards
    stay in view order on their stream (they share the scratch and add into
    ``out``).  The last view's backward runs on the caller's stream after
    both streams, exactly as in the sequential loop (replay, then the
    bucketed chain rule + all-reduce for world > 1)."""
    import torch

    from . import grad, raster
    dev = scene.device
    cur = torch.cuda.current_stream(dev)
    fs, bs = _streams(dev)
    fs.wait_stream(cur)
    bs.wait_stream(cur)
    W, H = int(cameras[0].width), int(cameras[0].height)
    fbufs = [fbuf, torch.empty_like(fbuf)]
    outs = [outputs, None]
    if outputs is None:
        outs[0] = {}
    for k in (0, 1):
        o = outs[k] if outs[k] is not None else {}
        outs[k] = {key: o.get(key) if o.get(key) is not None else torch.empty(shape, device=dev)
                   for key, shape in (("color", (H, W, 3)), ("depth", (H, W)),
                                      ("transmittance", (H, W)), ("alpha", (H, W)),
                                      ("normal", (H, W, 3)))}
    fwd_done = [torch.cuda.Event(), torch.cuda.Event()]
    bwd_done = [torch.cuda.Event(), torch.cuda.Event()]  # view's last reader of its buffers done
    rep_done = [torch.cuda.Event(), torch.cuda.Event()]
    # split: each view's chain rule (HBM-bound) on a third stream, beside the
    # next view's replay (issue-bound); the two alternate between two scratches
    split = pipe >= 2
    if split:
        if scratch is None:
            from . import _lib
            scratch = torch.empty(_lib.lib().hgs_backward_scratch_bytes(scene.count, 1),
                                  dtype=torch.uint8, device=dev)
        cs = _chain_stream(dev)
        cs.wait_stream(cur)
        scratches = [scratch, torch.empty_like(scratch)]
    n_views = len(cameras)
    frame = None
    for j, cam in enumerate(cameras):
        last = j == n_views - 1
        b = (n_views - 1 - j) & 1  # the last view renders into the caller's image set
        with torch.cuda.stream(fs):
            if j >= 2:
                fs.wait_event(bwd_done[b])  # view j - 2's backward read this buffer / image set
            imgs, frame = raster.rasterize(scene, cam, settings, flags, outputs=outs[b],
                                           events=fwd_events if last else None, async_=True,
                                           frame_buf=fbufs[b])
            heads[j].copy_(fbufs[b][:16], non_blocking=True)
            fwd_done[b].record(fs)
        if last:
            break
        with torch.cuda.stream(bs):
            bs.wait_event(fwd_done[b])
            pg = pixel_grads_of(j, imgs)
            if not split:
                grad.backward_device(frame, pg, *ext_grads, grads_out=acc, touched_out=touched,
                                     scratch=scratch, accumulate=j > 0)
                bwd_done[b].record(bs)
                continue
            if j >= 2:
                bs.wait_event(bwd_done[b])  # view j - 2's chain rule read this scratch
            grad.backward_device(frame, pg, *ext_grads, grads_out=acc, touched_out=touched,
                                 scratch=scratches[b], replay_only=True)
            rep_done[b].record(bs)
        with torch.cuda.stream(cs):
            cs.wait_event(rep_done[b])
            grad.chain_range(frame, 0, scene.count, acc, accumulate=j > 0)
            bwd_done[b].record(cs)
    cur.wait_stream(fs)
    cur.wait_stream(bs)
    if split:
        cur.wait_stream(cs)
        scratch = scratches[0]  # the last view's set (b = 0)
    # the sequential loop's epilogue: the last view's backward on the caller's stream
    pg = pixel_grads_of(n_views - 1, imgs)
    if world == 1:
        grad.backward_device(frame, pg, *ext_grads, grads_out=acc, touched_out=touched,
                             scratch=scratch, accumulate=True, events=events)
        _redo_failed(cameras, heads, view, pixel_grads_of, ext_grads, acc, touched, scratch)
        return frame
    grad.backward_device(frame, pg, *ext_grads, grads_out=acc, touched_out=touched,
                         scratch=scratch, replay_only=True, events=events)
    if _redo_failed(cameras, heads, view, pixel_grads_of, ext_grads, acc, touched, scratch,
                    last_excluded=True):
        frame = view(n_views - 1, cameras[-1], True, False)[1]
        grad.backward_device(frame, pg, *ext_grads, grads_out=acc, touched_out=touched,
                             scratch=scratch, replay_only=True)
    bucketed_allreduce(out, scene.count, scene.sh_bases, buckets,
                       lambda g0, g1: grad.chain_range(frame, g0, g1, acc, accumulate=True),
                       group=group)
    return frame


def _redo_failed(cameras, heads, view, pixel_grads_of, ext_grads, acc, touched, scratch,
                 last_excluded=False):
    """Re-render synchronously (growing the frame buffer) and accumulate the
    views whose asynchronous frame reported a status; True if the last view
    failed and ``last_excluded`` (the caller redoes it: its chain rule is
    still pending).  Other statuses raise as the reference exceptions."""
    import torch

    from . import _lib, grad
    torch.cuda.current_stream().synchronize()
    status = heads.view(torch.int32)[:, 0].tolist()
    last_failed = False
    for j, st in enumerate(status):
        if not st:
            continue
        if st != _lib.HGS_ERR_PAIR_CAPACITY:
            _lib.check(st, "hgs_forward (view %d)" % j)
        if last_excluded and j == len(cameras) - 1:
            last_failed = True
            continue
        imgs, fr = view(j, cameras[j], False, False)
        grad.backward_device(fr, pixel_grads_of(j, imgs), *ext_grads, grads_out=acc,
                             touched_out=touched, scratch=scratch, accumulate=True)
    return last_failed


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
