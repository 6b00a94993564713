"""Multi-GPU sharding of the evaluation path.

One process per GPU (torchrun), NCCL over NVLink for the only two exchanges
the path has:

* usage pass: every rank renders a subset of views of the server frame and
  the per-primitive int64 usage counts are all-reduced (SUM) -- integer, so
  the result is order independent and bit-exact at any world size;
* level sweep / keyframe probe: the (level, view) or (frame, view) items are
  dealt round-robin over ranks, each rank renders its items with SSE fused
  into compositing, and the per-item SSE values are all-gathered into the
  fixed item order.  Every rank then computes PSNR, means and decisions on
  the host in that order, so decisions are identical at 1, 2, 4 and 8 GPUs.

No parameters or images cross NVLink: every rank holds a replica of the frame
state and decodes deltas redundantly (a few hundred microseconds).  The
compute callbacks are injectable so the exchange logic is testable on CPU
with the gloo backend (tests/test_sharding.py).
"""

from __future__ import annotations

import math

import numpy as np


def _dist():
    import torch.distributed as dist

    return dist


def world_info(group=None):
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def item_partition(n_items: int, rank: int, world: int) -> np.ndarray:
    """Round-robin deal of item indices to ranks (balanced to +-1 item)."""
    return np.arange(rank, n_items, world, dtype=np.int64)


def block_partition(n_items: int, rank: int, world: int) -> np.ndarray:
    """Contiguous blocks of the item order (balanced to +-1 item).  Over
    frame-major (frame, view) items a rank touches ~n_frames/world + 1
    frames, so per-frame work such as the delta decode is barely repeated."""
    lo = (n_items * rank) // world
    hi = (n_items * (rank + 1)) // world
    return np.arange(lo, hi, dtype=np.int64)


def gather_ordered(local, n_items: int, rank: int, world: int, group=None, device=None, partition=None):
    """All-gather per-item float64 values into the global item order.
    ``local`` holds this rank's values in the order of ``partition``
    (default: round-robin ``item_partition``).  Returns a float64 tensor of
    length n_items on every rank."""
    import torch

    if world == 1:
        return local
    partition = partition or item_partition
    dist = _dist()
    per = math.ceil(n_items / world) + 1
    dev = device if device is not None else local.device
    buf = torch.zeros((per,), dtype=torch.float64, device=dev)
    buf[: local.numel()] = local
    parts = [torch.zeros((per,), dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.empty((n_items,), dtype=torch.float64, device=dev)
    for r in range(world):
        idx = partition(n_items, r, world)
        out[torch.from_numpy(idx).to(dev)] = parts[r][: idx.size]
    return out


def allreduce_counts_(counts, group=None):
    """In-place int64 SUM over ranks (exact)."""
    _, world = world_info(group)
    if world > 1:
        _dist().all_reduce(counts, op=_dist().ReduceOp.SUM, group=group)
    return counts


def mean_psnr(sse, pixels_per_view, n_views):
    """Per-frame mean over views of PSNR from SSE (host, fixed order)."""
    from .metrics import psnr_from_sse

    sse = np.asarray(sse)
    n_frames = sse.size // n_views
    return [float(np.mean([psnr_from_sse(sse[f * n_views + v], pixels_per_view[v]) for v in range(n_views)]))
            for f in range(n_frames)]


# ---------------------------------------------------------------------------
# sharded drivers (compute injectable)


def sharded_item_sse(n_items, sse_fn, group=None, device=None):
    """Evaluate ``sse_fn(item_indices) -> float64 tensor`` on this rank's
    share and return every item's SSE in global order on every rank."""
    rank, world = world_info(group)
    mine = item_partition(n_items, rank, world)
    local = sse_fn(mine)
    return gather_ordered(local, n_items, rank, world, group, device)


def sharded_usage(n_views, usage_fn, group=None):
    """``usage_fn(view_indices) -> int64 tensor`` summed over all views."""
    rank, world = world_info(group)
    counts = usage_fn(item_partition(n_views, rank, world))
    return allreduce_counts_(counts, group)


def probe_frames_sharded(frames, cams, targets, group=None, device=None):
    """Keyframe probes of many frames with (frame, view) items sharded over
    ranks; returns per-frame mean PSNR (identical on every rank)."""
    import torch

    from . import device as dv
    from .grouping import _device_targets
    from .rasterizer import render_views

    dev = dv.device_of(device)
    cams, frames = list(cams), list(frames)
    V = len(cams)
    tgts = [_device_targets(t, cams, dev) for t in targets]

    def sse_fn(idx):
        if idx.size == 0:
            return torch.zeros((0,), dtype=torch.float64, device=dev)
        items = [(int(i) // V, int(i) % V) for i in idx]
        vb = render_views(frames, cams, items, targets=[tgts[f][v] for f, v in items], device=dev)
        return vb.sse

    sse = sharded_item_sse(len(frames) * V, sse_fn, group, dev)
    px = [c.resolution[0] * c.resolution[1] * 3 for c in cams]
    return mean_psnr(sse.cpu().numpy(), px, V)


def probe_payloads_sharded(space, cams, payloads, payload_devs, targets, tau_db: float = 30.0, group=None,
                           device=None):
    """The pipelined device probe (grouping.probe_payload_items) of a batch
    of frames with the frame-major (frame, view) items split into contiguous
    blocks over the ranks: each rank decodes only the frames its block
    touches and renders only its views; one NCCL all-gather of the per-item
    SSE (8 bytes per view) gives every rank every frame's mean PSNR and
    keyframe decision, identical at any world size.  ``targets[t][v]`` need
    only exist for this rank's items.  Returns [(quality_db, is_keyframe)]."""
    from . import device as dv
    from .grouping import is_keyframe, probe_payload_items

    dev = dv.device_of(device)
    cams = list(cams)
    V = len(cams)
    n_items = len(payloads) * V
    rank, world = world_info(group)
    mine = block_partition(n_items, rank, world)
    items = [(int(i) // V, int(i) % V) for i in mine]
    if items:
        local = probe_payload_items(space, cams, payloads, payload_devs, targets, items, dev)
    else:
        import torch

        local = torch.zeros((0,), dtype=torch.float64, device=dev)
    sse = gather_ordered(local, n_items, rank, world, group, dev, partition=block_partition).cpu().numpy()
    px = [c.resolution[0] * c.resolution[1] * 3 for c in cams]
    return [(q, is_keyframe(q, tau_db)) for q in mean_psnr(sse, px, V)]


def probe_sequence_sharded(space, cams, payloads, targets, tau_db: float = 30.0, group=None, device=None):
    """grouping.probe_sequence from host buffers with the frame-major
    (frame, view) items split into contiguous blocks over the ranks: each
    rank copies H2D only its own items' targets (and the payloads of the
    frames its block touches), evaluates them, and one NCCL all-gather of the
    per-item SSE gives every rank every frame's quality and decision."""
    from . import device as dv
    from .grouping import is_keyframe, probe_sequence_items

    dev = dv.device_of(device)
    cams = list(cams)
    V = len(cams)
    n_items = len(payloads) * V
    rank, world = world_info(group)
    mine = block_partition(n_items, rank, world)
    local = probe_sequence_items(space, cams, payloads, targets, [(int(i) // V, int(i) % V) for i in mine], dev)
    sse = gather_ordered(local, n_items, rank, world, group, dev, partition=block_partition).cpu().numpy()
    px = [c.resolution[0] * c.resolution[1] * 3 for c in cams]
    return [(q, is_keyframe(q, tau_db)) for q in mean_psnr(sse, px, V)]


def usage_sharded(frame, cams, group=None, device=None):
    """render_with_usage counts with views sharded and an NCCL SUM."""
    import torch

    from . import device as dv
    from .rasterizer import render_views

    dev = dv.device_of(device)
    cams = list(cams)

    def usage_fn(views):
        if views.size == 0:
            return torch.zeros((frame.count,), dtype=torch.int64, device=dev)
        vb = render_views([frame], cams, [(0, int(v)) for v in views], usage_frames=[0], device=dev)
        return vb.usage[0]

    return sharded_usage(len(cams), usage_fn, group)


def build_level_space_sharded(delta, space, cams, ratios, usage, quant_step, base=None, frame_index=0, group=None):
    """pruning.build_level_space with the (level, view) items sharded over
    ranks; identical PruningLevelSpace on every rank.  Inputs are normalised
    and checked exactly as the single-GPU driver does (pruning.level_table),
    and each rank's renders are chunked by RENDER_PAIRS_PER_CALL."""
    import torch

    from . import pruning
    from .model import GaussianFrame, as_space
    from .rasterizer import render_views

    space = as_space(space)
    t = pruning.level_table(delta, space, ratios, usage, quant_step, base, removed=False)
    p = t.plan
    cams = list(cams)
    V = len(cams)
    if V == 0:
        levels = [pruning.PruningLevel(ratio=t.ratios[j], quality_db=100.0, size_bytes=t.sizes[j], pruned_indices=rm)
                  for j, rm in zip(t.keep, pruning.level_removed(t))]
        return pruning.PruningLevelSpace(levels=tuple(levels), frame_index=frame_index)
    dev = p.canon.device
    rank, world = world_info(group)
    mine = item_partition(len(t.keep) * V, rank, world)
    pruning._removed_prepare(p, t.delta.overlay())

    def run():
        # reference images only for the views this rank needs
        need_views = sorted({int(i) % V for i in mine})
        need_levels = sorted({int(i) // V for i in mine})
        kmin = {li: t.kmins[t.keep[li]] for li in need_levels}
        minrank = None
        if need_levels and pruning.tile_skip_enabled() and max(kmin.values()) > 0:
            # clean-tile skip, as in pruning.build_level_space
            minrank, (ref_planes, _) = pruning.tile_footprint(p, cams, max(kmin.values()))
        else:
            ref_planes = pruning.level_frame_planes(p, None)
        ref = GaussianFrame(device_params=ref_planes, count=p.n)
        refs = {}
        if need_views:
            rv = render_views([ref], cams, [(0, v) for v in need_views], want_images=True, device=dev)
            refs = dict(zip(need_views, rv.images))
        frames = {li: GaussianFrame(device_params=pruning.level_frame_planes(p, kmin[li]), count=p.n)
                  for li in need_levels}
        if mine.size == 0:
            local = torch.zeros((0,), dtype=torch.float64, device=dev)
        else:
            order = sorted(frames)
            pos = {li: k for k, li in enumerate(order)}
            items = [(pos[int(i) // V], int(i) % V) for i in mine]
            skip = None if minrank is None else [(minrank[int(i) % V], kmin[int(i) // V]) for i in mine]
            local = pruning.render_sse_chunked([frames[li] for li in order], cams, items,
                                               [refs[int(i) % V] for i in mine], device=dev, host=False,
                                               tile_skip=skip)
        pruning.level_removed(t)  # host-only work overlapping the enqueued renders
        return local

    # renders enqueued under deferred checking (re-run checked on a flag); the
    # collective follows on every rank exactly once
    local = pruning.deferred(dev, run)
    sse = gather_ordered(local, len(t.keep) * V, rank, world, group, dev).cpu().numpy()
    q = mean_psnr(sse, [c.resolution[0] * c.resolution[1] * 3 for c in cams], V)
    levels = [pruning.PruningLevel(ratio=t.ratios[j], quality_db=qq, size_bytes=t.sizes[j], pruned_indices=rm)
              for j, qq, rm in zip(t.keep, q, pruning.level_removed(t))]
    return pruning.PruningLevelSpace(levels=tuple(levels), frame_index=frame_index)
