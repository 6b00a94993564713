"""Tile rasterizer on B200 (drop-in for ``ss/rasterizer.py``).

``render`` / ``render_with_usage`` keep the reference signatures and return
the reference's ``RenderedImage`` / ``UsageFrequency``; ``forward`` is the
reference's pluggable kernel seam (``ss/_composite.pyx:18``).  The batched
entry point ``render_views`` evaluates many (frame, camera) items in one
pipeline pass and returns device tensors (images, per-item SSE, usage) for
the hot paths in ``pruning`` / ``grouping`` / ``streamsim``.

Numerics: projection follows ``_prepare`` op-for-op in fp64 (OpenBLAS FMA
order for the small matmuls); compositing evaluates every (pixel,
primitive) pair that could contribute exactly as ``_composite.pyx:53-68``
after an fp32 log-domain fast reject with a proven guard band.
"""

from __future__ import annotations

import numpy as np

from . import device as dv
from ._lib import CameraC, FrameC, ItemC, engine, ptr
from .camera import camera_struct
from .errors import StructuralError, ValidationError
from .model import GaussianFrame

KERNEL_BACKEND = "cuda-sm_100a"
EPS_CONTRIB = 1.0 / 255.0
ALPHA_CLAMP = 0.999
COV_BLUR = 0.3
RADIUS_SIGMA = 3.5
SH_C0 = 0.2820947917738781
SH_C1 = 0.4886025119029199


class RenderedImage:
    """(h, w, 3) float64 image in [0, 1] (ss/rasterizer.py:59-74)."""

    __slots__ = ("pixels", "resolution")

    def __init__(self, pixels, resolution):
        px = np.asarray(pixels, dtype=np.float64)
        w, h = resolution
        if px.shape != (h, w, 3):
            raise StructuralError("pixel buffer does not match resolution")
        if not np.all(np.isfinite(px)):
            raise ValidationError("non-finite pixel values")
        px = np.ascontiguousarray(px)
        px.setflags(write=False)
        object.__setattr__(self, "pixels", px)
        object.__setattr__(self, "resolution", (int(w), int(h)))

    def __setattr__(self, k, v):
        raise AttributeError("RenderedImage is immutable")

    def __array__(self, dtype=None, copy=None):
        # np.asarray(image) is its pixels: reference helpers that accept
        # "a RenderedImage or an array" (ss/metrics.py:23-26) take this one too
        return self.pixels if dtype is None else self.pixels.astype(dtype)


class UsageFrequency:
    """Per-primitive count of (pixel, view) pairs with perceptible weight."""

    __slots__ = ("counts",)

    def __init__(self, counts):
        object.__setattr__(self, "counts", counts)

    def __setattr__(self, k, v):
        raise AttributeError("UsageFrequency is immutable")

    def merged_with(self, other: "UsageFrequency") -> "UsageFrequency":
        if self.counts.shape != other.counts.shape:
            raise StructuralError("usage count length mismatch")
        return UsageFrequency(counts=self.counts + other.counts)


# ---------------------------------------------------------------------------
# batched device API


class ViewBatch:
    """Result of ``render_views``: device tensors, one entry per item."""

    __slots__ = ("sse", "images", "usage", "launches")

    def __init__(self, sse, images, usage, launches):
        self.sse = sse
        self.images = images
        self.usage = usage
        self.launches = launches


def _frame_planes(frame, dev):
    if isinstance(frame, GaussianFrame):
        return frame.planes(dev), frame.count, frame.width
    p = np.asarray(frame.params, dtype=np.float64)  # reference GaussianFrame or lookalike
    if p.ndim != 2:
        raise StructuralError("params must be (n, param_dim)")
    return dv.upload_params(p, dev), p.shape[0], p.shape[1]


def render_views(frames, cams, items, targets=None, want_images=False, usage_frames=None, device=None,
                 frozen=None, tile_skip=None):
    """Render ``items`` = [(frame_idx, cam_idx), ...] in one pipeline pass.

    targets: optional list (per item) of device (h, w, 3) float64 tensors;
      per-item SSE against them is returned in ``.sse`` (device float64).
    want_images: return clipped device images per item.
    usage_frames: iterable of frame indices whose items accumulate usage
      counts; ``.usage[f]`` is an int64 device tensor over the frame.
    frozen: optional list (per item) of frozen-order position tensors
      (``frozen_positions``) or None (ss/rasterizer.py:128-142).
    tile_skip: optional list (per item) of (minrank, keep_min) or None, for
      SSE-only items of a pruning-level sweep: tiles g with minrank[g] >=
      keep_min are known to equal the target and are not composited
      (``pruning.tile_footprint``; airgs_view_item.tile_minrank).
    """
    import torch

    dev = dv.device_of(device)
    eng = engine(dev)
    frames = list(frames)
    cams = list(cams)
    items = list(items)
    if not items:
        return ViewBatch(torch.zeros(0, dtype=torch.float64, device=dev), [], {}, 0)
    planes = []
    fc = (FrameC * len(frames))()
    for k, f in enumerate(frames):
        p, n, w = _frame_planes(f, dev)
        if n == 0:
            raise StructuralError("cannot render an empty frame")
        planes.append(p)
        fc[k].params = p.data_ptr()
        fc[k].count = n
        fc[k].ld = p.shape[1]
        fc[k].width = w
    cc = (CameraC * len(cams))(*[camera_struct(c) for c in cams])
    usage = {}
    for f in (usage_frames or ()):
        usage[f] = torch.zeros((fc[f].count,), dtype=torch.int64, device=dev)
    images = []
    ic = (ItemC * len(items))()
    for s, (fi, ci) in enumerate(items):
        ic[s].frame = fi
        ic[s].camera = ci
        if targets is not None and targets[s] is not None:
            ic[s].target = targets[s].data_ptr()
        if want_images:
            w, h = cams[ci].resolution
            img = torch.empty((h, w, 3), dtype=torch.float64, device=dev)
            images.append(img)
            ic[s].image = img.data_ptr()
        if fi in usage:
            ic[s].usage = usage[fi].data_ptr()
        if frozen is not None and frozen[s] is not None:
            ic[s].frozen_pos = frozen[s].data_ptr()
        if tile_skip is not None and tile_skip[s] is not None:
            mr, km = tile_skip[s]
            ic[s].tile_minrank = mr.data_ptr()
            ic[s].tile_keep_min = int(km)
    sse = torch.zeros((len(items),), dtype=torch.float64, device=dev)
    before = eng.launches
    eng.call("airgs_render", fc, len(frames), cc, len(cams), ic, len(items), ptr(sse), eng.stream())
    return ViewBatch(sse, images, usage, eng.launches - before)


# ---------------------------------------------------------------------------
# reference-compatible API


def render(frame, cam) -> RenderedImage:
    """Render one frame; pure and deterministic (ss/rasterizer.py:215-222)."""
    if frame.count == 0:
        raise StructuralError("cannot render an empty frame")
    vb = render_views([frame], [cam], [(0, 0)], want_images=True)
    return RenderedImage(pixels=vb.images[0].cpu().numpy(), resolution=cam.resolution)


def render_with_usage(frame, cams) -> tuple:
    """Per-camera images plus usage counts summed over cameras
    (ss/rasterizer.py:225-240)."""
    cams = list(cams)
    if not cams:
        raise StructuralError("at least one camera required")
    if frame.count == 0:
        raise StructuralError("cannot render an empty frame")
    vb = render_views([frame], cams, [(0, k) for k in range(len(cams))], want_images=True, usage_frames=[0])
    imgs = [RenderedImage(pixels=im.cpu().numpy(), resolution=c.resolution) for im, c in zip(vb.images, cams)]
    return imgs, UsageFrequency(counts=vb.usage[0].cpu().numpy())


class ForwardState:
    """What ``render_backward`` needs from ``render_forward``: the frame (host
    or device parameters), the camera and the frozen order, if any.  The
    backward recomputes the forward on the device with its contribution
    record (deterministic: the same order, masks and final transmittance)."""

    __slots__ = ("frame", "cam", "frozen")

    def __init__(self, frame, cam, frozen=None):
        self.frame = frame
        self.cam = cam
        self.frozen = frozen


def frozen_positions(frozen_order, n, device=None):
    """Device int64[n]: position of each primitive in ``frozen_order``, -1 if
    absent (the device form of _prepare's frozen_order argument)."""
    import torch

    dev = dv.device_of(device)
    pos = torch.full((n,), -1, dtype=torch.int64, device=dev)
    fo = torch.as_tensor(np.asarray(frozen_order, dtype=np.int64) if not isinstance(frozen_order, torch.Tensor)
                         else frozen_order, dtype=torch.int64).to(dev)
    if fo.numel():
        if int(fo.min()) < 0 or int(fo.max()) >= n:
            raise StructuralError("frozen order references a missing primitive")
        pos[fo] = torch.arange(fo.numel(), dtype=torch.int64, device=dev)
    return pos


def compositing_orders(frame, cams, frozen_orders=None) -> list:
    """Per-camera compositing orders of ``frame`` (ss/rasterizer.py:243-246):
    the kept primitives (z > near, alpha > 1/255) in stable depth order, or in
    the frozen order followed by the rest by depth."""
    import ctypes

    import torch

    dev = dv.device_of(None)
    eng = engine(dev)
    p, n, w = _frame_planes(frame, dev)
    fc = FrameC()
    fc.params, fc.count, fc.ld, fc.width = p.data_ptr(), n, p.shape[1], w
    out = []
    for k, cam in enumerate(cams):
        fz = None
        if frozen_orders is not None and frozen_orders[k] is not None:
            fz = frozen_positions(frozen_orders[k], n, dev)
        order = torch.empty((max(n, 1),), dtype=torch.int64, device=dev)
        kept = ctypes.c_int64(0)
        cc = camera_struct(cam)
        eng.call("airgs_compositing_order", ctypes.byref(fc), ctypes.byref(cc), ptr(fz), ptr(order),
                 ctypes.byref(kept), eng.stream())
        out.append(order[: kept.value].cpu().numpy())
    return out


def tile_lists(frame, cam, max_per_tile: int = 4096):
    """Debug view of the binning + sort stage for one camera
    (airgs_debug_tile_lists): returns ``(counts, lists)`` where ``counts`` is
    int32[tiles_y, tiles_x] and ``lists[g]`` the primitive indices of 16x16
    tile g (row-major) in compositing order."""
    import ctypes

    import torch

    dev = dv.device_of(None)
    eng = engine(dev)
    p, n, w = _frame_planes(frame, dev)
    if n == 0:
        raise StructuralError("cannot render an empty frame")
    fc = FrameC()
    fc.params, fc.count, fc.ld, fc.width = p.data_ptr(), n, p.shape[1], w
    cc = camera_struct(cam)
    W, H = cam.resolution
    tx, ty = (W + 15) // 16, (H + 15) // 16
    counts = torch.zeros((tx * ty,), dtype=torch.int32, device=dev)
    ids = torch.full((tx * ty * max_per_tile,), -1, dtype=torch.int32, device=dev)
    eng.call("airgs_debug_tile_lists", ctypes.byref(fc), ctypes.byref(cc), int(max_per_tile), ptr(counts), ptr(ids),
             eng.stream())
    c = counts.cpu().numpy()
    if c.size and int(c.max()) > max_per_tile:
        raise ValueError(f"a tile list holds {int(c.max())} entries > max_per_tile={max_per_tile}")
    flat = ids.view(tx * ty, max_per_tile).cpu().numpy()
    return c.reshape(ty, tx), [flat[g, : c[g]].astype(np.int64) for g in range(tx * ty)]


def render_forward(frame, cam, frozen_order=None):
    """Forward pass that records what backward needs (ss/rasterizer.py:248-257).
    Returns ``(image, state)``; ``image`` is the forward image (h, w, 3) (the
    reference's unclipped kernel output; compositing keeps it in [0, 1)).
    ``frozen_order`` reuses a compositing order (see compositing_orders)."""
    if frame.count == 0:
        raise StructuralError("cannot render an empty frame")
    fz = None if frozen_order is None else frozen_positions(frozen_order, frame.count)
    vb = render_views([frame], [cam], [(0, 0)], want_images=True, frozen=[fz])
    return vb.images[0].cpu().numpy(), ForwardState(frame, cam, fz)


def render_backward(state, d_image, as_numpy: bool = True):
    """Backpropagate ``d_image`` (dLoss/dpixel, (h, w, 3)) to the
    pre-activation parameters, depth order and contribution masks frozen to
    the recorded forward (ss/rasterizer.py:270-369).  Returns an (n, width)
    gradient array."""
    import ctypes

    import torch

    dev = dv.device_of(None)
    eng = engine(dev)
    frame, cam = state.frame, state.cam
    p, n, w = _frame_planes(frame, dev)
    wpx, hpx = cam.resolution
    if isinstance(d_image, torch.Tensor):
        dimg = d_image.to(device=dev, dtype=torch.float64).contiguous()
    else:
        dimg = torch.from_numpy(np.ascontiguousarray(np.asarray(d_image, dtype=np.float64))).to(dev)
    if tuple(dimg.shape) != (hpx, wpx, 3):
        raise StructuralError(f"d_image shape {tuple(dimg.shape)} != ({hpx}, {wpx}, 3)")
    fc = FrameC()
    fc.params, fc.count, fc.ld, fc.width = p.data_ptr(), n, p.shape[1], w
    cc = camera_struct(cam)
    grads = torch.empty((n, w), dtype=torch.float64, device=dev)
    eng.call("airgs_render_backward", ctypes.byref(fc), ctypes.byref(cc), ptr(state.frozen), ptr(dimg), ptr(grads),
             eng.stream())
    return grads.cpu().numpy() if as_numpy else grads


def _seam_inputs(means2d, conics, alphas, colors, bboxes, dev):
    import torch

    def t(a, dt):
        if isinstance(a, torch.Tensor):
            return a.to(device=dev, dtype=dt).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.float64 if dt == torch.float64
                                                    else np.int64)).to(dev)

    return (t(means2d, torch.float64), t(conics, torch.float64), t(alphas, torch.float64),
            t(colors, torch.float64), t(bboxes, torch.int64))


def _mask_offsets(bb):
    """Per-primitive offsets of the reference's mask layout and its total size
    (ss/_composite.pyx:29-35: the buffer covers every bbox area, offsets
    advance over the non-empty ones)."""
    import torch

    w = bb[:, 1] - bb[:, 0]
    h = bb[:, 3] - bb[:, 2]
    area = w * h
    valid = (w > 0) & (h > 0)
    off = torch.cumsum(torch.where(valid, area, torch.zeros_like(area)), 0) - torch.where(valid, area,
                                                                                          torch.zeros_like(area))
    return off.contiguous(), int(area.sum().item()) if area.numel() else 0


def forward(means2d, conics, alphas, colors, bboxes, height, width, record=False):
    """The reference kernel seam ``_composite.forward`` on the GPU.

    Inputs are numpy arrays (or CUDA tensors) of depth-ordered primitives;
    returns numpy ``(image (h,w,3) unclipped, t_final (h,w), usage (k,),
    masks)`` with ``masks`` the reference's uint8 contribution masks when
    ``record`` (ss/_composite.pyx:18-74), else None.
    """
    import torch

    dev = dv.device_of(None)
    eng = engine(dev)
    m2, co, al, cl, bb = _seam_inputs(means2d, conics, alphas, colors, bboxes, dev)
    k = m2.shape[0]
    img = torch.empty((int(height), int(width), 3), dtype=torch.float64, device=dev)
    tr = torch.empty((int(height), int(width)), dtype=torch.float64, device=dev)
    us = torch.zeros((max(k, 1),), dtype=torch.int64, device=dev)
    if not record:
        eng.call("airgs_composite_forward", k, ptr(m2), ptr(co), ptr(al), ptr(cl), ptr(bb), int(height),
                 int(width), ptr(img), ptr(tr), ptr(us), eng.stream())
        return img.cpu().numpy(), tr.cpu().numpy(), us[:k].cpu().numpy(), None
    off, total = _mask_offsets(bb)
    masks = torch.zeros((max(total, 1),), dtype=torch.uint8, device=dev)
    eng.call("airgs_composite_forward_record", k, ptr(m2), ptr(co), ptr(al), ptr(cl), ptr(bb), int(height),
             int(width), ptr(img), ptr(tr), ptr(us), ptr(off), ptr(masks), eng.stream())
    return img.cpu().numpy(), tr.cpu().numpy(), us[:k].cpu().numpy(), masks[:total].cpu().numpy()


def backward(means2d, conics, alphas, colors, bboxes, height, width, masks, t_final, d_image):
    """The reference kernel seam ``_composite.backward`` on the GPU
    (ss/_composite.pyx:77-152): returns numpy ``(d_means2d (k,2), d_conics
    (k,3), d_alphas (k,), d_colors (k,3))``."""
    import torch

    dev = dv.device_of(None)
    eng = engine(dev)
    m2, co, al, cl, bb = _seam_inputs(means2d, conics, alphas, colors, bboxes, dev)
    k = m2.shape[0]
    off, total = _mask_offsets(bb)
    mk = torch.as_tensor(np.ascontiguousarray(np.asarray(masks, dtype=np.uint8))).to(dev)
    if mk.numel() < total:
        raise StructuralError("masks shorter than the primitives' bbox areas")
    tf = torch.as_tensor(np.ascontiguousarray(np.asarray(t_final, dtype=np.float64))).to(dev)
    di = torch.as_tensor(np.ascontiguousarray(np.asarray(d_image, dtype=np.float64))).to(dev)
    if tuple(tf.shape) != (int(height), int(width)) or tuple(di.shape) != (int(height), int(width), 3):
        raise StructuralError("t_final / d_image shape mismatch")
    g9 = torch.zeros((max(k, 1), 9), dtype=torch.float64, device=dev)
    eng.call("airgs_composite_backward", k, ptr(m2), ptr(co), ptr(al), ptr(cl), ptr(bb), int(height), int(width),
             ptr(off), ptr(mk), ptr(tf), ptr(di), ptr(g9), eng.stream())
    g = g9[:k].cpu().numpy()
    return (np.ascontiguousarray(g[:, 0:2]), np.ascontiguousarray(g[:, 2:5]), np.ascontiguousarray(g[:, 5]),
            np.ascontiguousarray(g[:, 6:9]))


