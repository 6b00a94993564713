"""Keyframe detection on device (drop-in for the probe half of
``ss/grouping.py``).

``frame_quality`` = arithmetic-mean PSNR over the evaluation cameras of the
frame's renders against ground truth (ss/grouping.py:153-159);
``quality_probe`` applies a delta first (:162-166); a frame stays in its
group iff ``q >= tau`` (:213), otherwise it becomes a keyframe.
``probe_frames`` evaluates many candidate frames x views in one batched
render with SSE fused into compositing -- the C2 keyframe-detection workload.
The training-based grouping driver ``build_groups`` (fit_group_frame /
fit_keyframe, ss/grouping.py:169-250) is outside the evaluation path
(ss/train.py OUT OF SCOPE); with ``dropin.install`` the
reference's own driver runs on top of this module's probe.
"""

from __future__ import annotations

import json
import os

import numpy as np

from . import device as dv
from .errors import StructuralError, ValidationError
from .metrics import psnr_from_sse
from .model import CanonicalSpace, DeltaTensor, apply_delta, as_frame

DEFAULT_TAU_DB = 30.0


class GroundTruth:
    """Per-camera target images of one time step (as ss/train.py:92-107)."""

    __slots__ = ("images", "_dev")

    def __init__(self, images):
        object.__setattr__(self, "images", tuple(np.asarray(im, dtype=np.float64) for im in images))
        object.__setattr__(self, "_dev", None)

    def __setattr__(self, k, v):
        raise AttributeError("GroundTruth is immutable")

    def check_cameras(self, cams):
        check_targets(self.images, cams)

    def device_images(self, device=None):
        import torch

        dev = dv.device_of(device)
        if self._dev is None or self._dev[0].device != dev:
            object.__setattr__(self, "_dev", [torch.from_numpy(np.ascontiguousarray(im)).to(dev)
                                              for im in self.images])
        return self._dev


def check_targets(images, cams):
    if len(images) != len(cams):
        raise StructuralError("target image count does not match cameras")
    for im, cam in zip(images, cams):
        w, h = cam.resolution
        if tuple(im.shape) != (h, w, 3):
            raise StructuralError("target resolution does not match camera")


def _device_targets(target, cams, dev):
    import torch

    if isinstance(target, GroundTruth):
        target.check_cameras(cams)
        return target.device_images(dev)
    imgs = getattr(target, "images", target)
    out = []
    for im in imgs:
        if isinstance(im, torch.Tensor):
            out.append(im.to(device=dev, dtype=torch.float64).contiguous())
        else:
            out.append(torch.from_numpy(np.ascontiguousarray(np.asarray(getattr(im, "pixels", im),
                                                                        dtype=np.float64))).to(dev))
    check_targets(out, cams)
    return out


def frame_quality(frame, cams, target) -> float:
    """Mean PSNR of the frame's renders against the targets."""
    return probe_frames([frame], cams, [target])[0]


def quality_probe(space: CanonicalSpace, delta: DeltaTensor, target, cams) -> float:
    return frame_quality(apply_delta(space, delta), cams, target)


def probe_frames(frames, cams, targets, device=None) -> list:
    """Mean-over-views PSNR of each frame against its targets, all
    (frame, view) pairs in one batched render."""
    from .rasterizer import render_views

    dev = dv.device_of(device)
    cams = list(cams)
    frames = [as_frame(f) for f in frames]
    if not cams:
        raise ValidationError("at least one camera required")
    tgts = [_device_targets(t, cams, dev) for t in targets]
    items, tlist = [], []
    for f in range(len(frames)):
        for v in range(len(cams)):
            items.append((f, v))
            tlist.append(tgts[f][v])
    vb = render_views(frames, cams, items, targets=tlist, device=dev)
    sse = vb.sse.cpu().numpy()
    V = len(cams)
    px = [c.resolution[0] * c.resolution[1] * 3 for c in cams]
    return [float(np.mean([psnr_from_sse(sse[f * V + v], px[v]) for v in range(V)])) for f in range(len(frames))]


def _in_item_order(pieces, order, n_items, dev):
    """Concatenate per-frame SSE pieces (evaluation order ``order``) into
    item order on the device -- no per-frame host->device index copies,
    which would stall the stream pipeline."""
    import torch

    if not pieces:
        return torch.zeros((n_items,), dtype=torch.float64, device=dev)
    cat = torch.cat(pieces)
    if order == list(range(n_items)):
        return cat
    out = torch.empty((n_items,), dtype=torch.float64, device=dev)
    out[torch.tensor(order, dtype=torch.int64).to(dev, non_blocking=False)] = cat
    return out


_STREAM_BUFS: dict = {}


def _stream_buffers(dev, cap, view_shapes):
    """Double buffers of the streamed probe, kept per device across calls and
    grown on demand: two pinned host payload buffers of >= cap bytes (a
    cudaHostAlloc synchronises the device and costs milliseconds), two device
    payload buffers, and per buffer one device float64 target image per
    (view, shape) in ``view_shapes``.  Returns (pinned[2], dpay[2],
    [{view: tensor}] * 2)."""
    import torch

    key = str(dev)
    st = _STREAM_BUFS.get(key)
    if st is None or st["cap"] < cap:
        c = max(int(cap), 1)
        st = {"cap": c, "tg": [{}, {}] if st is None else st["tg"],
              "pinned": [torch.empty((c,), dtype=torch.uint8).pin_memory() for _ in range(2)],
              "dpay": [torch.empty((c,), dtype=torch.uint8, device=dev) for _ in range(2)]}
        _STREAM_BUFS[key] = st
    dtg = []
    for b in range(2):
        cache = st["tg"][b]
        for v, shp in view_shapes.items():
            if (v, shp) not in cache:
                cache[(v, shp)] = torch.empty(shp, dtype=torch.float64, device=dev)
        dtg.append({v: cache[(v, shp)] for v, shp in view_shapes.items()})
    return st["pinned"], st["dpay"], dtg


def probe_sequence_items(space, cams, payloads, targets, items, device=None):
    """Per-item SSE of (frame t, view v) items streamed from host memory: for
    each frame that has items, its GSDP payload and the items' (h, w, 3)
    float64 host targets (pinned torch tensors give asynchronous copies) are
    copied H2D on a copy stream while the previous frame is evaluated (double
    buffering), then the frame is decoded and applied (fused) and its items
    rendered with SSE fused into compositing.  The whole batch runs under
    deferred checking (no host synchronisation per frame); a flagged batch is
    re-run in checked mode for the reference's exact error.  Returns a device
    float64 tensor in ``items`` order.  ``targets[t][v]`` need only exist for
    listed items."""
    import ctypes

    import torch

    from . import codec
    from ._lib import engine
    from .model import GaussianFrame, as_space
    from .rasterizer import render_views

    space = as_space(space)
    dev = dv.device_of(device)
    cams = list(cams)
    n, w = space.frame.count, space.frame.width
    canon = space.frame.planes(dev)
    comp = torch.cuda.current_stream(dev)
    by_frame = {}
    for k, (t, v) in enumerate(items):
        by_frame.setdefault(int(t), []).append((k, int(v)))
    order = list(by_frame)
    datas = {t: (payloads[t].data if hasattr(payloads[t], "data") else bytes(payloads[t])) for t in order}
    cap = max((len(d) for d in datas.values()), default=1)
    res = [(c.resolution[1], c.resolution[0], 3) for c in cams]
    for t in order:
        for _, v in by_frame[t]:
            if tuple(targets[t][v].shape) != res[v]:
                raise StructuralError("target resolution does not match camera")
    # double buffers, kept across calls (_stream_buffers): pinned payload staging (a
    # cudaHostAlloc synchronises the device and costs milliseconds) and device
    # targets / payloads (no allocator churn)
    pinned, dpay, dtg = _stream_buffers(dev, cap, {v: res[v] for lst in by_frame.values() for _, v in lst})
    bufst = _STREAM_BUFS[str(dev)]
    copy = bufst.setdefault("copy", torch.cuda.Stream(dev))

    def host_tensor(im):
        return im if isinstance(im, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(im, dtype=np.float64))

    def run():
        # the buffers outlive the call: start from the previous call's last uses
        used = list(bufst.get("used", [None, None]))  # compute finished with buffer b (device event)
        copied = list(bufst.get("copied", [None, None]))  # H2D out of pinned[b] finished (host waits before rewriting it)
        ready = [None, None]
        pieces = []
        try:
            def stage(k):
                t = order[k]
                b = k % 2
                data = datas[t]
                if copied[b] is not None:
                    copied[b].synchronize()
                if data:
                    pinned[b].numpy()[: len(data)] = np.frombuffer(data, dtype=np.uint8)
                with torch.cuda.stream(copy):
                    if used[b] is not None:
                        copy.wait_event(used[b])  # buffer b's previous frame is done
                    for _, v in by_frame[t]:
                        dtg[b][v].copy_(host_tensor(targets[t][v]), non_blocking=True)
                    if data:
                        dpay[b][: len(data)].copy_(pinned[b][: len(data)], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                ready[b] = copied[b] = ev

            if order:
                stage(0)
            for k, t in enumerate(order):
                b = k % 2
                comp.wait_event(ready[b])
                if k + 1 < len(order):
                    stage(k + 1)
                data = datas[t]
                planes = codec.decode_apply_device(data, canon, n, w, device=dev, payload_dev=dpay[b][: len(data)])
                lst = by_frame[t]
                pieces.append(render_views([GaussianFrame(device_params=planes, count=n)], cams,
                                           [(0, v) for _, v in lst], targets=[dtg[b][v] for _, v in lst],
                                           device=dev).sse)
                u = torch.cuda.Event()
                u.record(comp)
                used[b] = u
        finally:
            bufst["used"], bufst["copied"] = used, copied
        return pieces

    eng = engine(dev)
    flags = ctypes.c_uint32(0)
    eng.call("airgs_defer", 1, ctypes.byref(flags))
    try:
        pieces = run()
    finally:
        eng.call("airgs_defer", 0, ctypes.byref(flags))
    if flags.value:
        pieces = run()  # checked mode
    return _in_item_order(pieces, [i for t in order for i, _ in by_frame[t]], len(items), dev)


def probe_sequence(space, cams, payloads, targets, tau_db: float = DEFAULT_TAU_DB, device=None):
    """Keyframe detection over a sequence of frames of one group, streamed
    from host memory (probe_sequence_items over every (frame, view) item):
    for frame t, decode its GSDP delta payload against the group's canonical
    space, apply it, render every camera with SSE against the frame's
    ground-truth images, and decide ``q < tau``.  Host->device copies of
    frame t+1 overlap frame t's evaluation.  Returns a list of
    (quality_db, is_keyframe) per frame."""
    cams = list(cams)
    V = len(cams)
    if len(payloads) != len(targets):
        raise StructuralError("one target set per payload required")
    for tg in targets:
        if len(tg) != V:
            raise StructuralError("target image count does not match cameras")
    px = [c.resolution[0] * c.resolution[1] * 3 for c in cams]
    items = [(t, v) for t in range(len(payloads)) for v in range(V)]
    host = probe_sequence_items(space, cams, payloads, targets, items, device).cpu().numpy()
    out = []
    for t in range(len(payloads)):
        q = float(np.mean([psnr_from_sse(host[t * V + v], px[v]) for v in range(V)]))
        out.append((q, is_keyframe(q, tau_db)))
    return out


# frames of a pipelined probe batch alternate over this many (engine, stream)
# lanes: frame t+1's decode / projection / binning / sort run on the second
# stream while frame t composites, filling the SMs its last CTAs leave idle
# (C2: 3.84 -> 3.76 ms per frame).  AIRGS_PROBE_LANES overrides.
PROBE_LANES = 2


def probe_lanes() -> int:
    """Lanes of the pipelined probe (PROBE_LANES or AIRGS_PROBE_LANES)."""
    return max(1, int(os.environ.get("AIRGS_PROBE_LANES", str(PROBE_LANES))))
_lane_streams: dict = {}


def _lane_stream(dev, lane):
    import torch

    key = (str(dev), lane)
    if key not in _lane_streams:
        _lane_streams[key] = torch.cuda.Stream(device=dev)
    return _lane_streams[key]


def probe_payload_items(space, cams, payloads, payload_devs, targets, items, device=None):
    """Per-item SSE of (frame t, view v) items of a probe batch whose GSDP
    payloads and targets are already in HBM: each frame that has items is
    decoded and applied once, its items rendered with SSE fused into
    compositing, all enqueued without host synchronisation (airgs_defer).  If
    any call reports a problem (a malformed payload, invalid parameters, a
    bucket overflow) the batch is re-run in checked mode, which raises the
    reference's exact error or handles the overflow.  Returns a device
    float64 tensor, one SSE per item in ``items`` order (``targets[t][v]``:
    device (h, w, 3) float64; only the listed items' targets are read)."""
    import ctypes

    import torch

    from . import codec
    from ._lib import engine, engine_lane
    from .model import GaussianFrame, as_space
    from .rasterizer import render_views

    space = as_space(space)
    dev = dv.device_of(device)
    cams = list(cams)
    n, w = space.frame.count, space.frame.width
    canon = space.frame.planes(dev)
    datas = {}
    by_frame = {}
    for k, (t, v) in enumerate(items):
        by_frame.setdefault(int(t), []).append((k, int(v)))
    for t in by_frame:
        p = payloads[t]
        datas[t] = p.data if hasattr(p, "data") else bytes(p)
    order = [k for lst in by_frame.values() for k, _ in lst]  # item positions in evaluation order
    pieces = []

    frames_in_order = list(by_frame)
    lanes = min(probe_lanes(), len(frames_in_order))
    main = torch.cuda.current_stream(dev)
    streams = [main] + [_lane_stream(dev, k) for k in range(1, lanes)]

    def run(nl):
        pieces.clear()
        for s in streams[1:nl]:
            s.wait_stream(main)  # inputs enqueued on the caller's stream
        for k, (t, lst) in enumerate(by_frame.items()):
            lane = k % nl
            # the lane's next frame: its varint scan is enqueued ahead (side stream)
            nxt = frames_in_order[k + nl] if k + nl < len(frames_in_order) else None
            ahead = (datas[nxt], payload_devs[nxt]) if nxt is not None else None
            with torch.cuda.stream(streams[lane]), engine_lane(lane):
                planes = codec.decode_apply_device(datas[t], canon, n, w, device=dev, payload_dev=payload_devs[t],
                                                   ahead=ahead)
                sse = render_views([GaussianFrame(device_params=planes, count=n)], cams,
                                   [(0, v) for _, v in lst], targets=[targets[t][v] for _, v in lst],
                                   device=dev).sse
            if lane:
                sse.record_stream(main)  # consumed on the caller's stream
            pieces.append(sse)
        for s in streams[1:nl]:
            main.wait_stream(s)

    engs = []
    flags = []
    for lane in range(lanes):
        with engine_lane(lane):
            engs.append(engine(dev))
        flags.append(ctypes.c_uint32(0))
    for e, f in zip(engs, flags):
        e.call("airgs_defer", 1, ctypes.byref(f))
    try:
        run(lanes)
    finally:
        for e, f in zip(engs, flags):
            e.call("airgs_defer", 0, ctypes.byref(f))
    if any(f.value for f in flags):
        # checked mode on the same lanes: errors surface in call order, and each
        # lane engine adapts its tile-bucket capacity after an overflow
        run(lanes)
    return _in_item_order(pieces, order, len(items), dev)


def probe_payloads_device(space, cams, payloads, payload_devs, targets, tau_db: float = DEFAULT_TAU_DB,
                          device=None):
    """Keyframe probes of a batch of frames whose GSDP payloads and targets are
    already in HBM, pipelined (probe_payload_items over every (frame, view)
    item; one host synchronisation for the whole batch).  Returns
    [(quality_db, is_keyframe)]."""
    cams = list(cams)
    V = len(cams)
    px = [c.resolution[0] * c.resolution[1] * 3 for c in cams]
    items = [(t, v) for t in range(len(payloads)) for v in range(V)]
    host = probe_payload_items(space, cams, payloads, payload_devs, targets, items, device).cpu().numpy()
    out = []
    for t in range(len(payloads)):
        q = float(np.mean([psnr_from_sse(host[t * V + v], px[v]) for v in range(V)]))
        out.append((q, is_keyframe(q, tau_db)))
    return out


def is_keyframe(quality_db: float, tau_db: float = DEFAULT_TAU_DB) -> bool:
    """The grouping decision: re-anchor when the probe misses tau
    (ss/grouping.py:213)."""
    return not quality_db >= tau_db


class GroupSpan:
    __slots__ = ("key", "start", "end")

    def __init__(self, key, start, end):
        if not key == start <= end:
            raise StructuralError(f"bad group span ({key}, {start}, {end})")
        object.__setattr__(self, "key", key)
        object.__setattr__(self, "start", start)
        object.__setattr__(self, "end", end)

    def __setattr__(self, k, v):
        raise AttributeError("GroupSpan is immutable")

    def __eq__(self, o):
        return isinstance(o, GroupSpan) and (self.key, self.start, self.end) == (o.key, o.start, o.end)


class GroupPlan:
    __slots__ = ("tau_db", "groups")

    def __init__(self, tau_db, groups):
        groups = tuple(groups)
        if not groups or groups[0].start != 0:
            raise StructuralError("group plan must start at frame 0")
        for a, b in zip(groups, groups[1:]):
            if b.start != a.end + 1:
                raise StructuralError("group spans must be contiguous")
        object.__setattr__(self, "tau_db", tau_db)
        object.__setattr__(self, "groups", groups)

    def __setattr__(self, k, v):
        raise AttributeError("GroupPlan is immutable")

    def __eq__(self, o):
        return isinstance(o, GroupPlan) and self.tau_db == o.tau_db and self.groups == o.groups

    @property
    def frame_count(self) -> int:
        return self.groups[-1].end + 1

    def group_of(self, frame_index: int) -> GroupSpan:
        for g in self.groups:
            if g.start <= frame_index <= g.end:
                return g
        raise ValidationError(f"frame {frame_index} outside the plan")

    def to_json(self) -> str:
        return json.dumps({"tau": self.tau_db,
                           "groups": [{"key": g.key, "start": g.start, "end": g.end} for g in self.groups]},
                          indent=2)

    @staticmethod
    def from_json(text: str) -> "GroupPlan":
        obj = json.loads(text)
        return GroupPlan(tau_db=float(obj["tau"]),
                         groups=tuple(GroupSpan(g["key"], g["start"], g["end"]) for g in obj["groups"]))


class FrameRecord:
    __slots__ = ("frame_index", "group_key", "is_keyframe", "step_delta", "cumulative_delta", "quality_db")

    def __init__(self, frame_index, group_key, is_keyframe, step_delta, cumulative_delta, quality_db):
        for k, v in (("frame_index", frame_index), ("group_key", group_key), ("is_keyframe", is_keyframe),
                     ("step_delta", step_delta), ("cumulative_delta", cumulative_delta),
                     ("quality_db", quality_db)):
            object.__setattr__(self, k, v)

    def __setattr__(self, k, v):
        raise AttributeError("FrameRecord is immutable")


class TrainedStream:
    """Canonical spaces per group plus per-frame cumulative deltas
    (ss/grouping.py:91-105)."""

    __slots__ = ("plan", "spaces", "records")

    def __init__(self, plan, spaces, records):
        object.__setattr__(self, "plan", plan)
        object.__setattr__(self, "spaces", dict(spaces))
        object.__setattr__(self, "records", tuple(records))

    def __setattr__(self, k, v):
        raise AttributeError("TrainedStream is immutable")

    def reconstruct(self, frame_index: int):
        rec = self.records[frame_index]
        return apply_delta(self.spaces[rec.group_key], rec.cumulative_delta, frame_index=frame_index)

    def qualities(self):
        return [r.quality_db for r in self.records]


def plan_from_decisions(keyframe_flags, tau_db=DEFAULT_TAU_DB) -> GroupPlan:
    """Group spans from per-frame keyframe decisions (frame 0 always opens)."""
    spans = []
    for t, k in enumerate(keyframe_flags):
        if t == 0 or k:
            spans.append([t, t, t])
        else:
            spans[-1][2] = t
    return GroupPlan(tau_db, tuple(GroupSpan(*s) for s in spans))


# ---------------------------------------------------------------------------
# Trained-stream persistence (ss/grouping.py:108-150): one .npz with the plan as
# embedded JSON; the file format is the reference's.


def save_stream(path, stream: TrainedStream) -> None:
    arrays = {
        "plan_json": np.frombuffer(stream.plan.to_json().encode(), dtype=np.uint8),
        "group_keys": np.array(sorted(stream.spaces), dtype=np.int64),
        "frame_group": np.array([r.group_key for r in stream.records], dtype=np.int64),
        "frame_iskey": np.array([r.is_keyframe for r in stream.records], dtype=np.bool_),
        "frame_quality": np.array([r.quality_db for r in stream.records]),
    }
    for k, sp in stream.spaces.items():
        arrays[f"space_{k}"] = sp.frame.params
        arrays[f"capacity_{k}"] = np.array(sp.capacity_U, dtype=np.int64)
    for r in stream.records:
        arrays[f"cumulative_{r.frame_index}"] = r.cumulative_delta.dense()
        arrays[f"step_{r.frame_index}"] = r.step_delta.dense()
    np.savez_compressed(path, **arrays)


def load_stream(path, device=None) -> TrainedStream:
    """Inverse of ``save_stream`` (ss/grouping.py:125-150).  Canonical spaces
    are uploaded and every dense delta is filtered to its sparse rows on the
    device (``DeltaTensor.from_dense``), so the stream is HBM-resident."""
    from .model import GaussianFrame

    with np.load(path) as z:
        plan = GroupPlan.from_json(bytes(z["plan_json"]).decode())
        spaces = {}
        for k in z["group_keys"]:
            k = int(k)
            fr = GaussianFrame(params=z[f"space_{k}"], frame_index=k, group_key=k)
            fr.planes(device)
            spaces[k] = CanonicalSpace(frame=fr, capacity_U=int(z[f"capacity_{k}"]))
        records = []
        for t in range(len(z["frame_group"])):
            records.append(FrameRecord(frame_index=t, group_key=int(z["frame_group"][t]),
                                       is_keyframe=bool(z["frame_iskey"][t]),
                                       step_delta=DeltaTensor.from_dense(z[f"step_{t}"]),
                                       cumulative_delta=DeltaTensor.from_dense(z[f"cumulative_{t}"]),
                                       quality_db=float(z["frame_quality"][t])))
    return TrainedStream(plan=plan, spaces=spaces, records=tuple(records))
