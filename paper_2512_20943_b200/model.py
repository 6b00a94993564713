"""Domain types of the evaluation path: frames, canonical spaces and sparse
deltas -- the reference's public API (``ss/model.py:125-311``) backed by HBM.

Each ``GaussianFrame`` / ``DeltaTensor`` may hold its data on the host (the
reference representation: an ``(n, width)`` float64 array, a dict of rows),
on the device (``device.py`` layouts), or both.  The other representation is
produced lazily on first use, so a chain such as
``decode_delta -> compose_deltas -> apply_delta -> render`` never leaves HBM,
while a caller that reads ``frame.params`` or ``delta.entries`` still gets
exactly the reference's objects.

Parameter row layout (unchanged): position(3) | quaternion(4) | log-scale(3) |
opacity-logit(1) | colour-logit(3) | SH (3 or 12).
"""

from __future__ import annotations

import numpy as np

from . import device as dv
from .errors import StructuralError, ValidationError

POS = slice(0, 3)
QUAT = slice(3, 7)
LOG_SCALE = slice(7, 10)
OPACITY = 10
COLOR = slice(11, 14)
SH_START = 14
EPS_SPARSE = 1e-9  # ss/model.py:35
SCENE_MAGIC = b"GSSC"  # ss/model.py:42-43
SCENE_VERSION = 1
TOMBSTONE_LOGIT = -100.0
LIVE_LOGIT_FLOOR = -50.0

_WIDTHS = {17: 0, 26: 1}


def sh_dim(degree: int) -> int:
    if degree not in (0, 1):
        raise ValidationError(f"sh degree must be 0 or 1, got {degree}")
    return 3 * (degree + 1) ** 2


def param_dim(degree: int) -> int:
    return SH_START + sh_dim(degree)


def degree_from_param_dim(dim: int) -> int:
    try:
        return _WIDTHS[int(dim)]
    except KeyError:
        raise StructuralError(f"no sh degree yields parameter width {dim}") from None


def sigmoid(x):
    return 0.5 * (1.0 + np.tanh(0.5 * np.asarray(x, dtype=np.float64)))


def logit(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


def _engine(dev=None):
    from ._lib import engine

    return engine(dev)


def _ptr(t):
    from ._lib import ptr

    return ptr(t)


# ---------------------------------------------------------------------------


class GaussianFrame:
    """Ordered primitive set of one frame in parameter space."""

    __slots__ = ("_host", "_dev", "_count", "_width", "frame_index", "group_key")

    def __init__(self, params=None, frame_index: int = 0, group_key: int = 0, *, device_params=None,
                 count=None):
        if frame_index < 0:
            raise StructuralError("frame_index must be non-negative")
        object.__setattr__(self, "frame_index", int(frame_index))
        object.__setattr__(self, "group_key", int(group_key))
        if device_params is not None:
            width = int(device_params.shape[0])
            degree_from_param_dim(width)
            object.__setattr__(self, "_dev", device_params)
            object.__setattr__(self, "_host", None)
            object.__setattr__(self, "_count", int(count))
            object.__setattr__(self, "_width", width)
            return
        p = np.asarray(params, dtype=np.float64)
        if p.ndim != 2:
            raise StructuralError("params must be (n, param_dim)")
        degree_from_param_dim(p.shape[1])
        p = np.array(p, dtype=np.float64, order="C")  # private copy
        p.setflags(write=False)
        object.__setattr__(self, "_host", p)
        object.__setattr__(self, "_dev", None)
        object.__setattr__(self, "_count", p.shape[0])
        object.__setattr__(self, "_width", p.shape[1])

    def __setattr__(self, k, v):
        raise AttributeError("GaussianFrame is immutable")

    # -- representations
    @property
    def params(self) -> np.ndarray:
        if self._host is None:
            h = dv.download_params(self._dev, self._count)
            h.setflags(write=False)
            object.__setattr__(self, "_host", h)
        return self._host

    def planes(self, device=None):
        """Plane-major device parameters ``(width, ld)`` (uploaded once)."""
        dev = dv.device_of(device)
        if self._dev is None or self._dev.device != dev:
            if self._dev is not None and self._host is None:
                return self._dev.to(dev)
            object.__setattr__(self, "_dev", dv.upload_params(self._host, dev))
        return self._dev

    @property
    def on_device(self) -> bool:
        return self._dev is not None

    @property
    def count(self) -> int:
        return self._count

    @property
    def sh_degree(self) -> int:
        return degree_from_param_dim(self._width)

    @property
    def width(self) -> int:
        return self._width

    def live_mask(self) -> np.ndarray:
        return self.params[:, OPACITY] > LIVE_LOGIT_FLOOR

    def live_count(self) -> int:
        if self._host is None and self._dev is not None:
            return int((self._dev[OPACITY, : self._count] > LIVE_LOGIT_FLOOR).sum().item())
        return int(np.count_nonzero(self.live_mask()))

    def with_params(self, params, frame_index=None, group_key=None) -> "GaussianFrame":
        return GaussianFrame(params=params,
                             frame_index=self.frame_index if frame_index is None else frame_index,
                             group_key=self.group_key if group_key is None else group_key)

    def __repr__(self):
        where = "device" if self._host is None else "host"
        return f"GaussianFrame(n={self._count}, width={self._width}, frame={self.frame_index}, {where})"


class CanonicalSpace:
    """A keyframe's primitive set: the anchor every delta of its group is
    applied to (ss/model.py:188-203)."""

    __slots__ = ("frame", "capacity_U")

    def __init__(self, frame: GaussianFrame, capacity_U: int):
        if frame.frame_index != frame.group_key:
            raise StructuralError("a keyframe must anchor itself")
        if capacity_U < frame.live_count():
            raise StructuralError("capacity_U below live primitive count")
        object.__setattr__(self, "frame", frame)
        object.__setattr__(self, "capacity_U", int(capacity_U))

    def __setattr__(self, k, v):
        raise AttributeError("CanonicalSpace is immutable")

    @property
    def key_index(self) -> int:
        return self.frame.frame_index


class DeltaTensor:
    """Sparse per-primitive parameter differences (a commutative monoid under
    ``compose_deltas``).  ``entries`` is the reference's dict view."""

    __slots__ = ("base_count", "param_width", "_entries", "_ov")

    def __init__(self, base_count: int, param_width: int, entries=None, *, overlay=None):
        object.__setattr__(self, "base_count", int(base_count))
        object.__setattr__(self, "param_width", int(param_width))
        if overlay is not None:
            object.__setattr__(self, "_entries", None)
            object.__setattr__(self, "_ov", overlay)
            return
        frozen = {}
        for idx, block in (entries or {}).items():
            idx = int(idx)
            if not 0 <= idx < self.base_count:
                raise StructuralError(f"delta index {idx} out of range")
            b = np.asarray(block, dtype=np.float64)
            if b.shape != (self.param_width,):
                raise StructuralError("delta block width mismatch")
            if not np.all(np.isfinite(b)):
                raise ValidationError(f"non-finite delta component at {idx}")
            b = b.copy()
            b.setflags(write=False)
            frozen[idx] = b
        object.__setattr__(self, "_entries", frozen)
        object.__setattr__(self, "_ov", None)

    def __setattr__(self, k, v):
        raise AttributeError("DeltaTensor is immutable")

    # -- representations
    @property
    def entries(self) -> dict:
        if self._entries is None:
            idx, rows = self._ov.entries()
            d = {}
            for i, r in zip(idx.tolist(), rows):
                r = r.copy()
                r.setflags(write=False)
                d[int(i)] = r
            object.__setattr__(self, "_entries", d)
        return self._entries

    def overlay(self, device=None) -> dv.Overlay:
        dev = dv.device_of(device)
        if self._ov is None or self._ov.rows.device != dev:
            idx = np.array(sorted(self._entries), dtype=np.int64)
            rows = (np.stack([self._entries[i] for i in idx.tolist()]) if idx.size
                    else np.zeros((0, self.param_width)))
            object.__setattr__(self, "_ov", dv.Overlay.from_entries(idx, rows, self.base_count,
                                                                   self.param_width, dev))
        return self._ov

    @property
    def entry_count(self) -> int:
        if self._entries is not None:
            return len(self._entries)
        return self._ov.count()

    def is_empty(self) -> bool:
        return self.entry_count == 0

    def indices(self) -> np.ndarray:
        if self._entries is not None:
            return np.array(sorted(self._entries), dtype=np.int64)
        return self._ov.entries()[0]

    def negate(self) -> "DeltaTensor":
        if self._ov is None and self.base_count == 0:
            return DeltaTensor(0, self.param_width, {})
        return _compose_overlays([(self, -1.0)], apply_eps=False, eps=EPS_SPARSE)

    def dense(self) -> np.ndarray:
        out = np.zeros((self.base_count, self.param_width), dtype=np.float64)
        for i, b in self.entries.items():
            out[i] = b
        return out

    def l1_norm(self) -> float:
        return float(sum(np.abs(b).sum() for b in self.entries.values()))

    @staticmethod
    def empty(base_count: int, param_width: int) -> "DeltaTensor":
        return DeltaTensor(base_count=base_count, param_width=param_width)

    @staticmethod
    def from_dense(dense, eps: float = EPS_SPARSE) -> "DeltaTensor":
        """Rows with max|.| > eps, computed on device (ss/model.py:262-266)."""
        dense = np.asarray(dense, dtype=np.float64)
        n, w = dense.shape
        if n == 0:
            return DeltaTensor(0, w, {})
        planes = dv.upload_params(dense)
        return _filter_planes(planes, n, w, eps)

    def __repr__(self):
        where = "device" if self._entries is None else "host"
        return f"DeltaTensor(base_count={self.base_count}, width={self.param_width}, {where})"


# ---------------------------------------------------------------------------
# coercion of reference objects (duck typing) for the drop-in


def as_frame(x) -> GaussianFrame:
    if isinstance(x, GaussianFrame):
        return x
    return GaussianFrame(params=x.params, frame_index=getattr(x, "frame_index", 0),
                         group_key=getattr(x, "group_key", 0))


def as_delta(x) -> DeltaTensor:
    if isinstance(x, DeltaTensor):
        return x
    return DeltaTensor(x.base_count, x.param_width, dict(x.entries))


def as_space(x) -> CanonicalSpace:
    if isinstance(x, CanonicalSpace):
        return x
    return CanonicalSpace(as_frame(x.frame), x.capacity_U)


# ---------------------------------------------------------------------------
# device-backed algebra


def _filter_planes(planes, n, w, eps, sign=1.0):
    """Dense planes -> overlay of rows with max|.| > eps."""
    import torch

    eng = _engine(planes.device)
    ones = torch.ones((planes.shape[1],), dtype=torch.uint8, device=planes.device)
    out = dv.Overlay.empty(n, w, planes.device)
    _compose_call(eng, [(planes, ones, sign)], n, w, planes.shape[1], eps, True, out)
    return DeltaTensor(n, w, overlay=out)


def _compose_call(eng, parts, n, w, ld, eps, apply_eps, out):
    import ctypes

    from ._lib import vp

    k = len(parts)
    rows = (vp * k)(*[vp(p[0].data_ptr()) for p in parts])
    pres = (vp * k)(*[vp(p[1].data_ptr()) for p in parts])
    signs = (ctypes.c_double * k)(*[float(p[2]) for p in parts])
    eng.call("airgs_delta_compose", k, rows, pres, signs, n, w, ld, float(eps), 1 if apply_eps else 0,
             _ptr(out.rows), _ptr(out.present), eng.stream())


def _compose_overlays(items, apply_eps=True, eps=EPS_SPARSE) -> DeltaTensor:
    """items: list of (DeltaTensor, sign), all over the same base."""
    first = items[0][0]
    n, w = first.base_count, first.param_width
    dev = dv.device_of(None)
    ovs = [(d.overlay(dev), s) for d, s in items]
    eng = _engine(dev)
    ld = dv.ld_for(n)
    out = dv.Overlay.empty(n, w, dev)
    if n == 0:
        return DeltaTensor(n, w, overlay=out)
    pending = [(o.rows, o.present, s) for o, s in ovs]
    # the C-ABI composes <= 8 overlays per call; chain unfiltered partial sums
    while len(pending) > 8:
        part = dv.Overlay.empty(n, w, dev)
        _compose_call(eng, pending[:8], n, w, ld, eps, False, part)
        pending = [(part.rows, part.present, 1.0)] + pending[8:]
    _compose_call(eng, pending, n, w, ld, eps, apply_eps, out)
    return DeltaTensor(n, w, overlay=out)


def compose_deltas(deltas, eps: float = EPS_SPARSE) -> DeltaTensor:
    """Componentwise sum over the union of indices, in list order, with one
    |.|max > eps filter at the end (ss/model.py:294-311)."""
    deltas = [as_delta(d) for d in deltas]
    if not deltas:
        return DeltaTensor.empty(0, param_dim(0))
    base, width = deltas[0].base_count, deltas[0].param_width
    for d in deltas:
        if d.base_count != base or d.param_width != width:
            raise StructuralError("cannot compose deltas over different bases")
    if base == 0:
        return DeltaTensor(0, width, {})
    return _compose_overlays([(d, 1.0) for d in deltas], apply_eps=True, eps=eps)


def apply_delta(space: CanonicalSpace, delta: DeltaTensor, frame_index=None) -> GaussianFrame:
    """canonical + delta rows (ss/model.py:269-284), on device."""
    space, delta = as_space(space), as_delta(delta)
    fr = space.frame
    if delta.base_count != fr.count:
        raise StructuralError(f"delta base_count {delta.base_count} != space count {fr.count}")
    if delta.param_width != fr.width:
        raise StructuralError("delta parameter width mismatch")
    key = space.key_index
    fi = key if frame_index is None else frame_index
    if fr.count == 0:
        return GaussianFrame(params=np.zeros((0, fr.width)), frame_index=fi, group_key=key)
    planes = apply_overlay(fr.planes(), fr.count, delta.overlay(fr.planes().device))
    return GaussianFrame(device_params=planes, count=fr.count, frame_index=fi, group_key=key)


def apply_overlay(canon, n, ov_a, sel=None, rank=None, keep_min=0, ov_b=None):
    """Device apply with the optional pruning-level selector (see
    airgs_delta_apply in include/airgs_b200.h)."""
    import torch

    eng = _engine(canon.device)
    out = torch.empty_like(canon)
    if canon.shape[1] > n:
        out[:, n:].zero_()
    eng.call("airgs_delta_apply", _ptr(canon), _ptr(ov_a.rows if ov_a else None),
             _ptr(ov_a.present if ov_a else None), _ptr(sel), _ptr(rank), int(keep_min),
             _ptr(ov_b.rows if ov_b else None), _ptr(ov_b.present if ov_b else None), n, canon.shape[0],
             canon.shape[1], _ptr(out), eng.stream())
    return out


def diff_frames(a: GaussianFrame, b: GaussianFrame, eps: float = EPS_SPARSE) -> DeltaTensor:
    """Delta with apply_delta(a) == b exactly where kept (ss/model.py:287-291)."""
    a, b = as_frame(a), as_frame(b)
    if a.count != b.count or a.width != b.width:
        raise StructuralError("frames must share primitive count and layout")
    n, w = a.count, a.width
    if n == 0:
        return DeltaTensor(0, w, {})
    import torch

    pa, pb = a.planes(), b.planes(a.planes().device)
    ones = torch.ones((pa.shape[1],), dtype=torch.uint8, device=pa.device)
    out = dv.Overlay.empty(n, w, pa.device)
    # b + (-a) == b - a exactly in IEEE arithmetic
    _compose_call(_engine(pa.device), [(pb, ones, 1.0), (pa, ones, -1.0)], n, w, pa.shape[1], eps, True, out)
    return DeltaTensor(n, w, overlay=out)


def quat_to_matrix(q: np.ndarray) -> np.ndarray:
    """Host helper kept for API parity (the device path has its own)."""
    w, x, y, z = (q[..., k] for k in range(4))
    m = np.empty(q.shape[:-1] + (3, 3), dtype=np.float64)
    m[..., 0, :] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1)
    m[..., 1, :] = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1)
    m[..., 2, :] = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)
    return m


# ---------------------------------------------------------------------------
# Scene container I/O ("GSSC", ss/model.py:318-350): little-endian, header then
# packed f64 rows.  The file format is the reference's, byte for byte.


def save_scene(path, frames) -> None:
    import struct

    frames = list(frames)
    if not frames:
        raise StructuralError("cannot save an empty scene")
    degree = frames[0].sh_degree
    with open(path, "wb") as fh:
        fh.write(SCENE_MAGIC)
        fh.write(struct.pack("<HIB", SCENE_VERSION, len(frames), degree))
        for fr in frames:
            if fr.sh_degree != degree:
                raise StructuralError("mixed sh degrees in one scene")
            fh.write(struct.pack("<I", fr.count))
            fh.write(fr.params.astype("<f8").tobytes())


def load_scene(path, device=None, to_device: bool = False):
    """Frames of a GSSC file (ss/model.py:332-350).  ``to_device=True``
    streams the whole file into HBM with one copy and builds every frame's
    plane-major parameters there (airgs_rows_to_planes: rows start at an odd
    byte offset), so the frames are device-resident without a host transpose."""
    import struct

    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != SCENE_MAGIC:
        raise ValidationError(f"bad scene magic {data[:4]!r}")
    if len(data) < 11:
        raise ValidationError("truncated scene file")
    version, frame_count, degree = struct.unpack_from("<HIB", data, 4)
    if version != SCENE_VERSION:
        raise ValidationError(f"unsupported scene version {version}")
    width = param_dim(degree)
    spans = []
    pos = 11
    for _ in range(frame_count):
        if pos + 4 > len(data):
            raise ValidationError("truncated scene file")
        (n,) = struct.unpack_from("<I", data, pos)
        pos += 4
        nbytes = 8 * n * width
        if pos + nbytes > len(data):
            raise ValidationError("truncated scene file")
        spans.append((pos, n))
        pos += nbytes
    if not to_device:
        return [GaussianFrame(params=np.frombuffer(data, dtype="<f8", count=n * width, offset=off).reshape(n, width),
                              frame_index=t, group_key=0) for t, (off, n) in enumerate(spans)]
    import torch

    dev = dv.device_of(device)
    eng = _engine(dev)
    raw = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev)
    frames = []
    for t, (off, n) in enumerate(spans):
        planes = torch.zeros((width, dv.ld_for(n)), dtype=torch.float64, device=dev)
        eng.call("airgs_rows_to_planes", _ptr(raw), off, n, width, _ptr(planes), planes.shape[1], eng.stream())
        frames.append(GaussianFrame(device_params=planes, count=n, frame_index=t, group_key=0))
    return frames
