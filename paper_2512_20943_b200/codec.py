"""Wire formats of the streaming path (``ss/codec.py``), decoded and encoded
on the GPU.

* GSAI ("attribute images"): 25-byte header, then per attribute plane
  ``(scale f64, offset f64)`` + ``w*h`` little-endian u16 pixels; pixel i of
  every plane belongs to primitive i.
* GSDP ("delta payload"): 24-byte header ``<4sIIId`` (magic, frame_index,
  base_key, entry_count, quant_step), ``entry_count`` gap varints, then
  ``entry_count * width`` little-endian i32 fixed-point components.

Only header fields are parsed on the host (validation and routing); every
byte of plane / varint / row data is produced or consumed by the
airgs_b200 kernels.
"""

from __future__ import annotations

import ctypes
import math
import struct

import numpy as np

from . import device as dv
from .errors import CapacityError, DecodeError, StructuralError
from .model import DeltaTensor, GaussianFrame, as_delta, as_frame, degree_from_param_dim

IMAGE_MAGIC = b"GSAI"
IMAGE_VERSION = 1
DELTA_MAGIC = b"GSDP"
BIT_DEPTH = 16
QMAX = (1 << BIT_DEPTH) - 1

_IMAGE_HEADER = struct.Struct("<4sHIHHHB")  # magic, version, n, m, w, h, bit_depth
_DELTA_HEADER = struct.Struct("<4sIIId")  # magic, frame_index, base_key, entry_count, quant_step
DELTA_HEADER_BYTES = _DELTA_HEADER.size
IMAGE_HEADER_BYTES = _IMAGE_HEADER.size + 8


def _engine(device=None):
    from ._lib import engine

    return engine(device)


def _ptr(t):
    from ._lib import ptr

    return ptr(t)


def _to_device_bytes(data: bytes, device=None):
    import torch

    dev = dv.device_of(device)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else torch.zeros(0, dtype=torch.uint8)
    return host.to(dev)


# ---------------------------------------------------------------------------
# varints (host helpers of the public API; the device path has its own)


def encode_varint(value: int) -> bytes:
    if value < 0:
        raise StructuralError(f"cannot varint-encode negative value {value}")
    out = bytearray()
    while True:
        low = value & 0x7F
        value >>= 7
        if value:
            out.append(low | 0x80)
        else:
            out.append(low)
            return bytes(out)


def decode_varint(data: bytes, offset: int = 0) -> tuple:
    value, shift, pos = 0, 0, offset
    while True:
        if pos >= len(data):
            raise DecodeError("truncated varint")
        byte = data[pos]
        pos += 1
        value |= (byte & 0x7F) << shift
        if byte < 0x80:
            return value, pos
        shift += 7
        if shift > 63:
            raise DecodeError("varint too long")


# ---------------------------------------------------------------------------
# GSAI


class AttributeImageSet:
    """Multi-channel 2D-image encoding of one frame.  Backed by the raw
    container bytes and/or the (m, h, w) u16 planes."""

    __slots__ = ("_images", "scales", "offsets", "count", "frame_index", "group_key", "bit_depth", "_blob", "_hw",
                 "_dev")

    def __init__(self, images=None, scales=None, offsets=None, count=0, frame_index=0, group_key=0,
                 bit_depth=BIT_DEPTH, *, blob=None, hw=None):
        object.__setattr__(self, "_images", None if images is None else np.asarray(images, dtype=np.uint16))
        object.__setattr__(self, "scales", np.asarray(scales, dtype=np.float64))
        object.__setattr__(self, "offsets", np.asarray(offsets, dtype=np.float64))
        object.__setattr__(self, "count", int(count))
        object.__setattr__(self, "frame_index", int(frame_index))
        object.__setattr__(self, "group_key", int(group_key))
        object.__setattr__(self, "bit_depth", int(bit_depth))
        object.__setattr__(self, "_blob", blob)
        object.__setattr__(self, "_hw", hw if hw is not None else (None if images is None else
                                                                  tuple(self._images.shape[1:])))
        object.__setattr__(self, "_dev", None)

    def __setattr__(self, k, v):
        raise AttributeError("AttributeImageSet is immutable")

    @property
    def images(self) -> np.ndarray:
        if self._images is None:
            m = self.scales.shape[0]
            h, w = self._hw
            out = np.empty((m, h, w), dtype=np.uint16)
            pos = IMAGE_HEADER_BYTES
            for j in range(m):
                out[j] = np.frombuffer(self._blob, dtype="<u2", count=w * h, offset=pos + 16).reshape(h, w)
                pos += 16 + 2 * w * h
            object.__setattr__(self, "_images", out)
        return self._images

    @property
    def width(self) -> int:
        return self._hw[1]

    @property
    def height(self) -> int:
        return self._hw[0]

    @property
    def num_attributes(self) -> int:
        return self.scales.shape[0]

    def to_bytes(self) -> bytes:
        if self._blob is not None:
            return self._blob
        m = self.num_attributes
        h, w = self._hw
        parts = [_IMAGE_HEADER.pack(IMAGE_MAGIC, IMAGE_VERSION, self.count, m, w, h, self.bit_depth),
                 struct.pack("<II", self.frame_index, self.group_key)]
        imgs = self.images
        for j in range(m):
            parts.append(struct.pack("<dd", self.scales[j], self.offsets[j]))
            parts.append(imgs[j].astype("<u2").tobytes())
        blob = b"".join(parts)
        object.__setattr__(self, "_blob", blob)
        return blob

    def device_blob(self, device=None):
        dev = dv.device_of(device)
        if self._dev is None or self._dev.device != dev:
            object.__setattr__(self, "_dev", _to_device_bytes(self.to_bytes(), dev))
        return self._dev

    @staticmethod
    def from_bytes(data: bytes) -> "AttributeImageSet":
        data = bytes(data)
        if len(data) < _IMAGE_HEADER.size:
            raise DecodeError("attribute image container too short")
        magic, version, n, m, w, h, depth = _IMAGE_HEADER.unpack_from(data, 0)
        if magic != IMAGE_MAGIC:
            raise DecodeError(f"bad attribute-image magic {magic!r}")
        if version != IMAGE_VERSION or depth != BIT_DEPTH:
            raise DecodeError("unsupported attribute-image version or bit depth")
        if len(data) < IMAGE_HEADER_BYTES and m:
            raise DecodeError("truncated attribute image container")
        frame_index, group_key = struct.unpack_from("<II", data, _IMAGE_HEADER.size) if len(data) >= 25 else (0, 0)
        scales = np.empty(m)
        offsets = np.empty(m)
        pos = IMAGE_HEADER_BYTES
        plane = 2 * w * h
        for j in range(m):
            if pos + 16 + plane > len(data):
                raise DecodeError("truncated attribute image container")
            scales[j], offsets[j] = struct.unpack_from("<dd", data, pos)
            pos += 16 + plane
        return AttributeImageSet(scales=scales, offsets=offsets, count=n, frame_index=frame_index,
                                 group_key=group_key, blob=data, hw=(h, w))


def encode_frame(frame: GaussianFrame, width: int = None, height: int = None) -> AttributeImageSet:
    """Pack a frame into per-attribute 16-bit planes on device
    (ss/codec.py:124-158)."""
    import torch

    frame = as_frame(frame)
    n, m = frame.count, frame.width
    if width is None or height is None:
        side = math.ceil(math.sqrt(n))
        width = width or side
        height = height or side
    if n > width * height:
        raise CapacityError(f"{n} primitives exceed {width}x{height} image capacity")
    planes_in = frame.planes()
    eng = _engine(planes_in.device)
    lohi = np.zeros(2 * m, dtype=np.float64)
    if n == 0:
        raise StructuralError("cannot encode an empty frame")
    eng.call("airgs_plane_minmax", _ptr(planes_in), n, m, planes_in.shape[1],
             lohi.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), eng.stream())
    scales = np.zeros(m)
    offsets = np.zeros(m)
    for j in range(m):
        lo, hi = float(lohi[2 * j]), float(lohi[2 * j + 1])
        offsets[j] = lo
        scales[j] = 0.0 if hi == lo else (hi - lo) / QMAX
    pp = width * height
    out = torch.empty((m, pp), dtype=torch.int16, device=planes_in.device)
    eng.call("airgs_gsai_encode", _ptr(planes_in), n, m, planes_in.shape[1],
             offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
             scales.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), pp, _ptr(out), eng.stream())
    images = out.cpu().numpy().view(np.uint16).reshape(m, height, width)
    return AttributeImageSet(images=images, scales=scales, offsets=offsets, count=n,
                             frame_index=frame.frame_index, group_key=frame.group_key)


def decode_frame(image_set: AttributeImageSet, device=None) -> GaussianFrame:
    """Attribute planes -> device-resident frame (ss/codec.py:161-169)."""
    import torch

    if not isinstance(image_set, AttributeImageSet):  # a reference AttributeImageSet
        image_set = AttributeImageSet.from_bytes(image_set.to_bytes())
    m = image_set.num_attributes
    degree_from_param_dim(m)
    n = image_set.count
    h, w = image_set.height, image_set.width
    if n > w * h:
        raise DecodeError("attribute image count exceeds its planes")
    blob = image_set.device_blob(device)
    eng = _engine(blob.device)
    out = torch.zeros((m, dv.ld_for(n)), dtype=torch.float64, device=blob.device)
    if n:
        eng.call("airgs_gsai_decode", _ptr(blob), blob.numel(), n, m, w * h, _ptr(out), out.shape[1], eng.stream())
    return GaussianFrame(device_params=out, count=n, frame_index=image_set.frame_index,
                         group_key=image_set.group_key)


# ---------------------------------------------------------------------------
# GSDP


class DeltaPayload:
    """Serialized sparse delta; ``payload_bytes`` is the exact wire size."""

    __slots__ = ("data", "frame_index", "base_key", "entry_count", "quant_step")

    def __init__(self, data, frame_index, base_key, entry_count, quant_step):
        for k, v in (("data", bytes(data)), ("frame_index", frame_index), ("base_key", base_key),
                     ("entry_count", entry_count), ("quant_step", quant_step)):
            object.__setattr__(self, k, v)

    def __setattr__(self, k, v):
        raise AttributeError("DeltaPayload is immutable")

    def __eq__(self, o):
        return isinstance(o, DeltaPayload) and (self.data, self.frame_index, self.base_key, self.entry_count,
                                                 self.quant_step) == (o.data, o.frame_index, o.base_key,
                                                                      o.entry_count, o.quant_step)

    @property
    def payload_bytes(self) -> int:
        return len(self.data)


def quantize_overlay(ov: dv.Overlay, quant_step: float, want_decoded: bool = True):
    """encode_delta's rule on device: (nz mask, decoded rows q*step or None)."""
    import torch

    if quant_step <= 0:
        raise StructuralError("quant_step must be positive")
    eng = _engine(ov.rows.device)
    nz = torch.zeros_like(ov.present)
    deq = torch.zeros_like(ov.rows) if want_decoded else None
    bad = ctypes.c_int64(-1)
    if ov.n:
        eng.call("airgs_quantize", _ptr(ov.rows), _ptr(ov.present), ov.n, ov.width, ov.ld, float(quant_step),
                 _ptr(nz), _ptr(deq), ctypes.byref(bad), eng.stream())
    return nz, deq


def encode_delta(delta: DeltaTensor, quant_step: float, frame_index: int = 0, base_key: int = 0) -> DeltaPayload:
    """Quantise to i32 fixed point on device; entries that quantise to all
    zeros are dropped (ss/codec.py:187-214)."""
    if quant_step <= 0:
        raise StructuralError("quant_step must be positive")
    delta = as_delta(delta)
    if delta.base_count == 0 or delta.is_empty():
        hdr = _DELTA_HEADER.pack(DELTA_MAGIC, frame_index, base_key, 0, quant_step)
        return DeltaPayload(hdr, frame_index, base_key, 0, quant_step)
    ov = delta.overlay()
    nz, _ = quantize_overlay(ov, quant_step, want_decoded=False)
    return _emit(ov, nz, quant_step, frame_index, base_key)


def _emit(ov, nz, quant_step, frame_index, base_key, count_hint=None):
    import torch

    eng = _engine(ov.rows.device)
    cnt = int(nz[: ov.n].sum().item()) if count_hint is None else int(count_hint)
    cap = 24 + cnt * (10 + 4 * ov.width)
    buf = torch.zeros((cap,), dtype=torch.uint8, device=ov.rows.device)
    nbytes = ctypes.c_int64(0)
    entries = ctypes.c_int64(0)
    eng.call("airgs_gsdp_encode", _ptr(ov.rows), _ptr(nz), ov.n, ov.width, ov.ld, float(quant_step), _ptr(buf), cap,
             ctypes.byref(nbytes), ctypes.byref(entries), eng.stream())
    body = buf[24: nbytes.value].cpu().numpy().tobytes()
    hdr = _DELTA_HEADER.pack(DELTA_MAGIC, frame_index, base_key, entries.value, quant_step)
    return DeltaPayload(hdr + body, frame_index, base_key, entries.value, quant_step)


def parse_delta_header(data: bytes):
    if len(data) < DELTA_HEADER_BYTES:
        raise DecodeError("delta payload shorter than its header")
    magic, frame_index, base_key, entry_count, quant_step = _DELTA_HEADER.unpack_from(data, 0)
    if magic != DELTA_MAGIC:
        raise DecodeError(f"bad delta magic {magic!r}")
    return frame_index, base_key, entry_count, quant_step


def decode_delta_device(data, base_count: int = None, param_width: int = None, device=None, payload_dev=None):
    """GSDP bytes -> device overlay.  Returns (DeltaTensor, idx tensor)."""
    import torch

    # a DeltaPayload of either package, or raw bytes
    data = bytes(data.data) if hasattr(data, "data") and not isinstance(data, (bytes, bytearray, memoryview)) \
        else bytes(data)
    _, _, entry_count, quant_step = parse_delta_header(data)
    dev = dv.device_of(device)
    pd = payload_dev if payload_dev is not None else _to_device_bytes(data, dev)
    eng = _engine(dev)
    if param_width is None or base_count is None:
        pos = ctypes.c_int64(0)
        err = ctypes.c_int32(0)
        eng.call("airgs_gsdp_varint_end", _ptr(pd), len(data), entry_count, ctypes.byref(pos), ctypes.byref(err),
                 eng.stream())
        if err.value == 1:
            raise DecodeError("truncated varint")
        if err.value == 2:
            raise DecodeError("varint too long")
        remaining = len(data) - pos.value
        if param_width is None:
            if entry_count == 0:
                raise DecodeError("param_width required to decode an empty delta")
            if remaining % (4 * entry_count):
                raise DecodeError("delta payload length inconsistent with entry count")
            param_width = remaining // (4 * entry_count)
        if remaining != 4 * entry_count * param_width:
            raise DecodeError("truncated delta payload")
        if base_count is None:
            if entry_count == 0:
                base_count = 0
            else:
                # largest index = sum of all gaps: decode against an open base
                ov, idx = _decode_call(eng, pd, data, entry_count, quant_step, param_width, 1 << 62, dev,
                                       probe=True)
                base_count = int(idx[-1].item()) + 1
    ov, idx = _decode_call(eng, pd, data, entry_count, quant_step, param_width, base_count, dev)
    return DeltaTensor(base_count, param_width, overlay=ov), idx


def _decode_call(eng, pd, data, entry_count, quant_step, width, base_count, dev, probe=False):
    import torch

    idx = torch.empty((max(entry_count, 1),), dtype=torch.int64, device=dev)
    ent = torch.zeros((1,), dtype=torch.int64, device=dev)
    if probe:  # indices only
        eng.call("airgs_gsdp_decode", _ptr(pd), len(data), entry_count, float(quant_step), width, 0,
                 _ptr(None), 0, _ptr(None), _ptr(idx), _ptr(ent), eng.stream())
        return None, idx[:entry_count]
    ov = dv.Overlay.empty(base_count, width, dev)
    eng.call("airgs_gsdp_decode", _ptr(pd), len(data), entry_count, float(quant_step), width, base_count,
             _ptr(ov.rows), ov.ld, _ptr(ov.present), _ptr(idx), _ptr(ent), eng.stream())
    return ov, idx[:entry_count]


def _payload_bytes(data):
    return bytes(data.data) if hasattr(data, "data") and not isinstance(data, (bytes, bytearray, memoryview)) \
        else bytes(data)


def decode_apply_device(data, canon, n: int, width: int, device=None, payload_dev=None, out=None, ahead=None):
    """decode_delta + apply_delta fused (airgs_gsdp_decode_apply): GSDP bytes
    applied to the plane-major canonical parameters ``canon`` (width, ld) ->
    a new (width, ld) device tensor, bit-identical to
    ``apply_overlay(canon, n, decode_delta_device(data, n, width)[0].overlay())``
    without the dense overlay.  ``ahead=(next_data, next_payload_dev)``: the
    frame the caller decodes next, whose varint scan is enqueued ahead on the
    engine's side stream under deferred checking
    (airgs_gsdp_decode_apply_ahead)."""
    import torch

    data = _payload_bytes(data)
    _, _, entry_count, quant_step = parse_delta_header(data)
    dev = dv.device_of(device)
    pd = payload_dev if payload_dev is not None else _to_device_bytes(data, dev)
    if out is None:
        out = torch.empty_like(canon)
    eng = _engine(dev)
    nd, n_entries = None, 0
    if ahead is not None and ahead[1] is not None:
        nd = _payload_bytes(ahead[0])
        try:
            n_entries = parse_delta_header(nd)[2]
        except DecodeError:  # (reported when that frame itself is decoded)
            nd = None
    if nd is not None:
        eng.call("airgs_gsdp_decode_apply_ahead", _ptr(pd), len(data), entry_count, _ptr(ahead[1]), len(nd),
                 n_entries, float(quant_step), int(width), _ptr(canon), int(n), int(canon.shape[1]), _ptr(out),
                 eng.stream())
        return out
    eng.call("airgs_gsdp_decode_apply", _ptr(pd), len(data), entry_count, float(quant_step), int(width),
             _ptr(canon), int(n), int(canon.shape[1]), _ptr(out), eng.stream())
    return out


def decode_delta(payload, base_count: int = None, param_width: int = None) -> DeltaTensor:
    """Inverse of encode_delta (ss/codec.py:217-248); device-resident result."""
    return decode_delta_device(payload, base_count, param_width)[0]
