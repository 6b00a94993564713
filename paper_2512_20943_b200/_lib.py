"""ctypes binding of ``lib/libairgs_b200.so`` (the C-ABI in
``include/airgs_b200.h``) plus the per-device engine that owns a context.

There is no CPU fallback: if the shared library is missing, or no sm_100
GPU is visible, every compute entry point raises.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AIRGS_B200_LIB") or os.path.join(_HERE, "lib", "libairgs_b200.so")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_i64_p = ctypes.POINTER(ctypes.c_int64)
vp = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64
f64 = ctypes.c_double


class CameraC(ctypes.Structure):
    _fields_ = [
        ("rot", ctypes.c_double * 9),
        ("trans", ctypes.c_double * 3),
        ("center", ctypes.c_double * 3),
        ("focal", ctypes.c_double),
        ("near_clip", ctypes.c_double),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
    ]


class FrameC(ctypes.Structure):
    _fields_ = [
        ("params", ctypes.c_void_p),
        ("count", ctypes.c_int64),
        ("ld", ctypes.c_int64),
        ("width", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class ItemC(ctypes.Structure):
    _fields_ = [
        ("frame", ctypes.c_int32),
        ("camera", ctypes.c_int32),
        ("target", ctypes.c_void_p),
        ("image", ctypes.c_void_p),
        ("usage", ctypes.c_void_p),
        ("frozen_pos", ctypes.c_void_p),
        ("tile_minrank", ctypes.c_void_p),
        ("tile_keep_min", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


# name -> (restype, argtypes); must match include/airgs_b200.h exactly
SIGNATURES = {
    "airgs_ctx_create": (ctypes.c_int, [ctypes.POINTER(vp), i32]),
    "airgs_ctx_destroy": (ctypes.c_int, [vp]),
    "airgs_last_error": (ctypes.c_char_p, [vp]),
    "airgs_launch_count": (i64, [vp]),
    "airgs_timing": (ctypes.c_int, [vp, i32, c_double_p, c_i64_p, c_double_p, c_i64_p]),
    "airgs_timing_stages": (ctypes.c_int, [vp, i32, c_double_p, c_i64_p, i32]),
    "airgs_tile_footprint": (ctypes.c_int, [vp, ctypes.POINTER(FrameC), ctypes.POINTER(CameraC), i32, vp, i32, vp,
                                            i64, vp]),
    "airgs_debug_tile_lists": (ctypes.c_int, [vp, ctypes.POINTER(FrameC), ctypes.POINTER(CameraC), i64, vp, vp, vp]),
    "airgs_eval_stats": (ctypes.c_int, [vp, i32, c_i64_p]),
    "airgs_eval_margins": (ctypes.c_int, [vp, c_double_p]),
    "airgs_defer": (ctypes.c_int, [vp, i32, ctypes.POINTER(ctypes.c_uint32)]),
    "airgs_render": (ctypes.c_int, [vp, ctypes.POINTER(FrameC), i32, ctypes.POINTER(CameraC), i32,
                                    ctypes.POINTER(ItemC), i32, vp, vp]),
    "airgs_render_backward": (ctypes.c_int, [vp, ctypes.POINTER(FrameC), ctypes.POINTER(CameraC), vp, vp, vp, vp]),
    "airgs_compositing_order": (ctypes.c_int, [vp, ctypes.POINTER(FrameC), ctypes.POINTER(CameraC), vp, vp, c_i64_p,
                                               vp]),
    "airgs_composite_forward": (ctypes.c_int, [vp, i64, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp]),
    "airgs_sse": (ctypes.c_int, [vp, vp, vp, i64, vp, vp]),
    "airgs_composite_forward_record": (ctypes.c_int, [vp, i64, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp,
                                                      vp]),
    "airgs_composite_backward": (ctypes.c_int, [vp, i64, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp]),
    "airgs_ssim": (ctypes.c_int, [vp, vp, vp, i32, i32, i32, c_double_p, vp, vp, vp]),
    "airgs_l1": (ctypes.c_int, [vp, vp, vp, i64, vp, vp, vp]),
    "airgs_rows_to_planes": (ctypes.c_int, [vp, vp, i64, i64, i32, vp, i64, vp]),
    "airgs_gsai_decode": (ctypes.c_int, [vp, vp, i64, i64, i32, i64, vp, i64, vp]),
    "airgs_gsdp_decode": (ctypes.c_int, [vp, vp, i64, i64, f64, i32, i64, vp, i64, vp, vp, vp, vp]),
    "airgs_gsdp_decode_apply": (ctypes.c_int, [vp, vp, i64, i64, f64, i32, vp, i64, i64, vp, vp]),
    "airgs_gsdp_decode_apply_ahead": (ctypes.c_int, [vp, vp, i64, i64, vp, i64, i64, f64, i32, vp, i64, i64, vp,
                                                     vp]),
    "airgs_gsdp_varint_end": (ctypes.c_int, [vp, vp, i64, i64, c_i64_p, ctypes.POINTER(i32), vp]),
    "airgs_plane_minmax": (ctypes.c_int, [vp, vp, i64, i32, i64, c_double_p, vp]),
    "airgs_gsai_encode": (ctypes.c_int, [vp, vp, i64, i32, i64, c_double_p, c_double_p, i64, vp, vp]),
    "airgs_gsdp_encode": (ctypes.c_int, [vp, vp, vp, i64, i32, i64, f64, vp, i64, c_i64_p, c_i64_p, vp]),
    "airgs_delta_compose": (ctypes.c_int, [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(vp), c_double_p, i64, i32,
                                           i64, f64, i32, vp, vp, vp]),
    "airgs_delta_apply": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, i32, vp, vp, i64, i32, i64, vp, vp]),
    "airgs_quantize": (ctypes.c_int, [vp, vp, vp, i64, i32, i64, f64, vp, vp, c_i64_p, vp]),
    "airgs_prune_rank": (ctypes.c_int, [vp, vp, vp, i64, vp, c_i64_p, vp]),
    "airgs_level_sizes": (ctypes.c_int, [vp, vp, vp, i64, i32, c_i64_p, i32, c_i64_p, vp]),
}

_STATUS = {
    -1: errors.StructuralError,
    -2: errors.ValidationError,
    -3: errors.CapacityError,
    -5: errors.DecodeError,
}

_lib = None
_lock = threading.Lock()


def load_library():
    """Load the shared library (no GPU needed) and bind every symbol."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"airgs_b200 CUDA library not built: {LIB_PATH} is missing "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'`)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class Engine:
    """One airgs context on one CUDA device (scratch workspace owner)."""

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("airgs_b200 requires a CUDA device (sm_100); none is visible")
        self.lib = load_library()
        self.device = int(device)
        self.torch_device = torch.device("cuda", self.device)
        ctx = vp()
        rc = self.lib.airgs_ctx_create(ctypes.byref(ctx), self.device)
        if rc != 0:
            raise RuntimeError(f"airgs_ctx_create failed on cuda:{self.device} (status {rc}); an sm_100 GPU is required")
        self.ctx = ctx

    def stream(self):
        import torch

        return vp(torch.cuda.current_stream(self.torch_device).cuda_stream)

    def call(self, name, *args):
        rc = getattr(self.lib, name)(self.ctx, *args)
        if rc != 0:
            msg = (self.lib.airgs_last_error(self.ctx) or b"").decode(errors="replace")
            exc = _STATUS.get(rc)
            if exc is None:
                raise RuntimeError(f"{name} failed (status {rc}): {msg}")
            raise exc(msg)
        return rc

    STAGES = ("composite", "project", "bin", "sort", "decode", "apply", "sse", "quantize")

    def timing(self, enable=-1):
        """Read (and optionally re-arm/reset) the per-stage event timers:
        returns {stage}_ms and {stage}_launches for every stage of
        airgs_timing_stages."""
        k = len(self.STAGES)
        ms, n = (ctypes.c_double * k)(), (ctypes.c_int64 * k)()
        self.lib.airgs_timing_stages(self.ctx, int(enable), ms, n, k)
        out = {}
        for j, name in enumerate(self.STAGES):
            out[f"{name}_ms"] = ms[j]
            out[f"{name}_launches"] = n[j]
        return out

    def eval_stats(self, enable=-1):
        """Read (and optionally re-arm/reset) the diagnostic evaluation counters:
        returns dict(bbox, live, contrib) (pairs of the reference's loop) and
        tile_pairs (binned (tile, primitive) list entries) and records (projected
        records written)."""
        c = (ctypes.c_int64 * 5)()
        self.call("airgs_eval_stats", int(enable), c)
        return {"bbox": c[0], "live": c[1], "contrib": c[2], "tile_pairs": c[3], "records": c[4]}

    MARGIN_KEYS = ("min_rel_weight_margin", "min_rel_termination_margin", "min_depth_gap_ulps", "depth_ties",
                   "min_bbox_floor_margin_px", "min_near_clip_margin", "min_rel_alpha_cull_margin")

    def eval_margins(self):
        """Decision margins accumulated since the counters were armed (see
        airgs_eval_margins); +inf where no such decision was taken."""
        m = (ctypes.c_double * 7)()
        self.call("airgs_eval_margins", m)
        return {k: float(v) for k, v in zip(self.MARGIN_KEYS, m)}

    @property
    def launches(self) -> int:
        return int(self.lib.airgs_launch_count(self.ctx))

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                self.lib.airgs_ctx_destroy(self.ctx)
        except Exception:
            pass


_engines: dict = {}
_tls = threading.local()


def engine(device=None) -> Engine:
    """The process-wide engine for ``device`` (default: torch's current), or
    the current thread's engine lane on it (see ``engine_lane``)."""
    import torch

    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    if isinstance(device, torch.device):
        device = device.index if device.index is not None else torch.cuda.current_device()
    device = int(device)
    key = device if getattr(_tls, "lane", 0) == 0 else (device, _tls.lane)
    with _lock:
        eng = _engines.get(key)
    if eng is None:
        eng = Engine(device)
        with _lock:
            _engines[key] = eng
    return eng


@contextlib.contextmanager
def engine_lane(lane: int):
    """Route this thread's calls to a second (third, ...) engine on the same
    device: its own context and scratch, so that independent work on another
    stream (e.g. the next frame of a probe batch) can be in flight at once."""
    prev = getattr(_tls, "lane", 0)
    _tls.lane = int(lane)
    try:
        yield
    finally:
        _tls.lane = prev


def ptr(t) -> vp:
    """Device pointer of a torch tensor (None -> NULL)."""
    return vp(0 if t is None else t.data_ptr())
