"""PSNR on device (drop-in for ``ss/metrics.py:37-43``).

The hot paths never call this: per-view SSE is fused into the compositing
kernel (``rasterizer.render_views``) and turned into PSNR by
``psnr_from_sse``.  ``psnr(a, b)`` keeps the reference signature for
callers holding images.
"""

from __future__ import annotations

import math

import numpy as np

from . import device as dv
from .errors import StructuralError

PSNR_CAP_DB = 100.0


def psnr_from_sse(sse: float, size: int) -> float:
    """min(100, 10*log10(1/mse)), exactly 100 when mse == 0."""
    mse = float(np.float64(sse) / np.float64(size)) if size else 0.0
    if mse <= 0.0:
        return PSNR_CAP_DB
    return min(PSNR_CAP_DB, float(10.0 * np.log10(1.0 / mse)))


def _as_tensor(x, dev):
    import torch

    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float64).contiguous()
    px = getattr(x, "pixels", x)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(px, dtype=np.float64))).to(dev)


def psnr(a, b) -> float:
    import torch

    from ._lib import engine, ptr

    dev = dv.device_of(None)
    ta, tb = _as_tensor(a, dev), _as_tensor(b, dev)
    if tuple(ta.shape) != tuple(tb.shape):
        raise StructuralError(f"resolution mismatch: {tuple(ta.shape)} vs {tuple(tb.shape)}")
    eng = engine(dev)
    out = torch.zeros((1,), dtype=torch.float64, device=dev)
    eng.call("airgs_sse", ptr(ta), ptr(tb), ta.numel(), ptr(out), eng.stream())
    return psnr_from_sse(float(out.item()), ta.numel())


def mean_quality(values) -> float:
    """Arithmetic mean over views exactly as ``float(np.mean([...]))``."""
    return float(np.mean(list(values)))


__all__ = ["PSNR_CAP_DB", "psnr", "psnr_from_sse", "mean_quality", "math"]
