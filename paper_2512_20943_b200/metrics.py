"""Image metrics on device: PSNR (drop-in for ``ss/metrics.py:37-43``) and
the trainer's loss terms SSIM / SSIM gradient / L1 / L1 gradient
(``ss/metrics.py:47-121``).

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


SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01**2
SSIM_C2 = 0.03**2


def _window_1d() -> np.ndarray:
    """The reference's 1-D Gaussian (ss/metrics.py:47-52), normalised to sum 1:
    its outer product is the reference's normalised 11x11 window."""
    half = (SSIM_WINDOW - 1) / 2.0
    x = np.arange(SSIM_WINDOW) - half
    g = np.exp(-(x**2) / (2.0 * SSIM_SIGMA**2))
    return np.ascontiguousarray(g / g.sum())


_WIN1 = _window_1d()


def _pair(a, b, dev):
    ta, tb = _as_tensor(a, dev), _as_tensor(b, dev)
    if tuple(ta.shape) != tuple(tb.shape):
        raise StructuralError(f"resolution mismatch: {tuple(ta.shape)} vs {tuple(tb.shape)}")
    if ta.dim() not in (2, 3) or (ta.dim() == 3 and ta.shape[2] != 3):
        raise StructuralError("images must be (h, w) or (h, w, 3)")
    return ta, tb


def _ssim_call(a, b, want_grad):
    import ctypes

    import torch

    from ._lib import engine, ptr

    dev = dv.device_of(None)
    ta, tb = _pair(a, b, dev)
    h, w = int(ta.shape[0]), int(ta.shape[1])
    ch = 1 if ta.dim() == 2 else 3
    eng = engine(dev)
    out = torch.zeros((1,), dtype=torch.float64, device=dev)
    grad = torch.empty_like(ta) if want_grad else None
    win = (ctypes.c_double * SSIM_WINDOW)(*_WIN1.tolist())
    eng.call("airgs_ssim", ptr(ta), ptr(tb), h, w, ch, win, ptr(out), ptr(grad) if want_grad else None,
             eng.stream())
    return out, grad


def ssim(a, b) -> float:
    """Mean local SSIM of the luminance channels; 1.0 for identical images
    (ss/metrics.py:77-86)."""
    out, _ = _ssim_call(a, b, False)
    return float(out.item())


def ssim_grad(a, b, as_numpy: bool = True):
    """d(mean SSIM)/d(pixels of a), same shape as ``a`` (ss/metrics.py:89-113)."""
    _, g = _ssim_call(a, b, True)
    return g.cpu().numpy() if as_numpy else g


def _l1_call(a, b, want_grad):
    import torch

    from ._lib import engine, ptr

    dev = dv.device_of(None)
    ta, tb = _as_tensor(a, dev), _as_tensor(b, dev)
    if tuple(ta.shape) != tuple(tb.shape):
        raise StructuralError(f"resolution mismatch: {tuple(ta.shape)} vs {tuple(tb.shape)}")
    eng = engine(dev)
    out = torch.zeros((1,), dtype=torch.float64, device=dev)
    grad = torch.empty_like(ta) if want_grad else None
    eng.call("airgs_l1", ptr(ta), ptr(tb), ta.numel(), ptr(out), ptr(grad) if want_grad else None, eng.stream())
    return out, grad


def l1(a, b) -> float:
    """mean |a - b| (ss/metrics.py:116-118)."""
    return float(_l1_call(a, b, False)[0].item())


def l1_grad(a, b, as_numpy: bool = True):
    """sign(a - b) / a.size (ss/metrics.py:121)."""
    _, g = _l1_call(a, b, True)
    return g.cpu().numpy() if as_numpy else g


def mean_quality(values) -> float:
    """Arithmetic mean over views exactly as ``float(np.mean([...]))``."""
    return float(np.mean(list(values)))


__all__ = ["PSNR_CAP_DB", "psnr", "psnr_from_sse", "mean_quality", "ssim", "ssim_grad", "l1", "l1_grad", "math"]
