"""HBM layouts shared by every module.

* Parameters live plane-major: a float64 tensor ``(width, ld)`` whose row c is
  attribute c of every primitive (the GSAI plane order), ``ld`` = count
  rounded up to a multiple of 8 so each plane starts 64-byte aligned.
* A sparse delta lives as a dense overlay: float64 ``rows (width, ld)`` plus
  ``present (ld,)`` uint8 -- entries are where ``present`` is 1.  Dense
  overlays turn compose / apply / prune into unit-stride streaming kernels.

Moving data between these layouts and the reference's host objects (numpy
``(n, width)`` arrays, dict-based deltas) is plumbing done with torch copies;
all arithmetic runs in the airgs_b200 kernels.
"""

from __future__ import annotations

import numpy as np


def _torch():
    import torch

    return torch


def ld_for(n: int) -> int:
    return max(8, (int(n) + 7) // 8 * 8)


def device_of(device=None):
    torch = _torch()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    if isinstance(device, int):
        return torch.device("cuda", device)
    return torch.device(device)


def upload_params(params: np.ndarray, device=None):
    """(n, width) float64 host array -> (width, ld) plane-major device tensor."""
    torch = _torch()
    dev = device_of(device)
    n, w = params.shape
    t = torch.zeros((w, ld_for(n)), dtype=torch.float64, device=dev)
    if n:
        # one copy of the row-major bytes, transposed to planes on the device
        # (no host-side transpose: airgs_rows_to_planes)
        from ._lib import engine, ptr

        import warnings

        rows = np.ascontiguousarray(np.asarray(params, dtype=np.float64))
        with warnings.catch_warnings():  # read-only frames: the tensor is only read by the copy
            warnings.simplefilter("ignore", UserWarning)
            raw = torch.from_numpy(rows.view(np.uint8).reshape(-1)).to(dev)
        eng = engine(dev)
        eng.call("airgs_rows_to_planes", ptr(raw), 0, n, w, ptr(t), t.shape[1], eng.stream())
    return t


def download_params(planes, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros((0, planes.shape[0]), dtype=np.float64)
    return np.ascontiguousarray(planes[:, :n].t().cpu().numpy())


class Overlay:
    """Dense device form of a sparse delta."""

    __slots__ = ("rows", "present", "n", "width")

    def __init__(self, rows, present, n, width):
        self.rows = rows
        self.present = present
        self.n = int(n)
        self.width = int(width)

    @staticmethod
    def empty(n, width, device=None):
        torch = _torch()
        dev = device_of(device)
        ld = ld_for(n)
        return Overlay(torch.zeros((width, ld), dtype=torch.float64, device=dev),
                       torch.zeros((ld,), dtype=torch.uint8, device=dev), n, width)

    @staticmethod
    def from_entries(idx: np.ndarray, rows: np.ndarray, n: int, width: int, device=None):
        torch = _torch()
        ov = Overlay.empty(n, width, device)
        if len(idx):
            dev = ov.rows.device
            ti = torch.from_numpy(np.asarray(idx, dtype=np.int64)).to(dev)
            tr = torch.from_numpy(np.ascontiguousarray(np.asarray(rows, dtype=np.float64).T)).to(dev)
            ov.rows[:, ti] = tr
            ov.present[ti] = 1
        return ov

    def entries(self):
        """(sorted int64 indices, (E, width) float64 rows) on the host."""
        torch = _torch()
        idx = torch.nonzero(self.present[: self.n]).flatten()
        if idx.numel() == 0:
            return np.zeros(0, dtype=np.int64), np.zeros((0, self.width), dtype=np.float64)
        rows = self.rows[:, idx].t().contiguous().cpu().numpy()
        return idx.cpu().numpy().astype(np.int64), rows

    def count(self) -> int:
        return int(self.present[: self.n].sum().item()) if self.n else 0

    @property
    def ld(self):
        return self.rows.shape[1]
