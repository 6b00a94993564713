"""Seeded synthetic scenes at the BASELINE.json shapes.

The reference's scene generator rejection-samples blob centres (O(n^2)) and
cannot reach 300k primitives, so the harness scales up the reference test
suite's ``random_frame`` recipe instead (tests/conftest.py:31-43 of the
reference): uniform positions, normalised N(0,1) quaternions, log-scales
around ln(sigma), opacity logits U(-1, 3), colour logits N(0, 1).  Motion:
20% movers drifting N(0, 0.004) per frame (random walk); appearance events
append new primitives next to existing ones.  Cameras: the reference ring
rig (radius 3, height 0.3, focal = W*40/48).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .camera import ring_rig


@dataclass(frozen=True)
class SceneConfig:
    name: str
    count: int
    views: int
    resolution: tuple  # (W, H)
    frames: int
    spread: float
    sigma: float
    levels: int = 4
    sh_degree: int = 0


CONFIGS = {
    # BASELINE.json configs[0..4]
    "C1": SceneConfig("toy", 10_000, 4, (256, 256), 5, 0.6, 0.02, levels=4),
    "C2": SceneConfig("n3dv", 300_000, 18, (1352, 1014), 300, 1.5, 0.006, levels=8),
    "C3": SceneConfig("sweep1080p", 300_000, 18, (1920, 1080), 8, 1.5, 0.006, levels=8),
    "C4": SceneConfig("meetroom", 150_000, 13, (1280, 720), 300, 1.5, 0.006, levels=8),
    "C5": SceneConfig("stress", 2_000_000, 32, (1920, 1080), 600, 1.5, 0.006, levels=8),
}


def param_width(sh_degree: int) -> int:
    return 14 + 3 * (sh_degree + 1) ** 2


def random_gaussians(rng, n, spread, sigma, sh_degree=0):
    w = param_width(sh_degree)
    p = np.zeros((n, w))
    p[:, 0:3] = rng.uniform(-spread, spread, (n, 3))
    q = rng.normal(size=(n, 4))
    p[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    p[:, 7:10] = math.log(sigma) + rng.uniform(-0.3, 0.3, (n, 3))
    p[:, 10] = rng.uniform(-1.0, 3.0, n)
    p[:, 11:14] = rng.normal(0.0, 1.0, (n, 3))
    p[:, 14:] = rng.normal(0.0, 0.1, (n, w - 14))
    return p


def cameras(cfg: SceneConfig):
    W, H = cfg.resolution
    return ring_rig(cfg.views, radius=3.0, center=(0.0, 0.0, 0.0), height=0.3, focal=float(W) * 40.0 / 48.0,
                    resolution=(W, H))


class Sequence:
    """Ground-truth parameter sequence: a canonical set, movers, and
    appearance events every ``event_every`` frames."""

    def __init__(self, cfg: SceneConfig, seed: int = 0, mover_fraction: float = 0.2, drift: float = 0.004,
                 event_every: int = 50, event_fraction: float = 0.01):
        self.cfg = cfg
        rng = np.random.default_rng(seed)
        self.base = random_gaussians(rng, cfg.count, cfg.spread, cfg.sigma, cfg.sh_degree)
        nm = int(round(mover_fraction * cfg.count))
        self.movers = np.sort(rng.choice(cfg.count, nm, replace=False))
        self.drift = drift
        self.seed = seed
        self.event_every = event_every
        self.event_fraction = event_fraction
        self._walk = {0: np.zeros((nm, 3))}
        self._rng_walk = np.random.default_rng(seed + 1)
        self._events = {}
        if event_every:
            erng = np.random.default_rng(seed + 2)
            ne = max(1, int(round(event_fraction * cfg.count)))
            for t in range(event_every, cfg.frames, event_every):
                hosts = erng.integers(0, cfg.count, ne)
                rows = random_gaussians(erng, ne, cfg.spread, cfg.sigma, cfg.sh_degree)
                rows[:, 0:3] = self.base[hosts, 0:3] + erng.normal(0.0, 2.0 * cfg.sigma, (ne, 3))
                self._events[t] = rows

    def _offset(self, t):
        while max(self._walk) < t:
            k = max(self._walk)
            self._walk[k + 1] = self._walk[k] + self._rng_walk.normal(0.0, self.drift, self._walk[k].shape)
        return self._walk[t]

    def frame(self, t: int) -> np.ndarray:
        """Ground-truth parameters at frame t (rows appended by events)."""
        p = self.base.copy()
        p[self.movers, 0:3] += self._offset(t)
        extra = [rows for f, rows in sorted(self._events.items()) if f <= t]
        return np.vstack([p] + extra) if extra else p

    def event_frames(self):
        return sorted(self._events)
