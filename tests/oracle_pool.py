"""Process-parallel CPU oracle jobs for the full-size GPU parity tests.

The oracle (``oracle/airgs_oracle.py``) is single-threaded; a full C2 view
takes ~3 s of CPU.  These helpers fan independent views / levels out over a
``spawn`` pool (fresh interpreters: the parent's CUDA context and thread
pools are never forked), passing parameter arrays through .npy files
(memory-mapped by the workers).  Test infrastructure only.
"""

from __future__ import annotations

import os
import sys
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _init():
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def cam_args(cam):
    return (np.asarray(cam.pose, dtype=np.float64), float(cam.focal), tuple(int(v) for v in cam.resolution),
            float(getattr(cam, "near_clip", 0.05)))


def _cam(args):
    pose, focal, res, near = args
    return types.SimpleNamespace(pose=pose, focal=focal, resolution=res, near_clip=near)


def job_render_full(args):
    """(params .npy path, camera args) -> (clipped image, usage counts)."""
    from oracle import airgs_oracle as orc

    path, cam = args
    return orc.render_full(np.load(path, mmap_mode="r"), _cam(cam))


def job_psnr(args):
    """(params path, camera args, target path or (target params path, cam)) -> psnr."""
    from oracle import airgs_oracle as orc

    path, cam, tgt = args
    img = orc.render(np.load(path, mmap_mode="r"), _cam(cam))
    if isinstance(tgt, tuple):
        ref = orc.render(np.load(tgt[0], mmap_mode="r"), _cam(tgt[1]))
    else:
        ref = np.load(tgt, mmap_mode="r")
    return orc.psnr(img, ref)


def job_render_to(args):
    """(params path, camera args, out path): write the oracle's render."""
    from oracle import airgs_oracle as orc

    path, cam, out = args
    np.save(out, orc.render(np.load(path, mmap_mode="r"), _cam(cam)))
    return out


def pool_map(fn, jobs, procs=None):
    import multiprocessing as mp

    jobs = list(jobs)
    if not jobs:
        return []
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    n = max(1, min(len(jobs), procs or cores))
    with mp.get_context("spawn").Pool(n, initializer=_init) as pool:
        return pool.map(fn, jobs, chunksize=1)


def save(tmp_path, name, arr):
    path = os.path.join(str(tmp_path), name + ".npy")
    np.save(path, np.ascontiguousarray(arr))
    return path
