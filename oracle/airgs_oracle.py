"""CPU ORACLE for the AirGS per-frame evaluation path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and only
as the checker or the timed CPU arm.  The product package
(``paper_2512_20943_b200``) never imports it and has no CPU fallback.

It restates the reference algorithm (``/root/reference/pkg/src/splatstream``,
abbreviated ``ss/`` below) with plain arrays instead of the reference's
dict-based ``DeltaTensor``: a sparse delta is a pair ``(idx, rows)`` with
``idx`` strictly increasing int64 and ``rows`` float64 ``(E, W)``.  Each
function cites the reference lines it follows.

Numerics notes (verified on this host):
  * numpy matmuls here evaluate ``fma(a2,b2, fma(a1,b1, a0*b0))`` per
    output element (OpenBLAS); we reproduce them with an exact fused
    multiply-add (``_fma``) so the restatement is bit-identical.
  * ``np.linalg.norm(x, axis=1)`` sums squares left to right.
  * elementwise numpy never fuses.

Parity pinning: ``tests/golden/*.npz`` are produced by running the real
reference (``tests/golden/make_golden.py``); ``tests/test_oracle.py`` checks
this module against every fixture.
"""

from __future__ import annotations

import ctypes
import math
import os
import struct

import numpy as np

# --- constants (ss/_kernels_py.py:19-20, ss/rasterizer.py:51-56, ss/model.py:35) ---
EPS_CONTRIB = 1.0 / 255.0
ALPHA_CLAMP = 0.999
COV_BLUR = 0.3
RADIUS_SIGMA = 3.5
SH_C0 = 0.2820947917738781
SH_C1 = 0.4886025119029199
EPS_SPARSE = 1e-9
PSNR_CAP_DB = 100.0
MIN_DROP = 1e-12
TILE = 16
GSAI_MAGIC = b"GSAI"
GSDP_MAGIC = b"GSDP"
GSAI_HEADER = struct.Struct("<4sHIHHHB")  # ss/codec.py:27
GSDP_HEADER = struct.Struct("<4sIIId")  # ss/codec.py:28
QMAX = 65535

_HERE = os.path.dirname(os.path.abspath(__file__))


class OracleError(Exception):
    """Raised with the reference exception class name as ``kind``."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


# ---------------------------------------------------------------------------
# exact fused multiply-add (to mirror OpenBLAS' FMA accumulation)


def _fma(a, b, c):
    """Correctly rounded a*b+c elementwise (libm fma() in the oracle C lib)."""
    a, b, c = np.broadcast_arrays(np.asarray(a, np.float64), np.asarray(b, np.float64),
                                  np.asarray(c, np.float64))
    a, b, c = (np.ascontiguousarray(x) for x in (a, b, c))
    out = np.empty(a.shape, dtype=np.float64)
    D = ctypes.c_double
    _load().oracle_fma(a.size, _ptr(a, D), _ptr(b, D), _ptr(c, D), _ptr(out, D))
    return out


def dot3_fma(x0, x1, x2, y0, y1, y2):
    """OpenBLAS order: fma(x2,y2, fma(x1,y1, x0*y0))."""
    return _fma(x2, y2, _fma(x1, y1, np.multiply(x0, y0)))


# ---------------------------------------------------------------------------
# cameras (ss/camera.py:16-65)


class CamTerms:
    __slots__ = ("R", "t", "center", "f", "W", "H", "near")

    def __init__(self, cam):
        pose = np.asarray(cam.pose, dtype=np.float64)
        self.R = pose[:3, :3].copy()
        self.t = pose[:3, 3].copy()
        self.center = -self.R.T @ self.t  # ss/camera.py:45-48
        self.f = float(cam.focal)
        self.W, self.H = int(cam.resolution[0]), int(cam.resolution[1])
        self.near = float(getattr(cam, "near_clip", 0.05))


# ---------------------------------------------------------------------------
# activation + projection (ss/rasterizer.py:100-212)


def sigmoid(x):  # ss/model.py:63-64
    return 0.5 * (1.0 + np.tanh(0.5 * np.asarray(x, dtype=np.float64)))


def sh_degree_of(width):
    if width == 17:
        return 0
    if width == 26:
        return 1
    raise OracleError("StructuralError", f"no sh degree yields parameter width {width}")


class Prepared:
    __slots__ = ("order", "means2d", "conics", "alphas", "colors", "bboxes", "depth",
                 "radius", "z_all", "alpha_all", "cov2d", "det")


def prepare(params, cam):
    """Projection of every primitive for one camera (ss/rasterizer.py:113-212)."""
    P = np.ascontiguousarray(params, dtype=np.float64)
    n = P.shape[0]
    if n == 0:
        raise OracleError("StructuralError", "cannot render an empty frame")
    deg = sh_degree_of(P.shape[1])
    ct = CamTerms(cam)
    q = P[:, 3:7]
    sq = q * q
    qn = np.sqrt(((sq[:, 0] + sq[:, 1]) + sq[:, 2]) + sq[:, 3])  # norm, left-to-right
    if np.any(qn == 0) or not np.all(np.isfinite(P)):
        raise OracleError("ValidationError", "frame contains invalid primitive parameters")
    qh = q / qn[:, None]
    s2 = np.exp(2.0 * P[:, 7:10])
    alpha = sigmoid(P[:, 10])
    R, t = ct.R, ct.t
    mu = P[:, 0:3]
    tc = np.empty((n, 3))
    for r in range(3):  # mu @ R.T + t (FMA order, verified)
        tc[:, r] = dot3_fma(mu[:, 0], mu[:, 1], mu[:, 2], R[r, 0], R[r, 1], R[r, 2]) + t[r]
    keep = (tc[:, 2] > ct.near) & (alpha > EPS_CONTRIB)
    idx = np.nonzero(keep)[0]
    order = idx[np.argsort(tc[idx, 2], kind="stable")]
    out = Prepared()
    out.order = order
    tco = tc[order]
    x, y, z = tco[:, 0], tco[:, 1], tco[:, 2]
    f = ct.f
    mx = f * x / z + 0.5 * ct.W
    my = f * y / z + 0.5 * ct.H
    out.means2d = np.stack([mx, my], axis=1)
    out.depth = z
    # quaternion -> rotation (ss/model.py:72-85), exact elementwise
    w_, x_, y_, z_ = (qh[order, j] for j in range(4))
    m = np.empty((order.size, 3, 3))
    m[:, 0, 0] = 1 - 2 * (y_ * y_ + z_ * z_)
    m[:, 0, 1] = 2 * (x_ * y_ - w_ * z_)
    m[:, 0, 2] = 2 * (x_ * z_ + w_ * y_)
    m[:, 1, 0] = 2 * (x_ * y_ + w_ * z_)
    m[:, 1, 1] = 1 - 2 * (x_ * x_ + z_ * z_)
    m[:, 1, 2] = 2 * (y_ * z_ - w_ * x_)
    m[:, 2, 0] = 2 * (x_ * z_ - w_ * y_)
    m[:, 2, 1] = 2 * (y_ * z_ + w_ * x_)
    m[:, 2, 2] = 1 - 2 * (x_ * x_ + y_ * y_)
    rs = m * s2[order][:, None, :]
    cov3 = np.empty_like(m)
    for i in range(3):
        for j in range(3):
            cov3[:, i, j] = dot3_fma(rs[:, i, 0], rs[:, i, 1], rs[:, i, 2], m[:, j, 0], m[:, j, 1], m[:, j, 2])
    # Jacobian (ss/rasterizer.py:160-166); J @ R_wc
    j00 = f / z
    j02 = -f * x / (z * z)
    j12 = -f * y / (z * z)
    M = np.empty((order.size, 2, 3))
    for c in range(3):
        # row 0: [j00, 0, j02] ; row 1: [0, j00, j12]   (zeros are real BLAS inputs)
        M[:, 0, c] = dot3_fma(j00, 0.0, j02, R[0, c], R[1, c], R[2, c])
        M[:, 1, c] = dot3_fma(0.0, j00, j12, R[0, c], R[1, c], R[2, c])
    MC = np.empty((order.size, 2, 3))
    for i in range(2):
        for j in range(3):
            MC[:, i, j] = dot3_fma(M[:, i, 0], M[:, i, 1], M[:, i, 2], cov3[:, 0, j], cov3[:, 1, j], cov3[:, 2, j])
    a2 = dot3_fma(MC[:, 0, 0], MC[:, 0, 1], MC[:, 0, 2], M[:, 0, 0], M[:, 0, 1], M[:, 0, 2]) + COV_BLUR
    b2 = dot3_fma(MC[:, 0, 0], MC[:, 0, 1], MC[:, 0, 2], M[:, 1, 0], M[:, 1, 1], M[:, 1, 2])
    c2 = dot3_fma(MC[:, 1, 0], MC[:, 1, 1], MC[:, 1, 2], M[:, 1, 0], M[:, 1, 1], M[:, 1, 2]) + COV_BLUR
    det = a2 * c2 - b2 * b2
    out.conics = np.stack([c2 / det, -b2 / det, a2 / det], axis=1)
    out.cov2d, out.det = np.stack([a2, b2, c2], axis=1), det
    d = a2 - c2
    eig = 0.5 * (a2 + c2) + np.sqrt(np.maximum(0.25 * (d * d) + b2 * b2, 0.0))
    rad = RADIUS_SIGMA * np.sqrt(eig)
    W, H = ct.W, ct.H
    bb = np.empty((order.size, 4), dtype=np.int64)
    bb[:, 0] = np.clip(np.floor(mx - rad), 0, W)
    bb[:, 1] = np.clip(np.ceil(mx + rad) + 1, 0, W)
    bb[:, 2] = np.clip(np.floor(my - rad), 0, H)
    bb[:, 3] = np.clip(np.ceil(my + rad) + 1, 0, H)
    out.bboxes = bb
    out.radius, out.z_all, out.alpha_all = rad, tc[:, 2], alpha  # (decision-margin checks)
    # colour (ss/rasterizer.py:183-198)
    dirs = mu[order] - ct.center
    sd = dirs * dirs
    dn = np.sqrt((sd[:, 0] + sd[:, 1]) + sd[:, 2])
    dn = np.where(dn == 0, 1.0, dn)
    dh = dirs / dn[:, None]
    sh = P[order, 14:]
    lin = P[order, 11:14] + SH_C0 * sh[:, 0:3]
    if deg >= 1:
        lin = lin + SH_C1 * (-dh[:, 1:2] * sh[:, 3:6] + dh[:, 2:3] * sh[:, 6:9] - dh[:, 0:1] * sh[:, 9:12])
    out.colors = sigmoid(lin)
    out.alphas = alpha[order]
    return out


# ---------------------------------------------------------------------------
# compositing (C restatement of ss/_composite.pyx:18-74)

_lib = None


def _load():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.run(["make", "-C", _HERE, "all"], check=True, capture_output=True)
        lib = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        for name in ("oracle_composite_gmajor",):
            fn = getattr(lib, name)
            fn.restype = None
            fn.argtypes = [ctypes.c_int64, dp, dp, dp, dp, ip, ctypes.c_int, ctypes.c_int, dp, dp, ip]
        fn = lib.oracle_fma
        fn.restype = None
        fn.argtypes = [ctypes.c_int64, dp, dp, dp, dp]
        fn = lib.oracle_eval_counts
        fn.restype = None
        fn.argtypes = [ctypes.c_int64, dp, dp, dp, dp, ip, ctypes.c_int, ctypes.c_int, ip]
        fn = lib.oracle_composite_tiles
        fn.restype = None
        fn.argtypes = [ctypes.c_int64, dp, dp, dp, dp, ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, ip]
        _lib = lib
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def composite(means2d, conics, alphas, colors, bboxes, height, width, pixel_major=False):
    """Returns (image (h,w,3), t_final (h,w), usage (k,)) -- unclipped."""
    lib = _load()
    m2 = np.ascontiguousarray(means2d, dtype=np.float64)
    co = np.ascontiguousarray(conics, dtype=np.float64)
    al = np.ascontiguousarray(alphas, dtype=np.float64)
    cl = np.ascontiguousarray(colors, dtype=np.float64)
    bb = np.ascontiguousarray(bboxes, dtype=np.int64)
    k = m2.shape[0]
    img = np.empty((height, width, 3))
    tr = np.empty((height, width))
    us = np.zeros(max(k, 1), dtype=np.int64)
    D, I = ctypes.c_double, ctypes.c_int64
    args = (k, _ptr(m2, D), _ptr(co, D), _ptr(al, D), _ptr(cl, D), _ptr(bb, I), int(height), int(width))
    if pixel_major:
        lib.oracle_composite_tiles(*args, TILE, _ptr(img, D), _ptr(tr, D), _ptr(us, I))
    else:
        lib.oracle_composite_gmajor(*args, _ptr(img, D), _ptr(tr, D), _ptr(us, I))
    return img, tr, us[:k]


def eval_counts(params, cam):
    """(bbox, live, contrib) pair counts of the reference loop for one view
    (_composite.pyx:42-73; live = pixel not yet terminated, 0.999*T > 1/255)."""
    lib = _load()
    pr = prepare(params, cam)
    ct = CamTerms(cam)
    D, I = ctypes.c_double, ctypes.c_int64
    m2 = np.ascontiguousarray(pr.means2d, dtype=np.float64)
    co = np.ascontiguousarray(pr.conics, dtype=np.float64)
    al = np.ascontiguousarray(pr.alphas, dtype=np.float64)
    bb = np.ascontiguousarray(pr.bboxes, dtype=np.int64)
    out = np.zeros(3, dtype=np.int64)
    lib.oracle_eval_counts(m2.shape[0], _ptr(m2, D), _ptr(co, D), _ptr(al, D), _ptr(al, D), _ptr(bb, I),
                           int(ct.H), int(ct.W), _ptr(out, I))
    return tuple(int(v) for v in out)


def tile_keys(bboxes, width, height, tile=TILE):
    """CPU restatement of the tile binning (no tiles exist in the reference,
    SURVEY.md s8(c)): for primitive position p (depth rank) with a non-empty
    clipped bbox, emit key (tile_id << 32) | p for every tile its bbox
    overlaps, tile_id = ty * tiles_x + tx; keys sorted ascending."""
    bb = np.asarray(bboxes, dtype=np.int64).reshape(-1, 4)
    tx_n = (width + tile - 1) // tile
    ne = (bb[:, 1] > bb[:, 0]) & (bb[:, 3] > bb[:, 2])
    p = np.nonzero(ne)[0]
    if p.size == 0:
        return np.zeros(0, dtype=np.int64)
    u0, u1 = bb[p, 0] // tile, (bb[p, 1] - 1) // tile
    v0, v1 = bb[p, 2] // tile, (bb[p, 3] - 1) // tile
    nu, nv = u1 - u0 + 1, v1 - v0 + 1
    cnt = nu * nv
    rep = np.repeat(np.arange(p.size), cnt)
    j = np.arange(rep.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    tx = u0[rep] + j % nu[rep]
    ty = v0[rep] + j // nu[rep]
    return np.sort(((ty * tx_n + tx) << 32) | p[rep])


def threshold_tile_ranges(pr, tile=TILE, with_ext=False):
    """Tile range of each prepared primitive under the B200 binning's
    weight-threshold narrowing (restated from render.cu k_project /
    rec_tile_range): a pixel can pass the reference's weight
    test (_composite.pyx:53-60) only if e <= t = ln(alpha/EPS), and
    min_dy e(dx, dy) = dx^2 / (2 Sxx), so |dx| > sqrt(2 t Sxx) rejects it.
    The half-extents are padded outwards (relative and absolute, in fp64, then
    cast to fp32 and padded again), and the clipped bbox is intersected with
    the pixel centres inside them.  Returns int64 (k, 4) [u0, u1, v0, v1] and a
    bool (k,) mask of primitives that reach at least one tile."""
    a2, c2, det = pr.cov2d[:, 0], pr.cov2d[:, 2], pr.det
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.log(pr.alphas / EPS_CONTRIB) * 1.0002 + 2e-4
        hx = np.sqrt(2.0 * np.maximum(t, 0.0) * (a2 + 1e-9 * a2)) * 1.0002 + 1e-3
        hy = np.sqrt(2.0 * np.maximum(t, 0.0) * (c2 + 1e-9 * c2)) * 1.0002 + 1e-3
    f32 = np.float32
    ok_x = (det > 0) & np.isfinite(hx)
    ok_y = (det > 0) & np.isfinite(hy)
    hxf = np.where(ok_x, hx.astype(f32) * f32(1.0001), f32(1e30)).astype(f32)
    hyf = np.where(ok_y, hy.astype(f32) * f32(1.0001), f32(1e30)).astype(f32)
    bb = pr.bboxes
    xa, xb, ya, yb = bb[:, 0].copy(), bb[:, 1] - 1, bb[:, 2].copy(), bb[:, 3] - 1
    mxf = (pr.means2d[:, 0] - 0.5).astype(f32)
    myf = (pr.means2d[:, 1] - 0.5).astype(f32)
    nx = hxf < f32(1e29)
    ny = hyf < f32(1e29)
    xa = np.where(nx, np.maximum(xa, np.ceil(mxf - hxf).astype(np.int64)), xa)
    xb = np.where(nx, np.minimum(xb, np.floor(mxf + hxf).astype(np.int64)), xb)
    ya = np.where(ny, np.maximum(ya, np.ceil(myf - hyf).astype(np.int64)), ya)
    yb = np.where(ny, np.minimum(yb, np.floor(myf + hyf).astype(np.int64)), yb)
    has = (bb[:, 1] > bb[:, 0]) & (bb[:, 3] > bb[:, 2]) & (xa <= xb) & (ya <= yb)
    rng = np.stack([xa // tile, xb // tile, ya // tile, yb // tile], axis=1)
    if with_ext:
        return rng, has, nx & ny
    return rng, has


def _quad_rect_min_lb32(A, B, C, rX, rY, x0, x1, y0, y1):
    """float32 restatement, op for op, of render.cu quad_rect_min_lb (the CUDA
    code is compiled without FMA contraction): a conservative lower bound of
    min A dx^2 + B dx dy + C dy^2 over [x0, x1] x [y0, y1], the edge vertices
    from the reciprocals rX = 1/(2C), rY = 1/(2A).  Arrays."""
    f = np.float32

    def edge(P, Q, r, X, lo, hi):
        with np.errstate(invalid="ignore", over="ignore"):
            t = np.minimum(np.maximum(((-B) * X) * r, lo), hi)
            a = (P * X) * X
            b = (B * X) * t
            c = (Q * t) * t
            return ((a + b) + c) - (f(1e-4) * ((a + np.abs(b)) + c) + f(1e-3))

    ex = np.minimum(edge(A, C, rX, x0, y0, y1), edge(A, C, rX, x1, y0, y1))
    ey = np.minimum(edge(C, A, rY, y0, x0, x1), edge(C, A, rY, y1, x0, x1))
    lb = np.minimum(ex, ey)
    inside = (x0 <= 0) & (x1 >= 0) & (y0 <= 0) & (y1 >= 0)
    return np.where(inside, f(0.0), lb).astype(f)


def ellipse_tile_keep(pr, rng, ok_ext, tile=TILE):
    """render.cu make_cull_rec / cull_keep restated: for primitives whose
    threshold tile range spans 2..4 tiles in both directions (with threshold
    extents and a positive definite fp32 conic), the binning drops a tile
    when a lower bound of e over the tile's pixel centres exceeds
    t = ln(alpha/EPS) (+ pad): no pixel there can pass the weight test.
    Returns keep(i, u, v), vectorised over primitive positions and tiles."""
    f32 = np.float32
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.maximum(np.log(pr.alphas / EPS_CONTRIB) * 1.0002 + 2e-4, 0.0)
    nu = rng[:, 1] - rng[:, 0] + 1
    nv = rng[:, 3] - rng[:, 2] + 1
    A = (0.5 * pr.conics[:, 0]).astype(f32)
    B = pr.conics[:, 1].astype(f32)
    C = (0.5 * pr.conics[:, 2]).astype(f32)
    cull = ok_ext & (nu >= 2) & (nv >= 2) & (nu <= 4) & (nv <= 4) & (A > 0) & (C > 0)
    with np.errstate(divide="ignore"):
        rX = (f32(1.0) / (f32(2.0) * C)).astype(f32)
        rY = (f32(1.0) / (f32(2.0) * A)).astype(f32)
    tf = t.astype(f32)
    mx = ((pr.means2d[:, 0] - rng[:, 0] * tile).astype(f32) - f32(0.5)).astype(f32)
    my = ((pr.means2d[:, 1] - rng[:, 2] * tile).astype(f32) - f32(0.5)).astype(f32)

    def keep(i, u, v):
        du, dv = u - rng[i, 0], v - rng[i, 2]
        x0 = ((du * tile).astype(f32) - mx[i]).astype(f32)
        x1 = ((du * tile + tile - 1).astype(f32) - mx[i]).astype(f32)
        y0 = ((dv * tile).astype(f32) - my[i]).astype(f32)
        y1 = ((dv * tile + tile - 1).astype(f32) - my[i]).astype(f32)
        lb = _quad_rect_min_lb32(A[i], B[i], C[i], rX[i], rY[i], x0, x1, y0, y1)
        return ~cull[i] | ~(lb > tf[i])

    return keep


def tile_lists_threshold(params, cam, tile=TILE, ellipse=True):
    """Expected per-tile lists of the B200 binning + sort stage for one view:
    ``tile_keys`` over the reference's clipped bboxes,
    restricted to the tiles of ``threshold_tile_ranges`` and (``ellipse``)
    to the tiles ``ellipse_tile_keep`` keeps, mapped back to primitive
    indices.  Returns {tile_id: int64 array of primitive indices in
    compositing order (prep.order position ascending)}."""
    pr = prepare(params, cam)
    ct = CamTerms(cam)
    keys = tile_keys(pr.bboxes, ct.W, ct.H, tile)
    rng, has, ok_ext = threshold_tile_ranges(pr, tile, with_ext=True)
    tx_n = (ct.W + tile - 1) // tile
    tid = keys >> 32
    pos = keys & 0xFFFFFFFF
    tyy, txx = tid // tx_n, tid % tx_n
    r = rng[pos]
    keep = has[pos] & (txx >= r[:, 0]) & (txx <= r[:, 1]) & (tyy >= r[:, 2]) & (tyy <= r[:, 3])
    if ellipse:
        kk = np.nonzero(keep)[0]
        keep[kk] = ellipse_tile_keep(pr, rng, ok_ext, tile)(pos[kk], txx[kk], tyy[kk])
    tid, pos = tid[keep], pos[keep]
    out = {}
    if tid.size:
        cuts = np.nonzero(np.diff(tid))[0] + 1
        for a, b in zip(np.r_[0, cuts], np.r_[cuts, tid.size]):
            out[int(tid[a])] = pr.order[pos[a:b]]
    return out


def render_full(params, cam, pixel_major=False):
    """(clipped image, usage over all n primitives) -- ss/rasterizer.py:215-240."""
    pr = prepare(params, cam)
    ct = CamTerms(cam)
    img, _, us = composite(pr.means2d, pr.conics, pr.alphas, pr.colors, pr.bboxes, ct.H, ct.W, pixel_major)
    counts = np.zeros(np.asarray(params).shape[0], dtype=np.int64)
    counts[pr.order] += us
    return np.clip(img, 0.0, 1.0), counts


def render(params, cam):
    return render_full(params, cam)[0]


def render_with_usage(params, cams):
    cams = list(cams)
    if not cams:
        raise OracleError("StructuralError", "at least one camera required")
    counts = np.zeros(np.asarray(params).shape[0], dtype=np.int64)
    images = []
    for cam in cams:
        img, c = render_full(params, cam)
        images.append(img)
        counts += c
    return images, counts


def psnr(a, b):  # ss/metrics.py:37-43
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise OracleError("StructuralError", f"resolution mismatch: {a.shape} vs {b.shape}")
    mse = float(np.mean((a - b) ** 2))
    if mse <= 0.0:
        return PSNR_CAP_DB
    return min(PSNR_CAP_DB, 10.0 * np.log10(1.0 / mse))


def frame_quality(params, cams, targets):  # ss/grouping.py:153-159
    return float(np.mean([psnr(render(params, c), t) for c, t in zip(cams, targets)]))


# ---------------------------------------------------------------------------
# GSAI attribute images (ss/codec.py:61-169)


def gsai_encode(params, frame_index=0, group_key=0, width=None, height=None):
    P = np.asarray(params, dtype=np.float64)
    n, m = P.shape
    if width is None or height is None:
        side = math.ceil(math.sqrt(n))
        width = width or side
        height = height or side
    if n > width * height:
        raise OracleError("CapacityError", f"{n} primitives exceed {width}x{height} image capacity")
    planes = np.zeros((m, width * height), dtype="<u2")
    scales = np.zeros(m)
    offsets = np.zeros(m)
    for j in range(m):
        lo, hi = float(P[:, j].min()), float(P[:, j].max())
        offsets[j] = lo
        if hi != lo:
            scales[j] = (hi - lo) / QMAX
            planes[j, :n] = np.clip(np.rint((P[:, j] - lo) / scales[j]), 0, QMAX).astype(np.uint16)
    blob = bytearray(GSAI_HEADER.pack(GSAI_MAGIC, 1, n, m, width, height, 16))
    blob += struct.pack("<II", frame_index, group_key)
    for j in range(m):
        blob += struct.pack("<dd", scales[j], offsets[j])
        blob += planes[j].tobytes()
    return bytes(blob)


def gsai_parse(blob):
    """-> (planes u16 (m, h*w), scales, offsets, n, frame_index, group_key, w, h)."""
    if len(blob) < GSAI_HEADER.size:
        raise OracleError("DecodeError", "attribute image container too short")
    magic, ver, n, m, w, h, depth = GSAI_HEADER.unpack_from(blob, 0)
    if magic != GSAI_MAGIC:
        raise OracleError("DecodeError", f"bad attribute-image magic {magic!r}")
    if ver != 1 or depth != 16:
        raise OracleError("DecodeError", "unsupported attribute-image version or bit depth")
    fi, gk = struct.unpack_from("<II", blob, GSAI_HEADER.size)
    pos = GSAI_HEADER.size + 8
    planes = np.empty((m, w * h), dtype=np.uint16)
    scales = np.empty(m)
    offsets = np.empty(m)
    for j in range(m):
        if pos + 16 + 2 * w * h > len(blob):
            raise OracleError("DecodeError", "truncated attribute image container")
        scales[j], offsets[j] = struct.unpack_from("<dd", blob, pos)
        planes[j] = np.frombuffer(blob, dtype="<u2", count=w * h, offset=pos + 16)
        pos += 16 + 2 * w * h
    return planes, scales, offsets, n, fi, gk, w, h


def gsai_decode(blob):
    planes, scales, offsets, n, fi, gk, _, _ = gsai_parse(blob)
    sh_degree_of(planes.shape[0])
    q = planes[:, :n].astype(np.float64)
    return (q * scales[:, None] + offsets[:, None]).T.copy(), fi, gk


# ---------------------------------------------------------------------------
# GSDP delta payloads (ss/codec.py:32-58,187-248)


def varint(v):
    out = bytearray()
    while v > 0x7F:
        out.append((v & 0x7F) | 0x80)
        v >>= 7
    out.append(v)
    return bytes(out)


def varint_len(v):
    v = np.asarray(v, dtype=np.uint64)
    n = np.ones(v.shape, dtype=np.int64)
    t = v >> np.uint64(7)
    while np.any(t):
        n += (t != 0)
        t = t >> np.uint64(7)
    return n


def quantize(rows, step):
    """Per-row fixed point and the keep mask (ss/codec.py:193-199)."""
    if step <= 0:
        raise OracleError("StructuralError", "quant_step must be positive")
    rows = np.asarray(rows, dtype=np.float64)
    q = np.rint(rows / step).astype(np.int64) if rows.size else np.zeros(rows.shape, np.int64)
    keep = np.any(q != 0, axis=1) if rows.size else np.zeros(rows.shape[0], bool)
    if np.any(np.abs(q[keep]) > 2**31 - 1):
        bad = int(np.nonzero(keep & np.any(np.abs(q) > 2**31 - 1, axis=1))[0][0])
        raise OracleError("StructuralError", f"delta at {bad} overflows i32 fixed point")
    return q, keep


def gsdp_encode(idx, rows, step, frame_index=0, base_key=0):
    idx = np.asarray(idx, dtype=np.int64)
    q, keep = quantize(rows, step)
    ki, kq = idx[keep], q[keep].astype("<i4")
    blob = bytearray(GSDP_HEADER.pack(GSDP_MAGIC, frame_index, base_key, ki.size, step))
    prev = 0
    for i in ki.tolist():
        blob += varint(i - prev)
        prev = i
    blob += kq.tobytes()
    return bytes(blob)


def gsdp_size(idx, rows, step):
    """Exact wire size without emitting bytes."""
    idx = np.asarray(idx, dtype=np.int64)
    _, keep = quantize(rows, step)
    ki = idx[keep]
    if ki.size == 0:
        return GSDP_HEADER.size
    gaps = np.diff(np.concatenate([[0], ki]))
    width = np.asarray(rows).shape[1]
    return int(GSDP_HEADER.size + varint_len(gaps).sum() + 4 * width * ki.size)


def gsdp_decode(blob, base_count=None, width=None):
    """-> (idx, rows, frame_index, base_key, step, base_count, width).

    Duplicate indices (zero gaps) keep the last row, as the reference's dict
    comprehension does (ss/codec.py:247)."""
    if len(blob) < GSDP_HEADER.size:
        raise OracleError("DecodeError", "delta payload shorter than its header")
    magic, fi, bk, cnt, step = GSDP_HEADER.unpack_from(blob, 0)
    if magic != GSDP_MAGIC:
        raise OracleError("DecodeError", f"bad delta magic {magic!r}")
    pos = GSDP_HEADER.size
    idx = []
    prev = 0
    for _ in range(cnt):
        val, shift = 0, 0
        while True:
            if pos >= len(blob):
                raise OracleError("DecodeError", "truncated varint")
            byte = blob[pos]
            pos += 1
            val |= (byte & 0x7F) << shift
            if not byte & 0x80:
                break
            shift += 7
            if shift > 63:
                raise OracleError("DecodeError", "varint too long")
        prev += val
        idx.append(prev)
    rem = len(blob) - pos
    if width is None:
        if cnt == 0:
            raise OracleError("DecodeError", "param_width required to decode an empty delta")
        if rem % (4 * cnt):
            raise OracleError("DecodeError", "delta payload length inconsistent with entry count")
        width = rem // (4 * cnt)
    if rem != 4 * cnt * width:
        raise OracleError("DecodeError", "truncated delta payload")
    q = np.frombuffer(blob, dtype="<i4", count=cnt * width, offset=pos).reshape(cnt, width)
    if base_count is None:
        base_count = idx[-1] + 1 if idx else 0
    idx = np.array(idx, dtype=np.int64)
    live = np.ones(cnt, dtype=bool)
    if cnt > 1:
        live[:-1] = idx[1:] != idx[:-1]
    if np.any((idx < 0) | (idx >= base_count)):
        bad = int(idx[(idx < 0) | (idx >= base_count)][0])
        raise OracleError("StructuralError", f"delta index {bad} out of range")
    return idx[live], q[live].astype(np.float64) * step, fi, bk, step, base_count, width


# ---------------------------------------------------------------------------
# sparse delta algebra (ss/model.py:241-311)


def compose(deltas, eps=EPS_SPARSE):
    """Union-sum in list order, one eps filter at the end (ss/model.py:294-311)."""
    deltas = [(np.asarray(i, np.int64), np.asarray(r, np.float64)) for i, r in deltas]
    if not deltas:
        return np.zeros(0, np.int64), np.zeros((0, 17))
    width = deltas[0][1].shape[1] if deltas[0][1].ndim == 2 else 17
    allidx = np.unique(np.concatenate([d[0] for d in deltas])) if deltas else np.zeros(0, np.int64)
    acc = np.zeros((allidx.size, width))
    seen = np.zeros(allidx.size, dtype=bool)
    for idx, rows in deltas:
        pos = np.searchsorted(allidx, idx)
        first = ~seen[pos]
        acc[pos[first]] = rows[first]
        acc[pos[~first]] = acc[pos[~first]] + rows[~first]
        seen[pos] = True
    keep = np.max(np.abs(acc), axis=1) > eps if acc.size else np.zeros(0, bool)
    return allidx[keep], acc[keep]


def apply(canonical, idx, rows):  # ss/model.py:269-284
    out = np.array(canonical, dtype=np.float64, copy=True)
    out[np.asarray(idx, np.int64)] += rows
    return out


def from_dense(dense, eps=EPS_SPARSE):  # ss/model.py:262-266
    dense = np.asarray(dense, dtype=np.float64)
    keep = np.max(np.abs(dense), axis=1) > eps
    return np.nonzero(keep)[0].astype(np.int64), dense[keep]


# ---------------------------------------------------------------------------
# pruning (ss/pruning.py:72-210)


def prune_order(idx, usage):
    """Entries by (usage asc, index desc) -- ss/pruning.py:72-76."""
    idx = np.asarray(idx, dtype=np.int64)
    u = np.asarray(usage, dtype=np.int64)[idx]
    return idx[np.lexsort((-idx, u))]


def prune(idx, rows, usage, ratio):
    order = prune_order(idx, usage)
    k = int(math.floor(ratio * len(order) + 0.5))
    removed = np.sort(order[:k])
    keep = ~np.isin(idx, removed)
    return np.asarray(idx)[keep], np.asarray(rows)[keep], removed


def level_plan(gap, canonical, ratios, usage, step, base=None):
    """The render-free half of build_level_space (ss/pruning.py:93-126):
    returns (reference params, [(ratio, size_bytes, removed, level params)])
    for the surviving (strictly shrinking) levels."""
    ratios = sorted(set(float(r) for r in ratios))
    if not ratios or ratios[0] != 0.0:
        raise OracleError("StructuralError", "ratios must include 0")
    gi, gr = gap
    width = np.asarray(canonical).shape[1]
    gr = np.asarray(gr, dtype=np.float64).reshape(-1, width)

    def recon(di, dr):
        if base is not None and len(base[0]):
            ci, cr = compose([base, (di, dr)])
        else:
            ci, cr = di, dr
        return apply(canonical, ci, cr)

    def dec(i, r):
        q, keep = quantize(r, step)
        return np.asarray(i)[keep], q[keep].astype(np.float64) * step

    ref = recon(*dec(gi, gr))
    out = []
    last = None
    for r in ratios:
        ki, kr, removed = prune(gi, gr, usage, r)
        size = gsdp_size(ki, kr, step)
        if last is not None and size >= last:
            continue
        out.append((r, size, removed, recon(*dec(ki, kr))))
        last = size
    return ref, out


def level_space(gap, canonical, cams, ratios, usage, step, base=None):
    """-> list of (ratio, quality_db, size_bytes, removed) (ss/pruning.py:93-137)."""
    ref, plan = level_plan(gap, canonical, ratios, usage, step, base)
    ref_imgs = [render(ref, c) for c in cams]
    return [(r, float(np.mean([psnr(render(fr, c), im) for c, im in zip(cams, ref_imgs)])), size, removed)
            for r, size, removed, fr in plan]


def select_level(qualities, sizes, bandwidth_B, rate_R, beta=2.0):
    """Algorithm 1: cliff scan + binary search (ss/pruning.py:140-178)."""
    L = len(qualities)
    if L == 1:
        return 0
    prev = qualities[0] - qualities[1]
    cand = [0]
    for i in range(1, L):
        drop = qualities[i - 1] - qualities[i]
        if drop / max(prev, MIN_DROP) > beta:
            break
        cand.append(i)
        prev = drop
    budget = bandwidth_B / rate_R / 8.0
    lo, hi, best = 0, len(cand) - 1, None
    while lo <= hi:
        mid = (lo + hi) // 2
        if sizes[cand[mid]] <= budget:
            best, hi = cand[mid], mid - 1
        else:
            lo = mid + 1
    return best if best is not None else L - 1


def ilp(spaces, budgets):
    """Separable exact optimum: per frame argmax quality under budget
    (ss/pruning.py:189-210).  spaces: list of (qualities, sizes)."""
    res = []
    for (qs, ss), b in zip(spaces, budgets):
        best = None
        for j, (q, s) in enumerate(zip(qs, ss)):
            if s <= b and (best is None or q > qs[best]):
                best = j
        res.append(best)
    return res
