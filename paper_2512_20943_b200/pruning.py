"""Usage-frequency pruning on device (drop-in for ``ss/pruning.py``).

``build_level_space`` runs entirely in HBM: quantise the gap once
(decode(encode(.)) values and the survive mask), order entries by
(usage asc, index desc) with a radix sort, compute every level's exact GSDP
size in one kernel, then materialise each surviving level's frame with the
pruning-level selector folded into ``apply`` and evaluate all (level, view)
pairs in one batched render whose SSE against the unpruned reconstruction is
fused into compositing.  Only level sizes, per-view SSE and (for the API
result) the pruned index sets come back to the host.

``select_pruning_level`` (Algorithm 1) and ``ilp_optimal`` are scalar
host logic over the level table, as in the reference.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import device as dv
from .codec import quantize_overlay
from .errors import StructuralError, ValidationError
from .metrics import psnr_from_sse
from .model import EPS_SPARSE, CanonicalSpace, DeltaTensor, _compose_call, apply_overlay, as_delta, as_space

MIN_DROP = 1e-12


class PruningLevel:
    __slots__ = ("ratio", "quality_db", "size_bytes", "pruned_indices")

    def __init__(self, ratio, quality_db, size_bytes, pruned_indices):
        object.__setattr__(self, "ratio", ratio)
        object.__setattr__(self, "quality_db", quality_db)
        object.__setattr__(self, "size_bytes", size_bytes)
        object.__setattr__(self, "pruned_indices", tuple(pruned_indices))

    def __setattr__(self, k, v):
        raise AttributeError("PruningLevel is immutable")

    def __eq__(self, o):
        return isinstance(o, PruningLevel) and (self.ratio, self.quality_db, self.size_bytes,
                                                 self.pruned_indices) == (o.ratio, o.quality_db, o.size_bytes,
                                                                          o.pruned_indices)

    def __repr__(self):
        return (f"PruningLevel(ratio={self.ratio}, quality_db={self.quality_db}, size_bytes={self.size_bytes}, "
                f"pruned={len(self.pruned_indices)})")


class PruningLevelSpace:
    __slots__ = ("levels", "frame_index")

    def __init__(self, levels, frame_index):
        levels = tuple(levels)
        if not levels or levels[0].ratio != 0.0:
            raise StructuralError("level space must start at ratio 0")
        if any(b.ratio <= a.ratio for a, b in zip(levels, levels[1:])):
            raise StructuralError("ratios must be strictly increasing")
        if any(b.size_bytes >= a.size_bytes for a, b in zip(levels, levels[1:])):
            raise StructuralError("sizes must be strictly decreasing")
        object.__setattr__(self, "levels", levels)
        object.__setattr__(self, "frame_index", frame_index)

    def __setattr__(self, k, v):
        raise AttributeError("PruningLevelSpace is immutable")

    def qualities(self):
        return [lv.quality_db for lv in self.levels]

    def sizes(self):
        return [lv.size_bytes for lv in self.levels]


class SelectionContext:
    __slots__ = ("bandwidth_B", "target_rate_R", "cliff_beta")

    def __init__(self, bandwidth_B, target_rate_R, cliff_beta=2.0):
        if bandwidth_B <= 0 or target_rate_R <= 0 or cliff_beta <= 0:
            raise ValidationError("selection context values must be positive")
        object.__setattr__(self, "bandwidth_B", bandwidth_B)
        object.__setattr__(self, "target_rate_R", target_rate_R)
        object.__setattr__(self, "cliff_beta", cliff_beta)

    def __setattr__(self, k, v):
        raise AttributeError("SelectionContext is immutable")

    @property
    def budget_bytes(self) -> float:
        """C = B / R bits per frame, in bytes."""
        return self.bandwidth_B / self.target_rate_R / 8.0


class FrameSelection:
    __slots__ = ("frame_index", "level", "quality_db", "feasible")

    def __init__(self, frame_index, level, quality_db, feasible):
        for k, v in (("frame_index", frame_index), ("level", level), ("quality_db", quality_db),
                     ("feasible", feasible)):
            object.__setattr__(self, k, v)

    def __setattr__(self, k, v):
        raise AttributeError("FrameSelection is immutable")

    def __eq__(self, o):
        return isinstance(o, FrameSelection) and (self.frame_index, self.level, self.quality_db, self.feasible) == (
            o.frame_index, o.level, o.quality_db, o.feasible)

    def __repr__(self):
        return f"FrameSelection({self.frame_index}, {self.level}, {self.quality_db}, {self.feasible})"


# ---------------------------------------------------------------------------
# device helpers


RENDER_PAIRS_PER_CALL = 96 * 1024 * 1024  # ~9 GB of 96-byte projected records per render call


def _engine(dev):
    from ._lib import engine

    return engine(dev)


def _ptr(t):
    from ._lib import ptr

    return ptr(t)


def _usage_tensor(usage, n, dev):
    import torch

    counts = usage.counts if hasattr(usage, "counts") else usage
    if isinstance(counts, torch.Tensor):
        if counts.shape[0] < n:
            raise StructuralError("usage counts do not cover the primitive set")
        return counts[:n].to(device=dev, dtype=torch.int64).contiguous()
    counts = np.asarray(counts)
    if counts.shape[0] < n:
        raise StructuralError("usage counts do not cover the primitive set")
    return torch.from_numpy(np.ascontiguousarray(counts[:n].astype(np.int64))).to(dev)


def prune_ranks(ov: dv.Overlay, usage_t):
    """rank[i] = position of entry i in the (usage asc, index desc) order;
    INT32_MAX for absent.  Returns (rank tensor, entry count)."""
    import torch

    eng = _engine(ov.rows.device)
    rank = torch.empty((ov.ld,), dtype=torch.int32, device=ov.rows.device)
    cnt = ctypes.c_int64(0)
    eng.call("airgs_prune_rank", _ptr(ov.present), _ptr(usage_t), ov.n, _ptr(rank), ctypes.byref(cnt), eng.stream())
    return rank, int(cnt.value)


def level_sizes(nz, rank, n, width, kmins, dev):
    eng = _engine(dev)
    L = len(kmins)
    k = (ctypes.c_int64 * L)(*[int(v) for v in kmins])
    out = (ctypes.c_int64 * L)()
    eng.call("airgs_level_sizes", _ptr(nz), _ptr(rank), n, width, k, L, out, eng.stream())
    return [int(v) for v in out]


def _k_of(ratio, entries):
    return int(math.floor(ratio * entries + 0.5))


# ---------------------------------------------------------------------------
# reference API


def prune_order(delta: DeltaTensor, usage_counts) -> list:
    """Entry indices, lowest usage first, ties prune the higher index first
    (ss/pruning.py:72-76)."""
    delta = as_delta(delta)
    ov = delta.overlay()
    if ov.n == 0:
        return []
    rank, e = prune_ranks(ov, _usage_tensor(usage_counts, ov.n, ov.rows.device))
    idx, _ = ov.entries()
    r = rank[: ov.n].cpu().numpy()[idx]
    return [int(i) for i in idx[np.argsort(r, kind="stable")]]


def prune_delta(delta: DeltaTensor, usage_counts, ratio: float):
    """Remove the ``ratio`` fraction of lowest-usage entries
    (ss/pruning.py:79-90).  Returns (kept DeltaTensor, sorted removed tuple)."""
    delta = as_delta(delta)
    ov = delta.overlay()
    if ov.n == 0:
        return DeltaTensor(delta.base_count, delta.param_width, {}), ()
    rank, e = prune_ranks(ov, _usage_tensor(usage_counts, ov.n, ov.rows.device))
    k = _k_of(ratio, e)
    keep = (rank >= k).to(ov.present.dtype) * ov.present
    kept = DeltaTensor(delta.base_count, delta.param_width,
                       overlay=dv.Overlay(ov.rows, keep, ov.n, ov.width))
    removed_mask = (ov.present.bool() & (rank < k))[: ov.n]
    removed = tuple(int(i) for i in np.nonzero(removed_mask.cpu().numpy())[0])
    return kept, removed


class LevelPlan:
    """Device state shared by every pruning level of one gap (see
    ``build_level_space``)."""

    __slots__ = ("canon", "n", "width", "A", "B", "nz", "rank", "entries", "idx_host", "rank_host")


def plan_levels(delta: DeltaTensor, space: CanonicalSpace, usage, quant_step: float, base: DeltaTensor = None):
    import torch

    fr = space.frame
    dev = dv.device_of(None)
    n, w = fr.count, fr.width
    canon = fr.planes(dev)
    G = delta.overlay(dev)
    usage_t = _usage_tensor(usage, n, dev)
    nz, D = quantize_overlay(G, quant_step, want_decoded=True)
    eng = _engine(dev)
    Dov = dv.Overlay(D, nz, n, w)
    if base is not None and not base.is_empty():
        Bov = base.overlay(dev)
        A = dv.Overlay.empty(n, w, dev)
        _compose_call(eng, [(Bov.rows, Bov.present, 1.0), (Dov.rows, Dov.present, 1.0)], n, w, A.ld, EPS_SPARSE,
                      True, A)
        Bonly = dv.Overlay.empty(n, w, dev)
        _compose_call(eng, [(Bov.rows, Bov.present, 1.0)], n, w, Bonly.ld, EPS_SPARSE, True, Bonly)
    else:
        A, Bonly = Dov, None
    rank, entries = prune_ranks(G, usage_t)
    p = LevelPlan()
    p.canon, p.n, p.width = canon, n, w
    p.A, p.B, p.nz, p.rank, p.entries = A, Bonly, nz, rank, entries
    p.idx_host = None
    p.rank_host = None
    return p


def level_frame_planes(p: LevelPlan, kmin):
    """Parameters of the level that prunes ranks < kmin (None: unpruned)."""
    if kmin is None:
        return apply_overlay(p.canon, p.n, p.A)
    return apply_overlay(p.canon, p.n, p.A, sel=p.nz, rank=p.rank, keep_min=int(kmin), ov_b=p.B)


def _removed_prepare(p: LevelPlan, G):
    """Entry indices (ascending) and their prune ranks on the host: two small
    downloads (the rows themselves stay on the device)."""
    if p.idx_host is None:
        import torch

        idx = torch.nonzero(G.present[: G.n]).flatten()
        p.idx_host = idx.cpu().numpy().astype(np.int64)
        p.rank_host = p.rank[idx].cpu().numpy() if idx.numel() else np.zeros(0, dtype=np.int32)


def _removed_sets(p: LevelPlan, G, kmins):
    _removed_prepare(p, G)
    return [tuple(p.idx_host[p.rank_host < k].tolist()) for k in kmins]


class LevelTable:
    """Validated inputs and the size-only half of a level space: the device
    plan, every requested ratio's entry cut ``kmin``, exact payload sizes,
    the surviving (strictly shrinking) levels and their pruned index sets."""

    __slots__ = ("plan", "ratios", "kmins", "sizes", "keep", "removed", "delta")


def level_table(delta, space, ratios, usage, quant_step: float, base=None, removed=True) -> LevelTable:
    """Input normalisation and checks of ``build_level_space``
    (ss/pruning.py:93-126), shared by the single-GPU and sharded drivers.
    ``removed=False`` leaves the pruned index sets to ``level_removed`` (the
    drivers build them on the host while the level renders run)."""
    delta, space = as_delta(delta), as_space(space)
    base = None if base is None else as_delta(base)
    ratios = sorted(set(float(r) for r in ratios))
    if not ratios or ratios[0] != 0.0:
        raise StructuralError("ratios must include 0")
    counts = usage.counts if hasattr(usage, "counts") else usage
    if len(counts) < space.frame.count:
        raise StructuralError("usage counts do not cover the primitive set")
    if delta.base_count != space.frame.count:
        raise StructuralError(f"delta base_count {delta.base_count} != space count {space.frame.count}")
    if not quant_step > 0:
        raise StructuralError("quant_step must be positive")
    t = LevelTable()
    t.plan = p = plan_levels(delta, space, usage, quant_step, base)
    t.ratios = ratios
    t.kmins = [_k_of(r, p.entries) for r in ratios]
    t.sizes = level_sizes(p.nz, p.rank, p.n, p.width, t.kmins, p.canon.device)
    t.keep, last = [], None
    for j, s in enumerate(t.sizes):
        if last is not None and s >= last:
            continue  # duplicate level (ss/pruning.py:125-126)
        t.keep.append(j)
        last = s
    t.removed = None
    t.delta = delta
    if removed:
        level_removed(t)
    return t


def level_removed(t: LevelTable):
    """The surviving levels' pruned index sets (sorted tuples, as the
    reference's PruningLevel.pruned_indices)."""
    if t.removed is None:
        t.removed = _removed_sets(t.plan, t.delta.overlay(), [t.kmins[j] for j in t.keep])
    return t.removed


def render_sse_chunked(frames, cams, items, targets, device=None, host=True, tile_skip=None):
    """SSE of (frame, view) items against their targets, at most
    RENDER_PAIRS_PER_CALL (item, primitive) records per render call (C5: 2M
    primitives x 8 levels x 32 views would not fit one call's scratch).
    ``host=False`` returns the device tensor without synchronising."""
    import torch

    from .rasterizer import render_views

    if not items:
        return np.zeros(0) if host else None
    n = max(fr.count for fr in frames)
    per_call = max(1, RENDER_PAIRS_PER_CALL // max(n, 1))
    parts = [render_views(frames, cams, items[k:k + per_call], targets=targets[k:k + per_call], device=device,
                          tile_skip=None if tile_skip is None else tile_skip[k:k + per_call]).sse
             for k in range(0, len(items), per_call)]
    sse = torch.cat(parts) if len(parts) > 1 else parts[0]
    return sse.cpu().numpy() if host else sse


def tile_skip_enabled() -> bool:
    """Clean-tile skip of the level renders (default on; AIRGS_LEVEL_TILE_SKIP=0
    renders every tile, for A/B checks -- the qualities are bit-identical)."""
    import os

    return os.environ.get("AIRGS_LEVEL_TILE_SKIP", "1") != "0"


def tile_footprint(p: LevelPlan, cams, rank_cap: int):
    """minrank[v] (device int32 [tiles of view v]): the lowest prune rank of
    an entry whose primitive reaches that tile of view v in the unpruned
    reference render or with its entry pruned.  A level pruning ranks < k
    changes only primitives of rank < k, so every tile with minrank >= k
    composites exactly as in the reference render: SSE 0 without rendering
    (the reference re-renders whole levels, ss/pruning.py:122-131)."""
    import torch

    from ._lib import CameraC, FrameC
    from .camera import camera_struct

    dev = p.canon.device
    eng = _engine(dev)
    cams = list(cams)
    tiles = [((c.resolution[0] + 15) // 16) * ((c.resolution[1] + 15) // 16) for c in cams]
    stride = max(tiles)
    minrank = torch.full((len(cams), stride), 2**31 - 1, dtype=torch.int32, device=dev)
    cc = (CameraC * len(cams))(*[camera_struct(c) for c in cams])
    planes = [level_frame_planes(p, None), level_frame_planes(p, 2**31 - 1)]
    for pl in planes:
        fc = FrameC(pl.data_ptr(), p.n, pl.shape[1], p.width, 0)
        eng.call("airgs_tile_footprint", ctypes.byref(fc), cc, len(cams), _ptr(p.rank), int(rank_cap),
                 _ptr(minrank), stride, eng.stream())
    return [minrank[v, :tiles[v]] for v in range(len(cams))], planes


def deferred(dev, run):
    """Run ``run()`` (device work that may synchronise only at its end) under
    deferred checking: the calls enqueue without host round trips and fold
    any problem into one device word; if it is set, ``run()`` is repeated in
    checked mode, which raises the reference's exact error or handles the
    condition (bucket overflow).  Returns run()'s result."""
    return deferred_lanes(dev, lambda nl: run(), 1)


def deferred_lanes(dev, run, lanes):
    """deferred() over ``lanes`` engine lanes: ``run(nl)`` may spread its calls
    over nl lanes (grouping's lane streams); every lane engine folds its
    problems into its own word.  The checked re-run keeps the lanes: a
    checked call synchronises on its own flags, so errors still surface in
    call order, and every lane engine adapts its tile-bucket capacity after
    an overflow (a deferred call cannot)."""
    from ._lib import engine, engine_lane

    engs, flags = [], []
    for lane in range(lanes):
        with engine_lane(lane):
            engs.append(engine(dev))
        flags.append(ctypes.c_uint32(0))
    for e, f in zip(engs, flags):
        e.call("airgs_defer", 1, ctypes.byref(f))
    try:
        out = run(lanes)
    finally:
        for e, f in zip(engs, flags):
            e.call("airgs_defer", 0, ctypes.byref(f))
    if any(f.value for f in flags):
        out = run(lanes)
    return out


def build_level_space(delta: DeltaTensor, space: CanonicalSpace, cams, ratios, usage, quant_step: float,
                      base: DeltaTensor = None, frame_index: int = 0) -> PruningLevelSpace:
    """Dense (quality, size) space over pruning ratios (ss/pruning.py:93-137).

    Quality of a level = mean over ``cams`` of PSNR of its reconstruction
    against the unpruned quantised reconstruction; sizes are exact GSDP
    payload sizes; a level whose size does not shrink is dropped.  The
    reference render and every (level, view) render are enqueued under
    deferred checking; the pruned index sets are built on the host while they
    run, and one synchronisation reads the SSE.
    """
    from .model import GaussianFrame
    from .rasterizer import render_views

    space = as_space(space)
    t = level_table(delta, space, ratios, usage, quant_step, base, removed=False)
    p = t.plan
    cams = list(cams)
    qualities = [100.0] * len(t.keep)
    if cams:
        dev = p.canon.device
        # a level that prunes no entry has the reference's parameters bit for bit:
        # SSE 0, the reference's 100 dB cap, no render (the mandatory ratio-0 level,
        # ss/pruning.py:102-104)
        todo = [li for li, j in enumerate(t.keep) if t.kmins[j] > 0]
        V = len(cams)
        skip = tile_skip_enabled()

        def run(nl):
            import torch

            from ._lib import engine_lane
            from .grouping import _lane_stream

            kmins = [t.kmins[t.keep[li]] for li in todo]
            if skip:
                minrank, (ref_planes, _) = tile_footprint(p, cams, max(kmins))
            else:
                minrank, ref_planes = None, level_frame_planes(p, None)
            ref = GaussianFrame(device_params=ref_planes, count=p.n, frame_index=frame_index,
                                group_key=space.key_index)
            rv = render_views([ref], cams, [(0, v) for v in range(V)], want_images=True, device=dev)
            frames = [GaussianFrame(device_params=level_frame_planes(p, k), count=p.n) for k in kmins]

            def level_skip(fi):
                return None if minrank is None else [(minrank[v], kmins[fi]) for v in range(V)]

            if nl == 1:
                items = [(fi, v) for fi in range(len(frames)) for v in range(V)]
                targets = [rv.images[v] for _ in range(len(frames)) for v in range(V)]
                sk = None if minrank is None else [x for fi in range(len(frames)) for x in level_skip(fi)]
                out = render_sse_chunked(frames, cams, items, targets, device=dev, host=False, tile_skip=sk)
            else:
                # one render call per level, alternating over the engine lanes: level
                # k+1's projection / binning / sort overlap level k's compositing
                main = torch.cuda.current_stream(dev)
                streams = [main] + [_lane_stream(dev, k) for k in range(1, nl)]
                for st in streams[1:]:
                    st.wait_stream(main)  # the reference images and level planes
                parts = []
                for fi, fr in enumerate(frames):
                    lane = fi % nl
                    with torch.cuda.stream(streams[lane]), engine_lane(lane):
                        sse = render_sse_chunked([fr], cams, [(0, v) for v in range(V)],
                                                 [rv.images[v] for v in range(V)], device=dev, host=False,
                                                 tile_skip=level_skip(fi))
                    if lane:
                        sse.record_stream(main)
                        for v in range(V):
                            rv.images[v].record_stream(streams[lane])
                            if minrank is not None:
                                minrank[v].record_stream(streams[lane])
                    parts.append(sse)
                for st in streams[1:]:
                    main.wait_stream(st)
                out = torch.cat(parts)
            level_removed(t)  # host-only work (after _removed_prepare), overlapping the enqueued renders
            return out

        from .grouping import probe_lanes

        _removed_prepare(p, t.delta.overlay())
        sse_dev = deferred_lanes(dev, run, min(probe_lanes(), max(len(todo), 1))) if todo else None
        if todo:
            sse = sse_dev.cpu().numpy()
            sizes_px = [c.resolution[0] * c.resolution[1] * 3 for c in cams]
            for fi, li in enumerate(todo):
                qualities[li] = float(np.mean([psnr_from_sse(sse[fi * V + v], sizes_px[v]) for v in range(V)]))
    levels = [PruningLevel(ratio=t.ratios[j], quality_db=q, size_bytes=t.sizes[j], pruned_indices=rm)
              for j, q, rm in zip(t.keep, qualities, level_removed(t))]
    return PruningLevelSpace(levels=tuple(levels), frame_index=frame_index)


def select_pruning_level(space: PruningLevelSpace, ctx: SelectionContext) -> int:
    """Algorithm 1: cliff scan, then binary search for the smallest-index
    candidate within budget, else the last (smallest) level
    (ss/pruning.py:140-178, PAPER Alg. 1)."""
    lv = space.levels
    if len(lv) == 1:
        return 0
    q = [x.quality_db for x in lv]
    prev_drop = q[0] - q[1]
    cand = [0]
    for i in range(1, len(lv)):
        drop = q[i - 1] - q[i]
        if drop / max(prev_drop, MIN_DROP) > ctx.cliff_beta:
            break
        cand.append(i)
        prev_drop = drop
    budget = ctx.budget_bytes
    lo, hi, best = 0, len(cand) - 1, None
    while lo <= hi:
        mid = (lo + hi) // 2
        if lv[cand[mid]].size_bytes <= budget:
            best, hi = cand[mid], mid - 1
        else:
            lo = mid + 1
    return len(lv) - 1 if best is None else best


def selection_margins(space: PruningLevelSpace, ctx: SelectionContext, entries: int = None) -> dict:
    """Decision margins of ``select_pruning_level`` and the prune counts
    (SURVEY.md s8(a) numerics contract): min |drop/prev - beta| over the
    cliff tests actually evaluated, min |size - budget| over the budget tests,
    and, when ``entries`` is given, min distance of ``ratio * E + 0.5`` to an
    integer over the levels (the floor in ss/pruning.py:83)."""
    lv = space.levels
    out = {"min_abs_cliff_ratio_minus_beta": float("inf"), "min_abs_size_minus_budget_bytes": float("inf")}
    if len(lv) > 1:
        q = [x.quality_db for x in lv]
        prev = q[0] - q[1]
        for i in range(1, len(lv)):
            drop = q[i - 1] - q[i]
            r = drop / max(prev, MIN_DROP)
            out["min_abs_cliff_ratio_minus_beta"] = min(out["min_abs_cliff_ratio_minus_beta"], abs(r - ctx.cliff_beta))
            if r > ctx.cliff_beta:
                break
            prev = drop
        out["min_abs_size_minus_budget_bytes"] = float(min(abs(x.size_bytes - ctx.budget_bytes) for x in lv))
    if entries is not None:
        fr = [x.ratio * entries + 0.5 for x in lv]
        out["min_k_floor_margin"] = float(min((abs(v - round(v)) for v in fr), default=float("inf")))
    return out


def ilp_optimal(level_spaces, budgets_bytes) -> list:
    """Exact optimum of the separable selection program: per frame, the
    highest-quality level within budget (first index wins ties)."""
    spaces, budgets = list(level_spaces), list(budgets_bytes)
    if len(spaces) != len(budgets):
        raise StructuralError("one budget per frame required")
    out = []
    for sp, b in zip(spaces, budgets):
        best = None
        for j, x in enumerate(sp.levels):
            if x.size_bytes <= b and (best is None or x.quality_db > sp.levels[best].quality_db):
                best = j
        out.append(FrameSelection(sp.frame_index, None, float("-inf"), False) if best is None
                   else FrameSelection(sp.frame_index, best, sp.levels[best].quality_db, True))
    return out


def levels_to_csv_rows(spaces) -> list:
    return [{"frame": sp.frame_index, "ratio": lv.ratio, "quality_db": lv.quality_db, "size_bytes": lv.size_bytes}
            for sp in spaces for lv in sp.levels]
