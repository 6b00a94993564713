"""Install the B200 path into an imported reference package.

    import splatstream
    from paper_2512_20943_b200 import dropin
    dropin.install(splatstream)

Replaces the compositing kernel seam (``splatstream.rasterizer._kernels``,
ss/rasterizer.py:39-49) and the module-level entry points of the evaluation
path -- including every ``from .x import f`` alias of them inside the
reference's modules -- with this package's device implementations.  The
reference callers (``streamsim.run_session``, ``grouping.build_groups``, the
CLI) then reach the GPU for every render, probe, decode, compose, apply and
level sweep.  Objects flow through duck typing (``.params``, ``.count``,
``.entries``, ``.pose`` ...), so reference dataclasses are accepted as
inputs; this package's exceptions become subclasses of the reference's.
The reference's own test modules run against it unchanged
(tests/test_gpu_dropin.py).
"""

from __future__ import annotations

import importlib
import sys
import types

from . import codec, grouping, metrics, model, pruning, rasterizer, streamsim

#   reference module        attribute                 replacement
PATCHES = (
    ("rasterizer", "render", rasterizer.render),
    ("rasterizer", "render_with_usage", rasterizer.render_with_usage),
    ("metrics", "psnr", metrics.psnr),
    ("codec", "decode_frame", codec.decode_frame),
    ("codec", "decode_delta", codec.decode_delta),
    ("codec", "encode_delta", codec.encode_delta),
    ("codec", "encode_frame", codec.encode_frame),
    ("model", "apply_delta", model.apply_delta),
    ("model", "compose_deltas", model.compose_deltas),
    ("pruning", "prune_delta", pruning.prune_delta),
    ("pruning", "prune_order", pruning.prune_order),
    ("pruning", "build_level_space", pruning.build_level_space),
    ("grouping", "frame_quality", grouping.frame_quality),
    ("grouping", "quality_probe", grouping.quality_probe),
)


class _KernelSeam(types.ModuleType):
    """Module-protocol object standing in for ``splatstream._composite``."""

    EPS_CONTRIB = rasterizer.EPS_CONTRIB
    ALPHA_CLAMP = rasterizer.ALPHA_CLAMP

    def __init__(self):
        super().__init__("splatstream_b200_kernels")

    @staticmethod
    def forward(means2d, conics, alphas, colors, bboxes, height, width, record=False):
        return rasterizer.forward(means2d, conics, alphas, colors, bboxes, height, width, record)

    @staticmethod
    def backward(*args, **kwargs):
        return rasterizer.backward(*args, **kwargs)


# the leaf classes (each also reaches the reference's SplatStreamError root
# through its reference twin; the roots themselves cannot be re-based)
ERROR_CLASSES = ("StructuralError", "ValidationError", "CapacityError", "DecodeError",
                 "ProtocolError", "TraceExhaustedError", "MissingArtifactError", "InfeasibleError", "TrainingError")


def _adopt_error_classes(pkg_name) -> int:
    """Make this package's exception classes subclasses of the reference's
    (``ss/errors.py``), so ``except splatstream.errors.StructuralError`` in
    reference callers (and ``pytest.raises`` in its tests) catches what the
    device path raises.  Returns how many classes were adopted."""
    from . import errors

    try:
        ref = importlib.import_module(f"{pkg_name}.errors")
    except ImportError:
        return 0
    done = 0
    for name in ERROR_CLASSES:
        ours, theirs = getattr(errors, name, None), getattr(ref, name, None)
        if ours is None or theirs is None or issubclass(ours, theirs):
            continue
        ours.__bases__ = ours.__bases__ + (theirs,)
        done += 1
    return done


def _rebind_aliases(pkg_name, original, fn) -> list:
    """Replace every module-level alias of ``original`` in the reference's
    loaded modules (``from .model import apply_delta`` in streamsim,
    grouping, pruning, train ...) with ``fn``."""
    hits = []
    for mname, mod in list(sys.modules.items()):
        if mod is None or not (mname == pkg_name or mname.startswith(pkg_name + ".")):
            continue
        for attr, val in list(vars(mod).items()):
            if val is original:
                setattr(mod, attr, fn)
                hits.append((mname[len(pkg_name) + 1:] or pkg_name, attr))
    return hits


def install(pkg, modules=None) -> list:
    """Patch ``pkg`` (the imported reference package); returns the list of
    (module, attribute) pairs replaced.  Every alias of a replaced function
    in the reference's modules (``from .model import apply_delta``) is
    rebound too, so reference callers such as ``SessionState.client_frame``,
    ``TrainedStream.reconstruct`` and ``transmit_delta`` reach the device
    path; the exception classes become subclasses of the reference's."""
    name = pkg.__name__
    # import every reference module first, so that their from-imports exist to rebind
    for sub in ("model", "codec", "rasterizer", "metrics", "pruning", "grouping", "streamsim", "train"):
        try:
            importlib.import_module(f"{name}.{sub}")
        except ImportError:
            pass
    _adopt_error_classes(name)
    done = []
    table = list(PATCHES) + [("streamsim", "step_frame", streamsim.step_frame),
                             ("streamsim", "client_reconstruct", streamsim.client_reconstruct),
                             ("streamsim", "transmit_delta", streamsim.transmit_delta)]
    for mod_name, attr, fn in table:
        if modules and mod_name not in modules:
            continue
        mod = sys.modules.get(f"{name}.{mod_name}") or importlib.import_module(f"{name}.{mod_name}")
        original = getattr(mod, attr, None)
        if original is None or original is fn:
            continue
        for hit in _rebind_aliases(name, original, fn):
            if hit not in done:
                done.append(hit)
    ras = sys.modules.get(f"{name}.rasterizer")
    if ras is not None and (not modules or "rasterizer" in modules):
        ras._kernels = _KernelSeam()
        ras.KERNEL_BACKEND = rasterizer.KERNEL_BACKEND
        done.append(("rasterizer", "_kernels"))
    return done
