"""Install the B200 path into an imported reference package.

    import splatstream
    from paper_2512_20943_b200 import dropin
    dropin.install(splatstream)

Replaces the compositing kernel seam (``splatstream.rasterizer._kernels``,
ss/rasterizer.py:39-49) and the module-level entry points of the evaluation
path with this package's device implementations.  The reference callers
(``streamsim.step_frame``, ``grouping.build_groups``, the CLI) then run on the
GPU unchanged.  Objects flow through duck typing (``.params``, ``.count``,
``.entries``, ``.pose`` ...), so reference dataclasses are accepted as inputs.
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


def install(pkg, modules=None) -> list:
    """Patch ``pkg`` (the imported reference package); returns the list of
    (module, attribute) pairs replaced.  Modules that imported a patched name
    with ``from . import x`` (e.g. ``pruning`` using ``codec.encode_delta``)
    see the replacement because they resolve it through the module object."""
    done = []
    name = pkg.__name__
    for mod_name, attr, fn in PATCHES:
        if modules and mod_name not in modules:
            continue
        mod = sys.modules.get(f"{name}.{mod_name}") or importlib.import_module(f"{name}.{mod_name}")
        if hasattr(mod, attr):
            setattr(mod, attr, fn)
            done.append((mod_name, attr))
    ras = sys.modules.get(f"{name}.rasterizer")
    if ras is not None and (not modules or "rasterizer" in modules):
        ras._kernels = _KernelSeam()
        ras.KERNEL_BACKEND = rasterizer.KERNEL_BACKEND
        done.append(("rasterizer", "_kernels"))
    sim = sys.modules.get(f"{name}.streamsim")
    if sim is not None and (not modules or "streamsim" in modules):
        sim.step_frame = streamsim.step_frame
        sim.client_reconstruct = streamsim.client_reconstruct
        done.append(("streamsim", "step_frame"))
    return done
