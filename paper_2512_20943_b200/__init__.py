"""paper_2512_20943_b200 -- B200-native AirGS per-frame evaluation path.

Drop-in for the reference package's evaluation entry points
(``splatstream.codec`` decode, ``rasterizer.render`` / ``render_with_usage``,
``metrics.psnr``, ``grouping.frame_quality`` / ``quality_probe``,
``pruning.build_level_space`` / ``select_pruning_level`` / ``ilp_optimal``,
``model.apply_delta`` / ``compose_deltas``), computed by hand-written sm_100a
CUDA kernels behind the C-ABI in ``include/airgs_b200.h``.  No CPU fallback.
"""

__version__ = "0.1.0"

from . import errors  # noqa: F401

__all__ = ["camera", "codec", "errors", "grouping", "metrics", "model", "pruning", "rasterizer", "streamsim",
           "synth", "sharding"]
