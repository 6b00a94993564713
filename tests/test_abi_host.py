"""CPU: the C-ABI library loads and exports every symbol include/airgs_b200.h
declares (no compute calls without a GPU), plus the host-side logic of the
drop-in that needs no device (selection, ILP, plans, cameras, varints,
header validation, error taxonomy)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "airgs_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"AIRGS_API\s+[\w\s\*]+?\b(airgs_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "airgs_render" in syms and "airgs_composite_forward" in syms and "airgs_gsdp_decode" in syms
    assert len(syms) >= 15


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2512_20943_b200 import _lib

    lib = _lib.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_bindings_cover_exactly_the_header():
    from paper_2512_20943_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_struct_layouts_match_header():
    import ctypes

    from paper_2512_20943_b200 import _lib

    assert ctypes.sizeof(_lib.CameraC) == 9 * 8 + 3 * 8 + 3 * 8 + 8 + 8 + 4 + 4
    assert ctypes.sizeof(_lib.FrameC) == 8 + 8 + 8 + 4 + 4
    assert ctypes.sizeof(_lib.ItemC) == 4 + 4 + 8 + 8 + 8 + 8 + 8 + 4 + 4
    assert _lib.ItemC.tile_minrank.offset == 40 and _lib.ItemC.tile_keep_min.offset == 48


def test_status_codes_map_to_reference_taxonomy():
    from paper_2512_20943_b200 import _lib, errors

    assert _lib._STATUS[-1] is errors.StructuralError
    assert _lib._STATUS[-2] is errors.ValidationError
    assert _lib._STATUS[-3] is errors.CapacityError
    assert _lib._STATUS[-5] is errors.DecodeError
    for cls, code in [(errors.StructuralError, "STRUCTURAL"), (errors.DecodeError, "DECODE"),
                      (errors.InfeasibleError, "INFEASIBLE"), (errors.TrainingError, "TRAINING")]:
        assert issubclass(cls, errors.SplatStreamError) and cls.code == code


def test_engine_refuses_without_gpu():
    import torch

    from paper_2512_20943_b200 import _lib

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        _lib.Engine(0)


def test_cameras_bit_identical_to_reference_rig():
    from paper_2512_20943_b200.camera import ring_rig

    g = load_golden("render.npz")
    for cid, (n, res) in enumerate([(3, (48, 40)), (2, (33, 29)), (3, (96, 72)), (2, (64, 64))]):
        cams = ring_rig(n, radius=3.0, height=0.3, focal=res[0] * 40.0 / 48.0, resolution=res)
        for c, pose in zip(cams, g[f"c{cid}_cam_pose"]):
            np.testing.assert_array_equal(c.pose, pose)


def test_camera_validation():
    from paper_2512_20943_b200.camera import Camera, look_at
    from paper_2512_20943_b200.errors import StructuralError

    with pytest.raises(StructuralError):
        Camera(pose=np.eye(3), focal=1.0, resolution=(16, 16))
    with pytest.raises(StructuralError):
        Camera(pose=np.eye(4), focal=1.0, resolution=(4, 16))
    with pytest.raises(StructuralError):
        look_at((0, 0, 0), (0, 0, 0))
    c = look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), focal=40.0, resolution=(32, 32))
    np.testing.assert_allclose(c.center, [0.0, 0.0, -2.5], atol=1e-15)
    assert Camera.from_dict(c.to_dict()) == c


def test_near_clip_must_be_finite():
    """A negative near plane is accepted as the reference accepts it (kept
    depths near_clip < z <= 0 order before positive ones, render.cu
    list_key32; tests/test_gpu_render.py::test_negative_near_clip_matches_oracle);
    a non-finite one is refused with the reference's ValidationError class."""
    from paper_2512_20943_b200.camera import camera_struct, look_at
    from paper_2512_20943_b200.errors import ValidationError

    camera_struct(look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), near_clip=0.0))
    camera_struct(look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), near_clip=-0.25))
    for bad in (float("nan"), float("inf"), float("-inf")):
        with pytest.raises(ValidationError):
            camera_struct(look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), near_clip=bad))


def _space(qualities, sizes, frame_index=0):
    from paper_2512_20943_b200.pruning import PruningLevel, PruningLevelSpace

    n = len(qualities)
    return PruningLevelSpace(levels=tuple(PruningLevel(i / n, float(q), int(s), ()) for i, (q, s) in
                                          enumerate(zip(qualities, sizes))), frame_index=frame_index)


def test_selection_hand_traced_example():
    from paper_2512_20943_b200.pruning import SelectionContext, select_pruning_level

    space = _space([60.0, 59.9, 59.7, 50.0, 45.0], [1200, 900, 700, 500, 300])
    assert select_pruning_level(space, SelectionContext(bandwidth_B=700 * 8, target_rate_R=1.0)) == 2
    assert select_pruning_level(space, SelectionContext(bandwidth_B=1200 * 8, target_rate_R=1.0)) == 0
    assert select_pruning_level(space, SelectionContext(bandwidth_B=300 * 8, target_rate_R=1.0)) == 4
    assert select_pruning_level(_space([100.0], [24]), SelectionContext(1.0, 1.0)) == 0


def test_selection_matches_oracle_on_random_spaces():
    """Algorithm 1 vs the oracle and vs the ILP on 1000 random spaces
    (reference tests/test_acceptance.py:91-114)."""
    from oracle import airgs_oracle as orc
    from paper_2512_20943_b200.pruning import SelectionContext, ilp_optimal, select_pruning_level

    rng = np.random.default_rng(3)
    for _ in range(1000):
        L = int(rng.integers(1, 9))
        q = sorted(rng.uniform(20, 100, L), reverse=True)
        q[0] = 100.0
        s = sorted(rng.choice(np.arange(24, 5000), L, replace=False), reverse=True)
        sp = _space(q, s)
        B = float(rng.uniform(24, 6000)) * 8
        beta = float(rng.uniform(0.5, 4.0))
        ctx = SelectionContext(bandwidth_B=B, target_rate_R=1.0, cliff_beta=beta)
        assert select_pruning_level(sp, ctx) == orc.select_level(q, s, B, 1.0, beta)
        got = ilp_optimal([sp], [B / 8])[0]
        want = orc.ilp([(q, s)], [B / 8])[0]
        assert got.level == want and got.feasible == (want is not None)


def test_selection_context_and_space_validation():
    from paper_2512_20943_b200.errors import StructuralError, ValidationError
    from paper_2512_20943_b200.pruning import PruningLevel, PruningLevelSpace, SelectionContext, ilp_optimal

    assert SelectionContext(bandwidth_B=8000.0, target_rate_R=2.0).budget_bytes == 500.0
    with pytest.raises(ValidationError):
        SelectionContext(bandwidth_B=0.0, target_rate_R=1.0)
    with pytest.raises(StructuralError):
        PruningLevelSpace(levels=(PruningLevel(0.5, 50.0, 100, ()),), frame_index=0)
    with pytest.raises(StructuralError):
        _space([50, 40], [100, 100])
    with pytest.raises(StructuralError):
        ilp_optimal([_space([60, 50], [10, 5])], [10, 10])
    out = ilp_optimal([_space([60, 55, 40], [300, 200, 100], t) for t in range(2)], [250, 90])
    assert (out[0].level, out[0].quality_db, out[0].feasible) == (1, 55.0, True)
    assert out[1].feasible is False and out[1].level is None


def test_group_plan():
    from paper_2512_20943_b200.errors import StructuralError, ValidationError
    from paper_2512_20943_b200.grouping import GroupPlan, GroupSpan, is_keyframe, plan_from_decisions

    with pytest.raises(StructuralError):
        GroupSpan(key=1, start=2, end=3)
    with pytest.raises(StructuralError):
        GroupPlan(tau_db=30, groups=(GroupSpan(0, 0, 2), GroupSpan(4, 4, 5)))
    plan = GroupPlan(tau_db=31.5, groups=(GroupSpan(0, 0, 4), GroupSpan(5, 5, 9)))
    assert GroupPlan.from_json(plan.to_json()) == plan
    assert plan.frame_count == 10 and plan.group_of(7).key == 5
    with pytest.raises(ValidationError):
        plan.group_of(10)
    assert plan_from_decisions([True, False, False, True, False]) == GroupPlan(
        30.0, (GroupSpan(0, 0, 2), GroupSpan(3, 3, 4)))
    assert is_keyframe(29.999, 30.0) and not is_keyframe(30.0, 30.0)


def test_varints_and_headers():
    from paper_2512_20943_b200 import codec
    from paper_2512_20943_b200.errors import DecodeError, StructuralError

    for v in (0, 1, 127, 128, 300, 2**35, 2**63 - 1):
        data = codec.encode_varint(v)
        assert codec.decode_varint(data) == (v, len(data))
    assert [len(codec.encode_varint(v)) for v in (0, 1, 127, 128)] == [1, 1, 1, 2]
    with pytest.raises(StructuralError):
        codec.encode_varint(-1)
    with pytest.raises(DecodeError):
        codec.decode_varint(codec.encode_varint(300)[:-1])
    with pytest.raises(DecodeError):
        codec.decode_varint(bytes([0xFF] * 11))
    g = load_golden("codec.npz")
    blob = g["gsai1_blob"].tobytes()
    ims = codec.AttributeImageSet.from_bytes(blob)
    assert ims.count == 37 and ims.num_attributes == 26 and ims.to_bytes() == blob
    with pytest.raises(DecodeError):
        codec.AttributeImageSet.from_bytes(b"XXXX" + blob[4:])
    with pytest.raises(DecodeError):
        codec.AttributeImageSet.from_bytes(blob[: len(blob) // 2])
    with pytest.raises(DecodeError):
        codec.parse_delta_header(b"GSDP" + bytes(10))


def test_synthetic_generator_is_seeded():
    from paper_2512_20943_b200 import synth

    cfg = synth.SceneConfig("t", 1000, 2, (64, 48), 20, 0.6, 0.02)
    a = synth.Sequence(cfg, seed=3, event_every=5)
    b = synth.Sequence(cfg, seed=3, event_every=5)
    np.testing.assert_array_equal(a.frame(7), b.frame(7))
    assert a.frame(4).shape[0] == 1000 and a.frame(7).shape[0] == 1010
    assert synth.CONFIGS["C2"].count == 300_000 and synth.CONFIGS["C2"].resolution == (1352, 1014)


def test_dropin_installs_into_the_reference_package():
    """The reference package itself (read in this container only) gets its
    seam and entry points replaced; no GPU call is made."""
    import importlib.util
    import glob
    import sys

    if not os.path.exists("/root/reference/pkg/src/splatstream"):
        pytest.skip("reference tree not present")
    hits = glob.glob(os.path.join(ROOT, "oracle", "_ref", "_composite*.so"))
    if hits and "splatstream._composite" not in sys.modules:
        spec = importlib.util.spec_from_file_location("splatstream._composite", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        sys.modules["splatstream._composite"] = mod
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import splatstream
        from splatstream import pruning as ref_pruning, rasterizer as ref_ras, streamsim as ref_sim  # noqa: F401

        from paper_2512_20943_b200 import dropin, pruning, rasterizer

        done = dropin.install(splatstream)
        assert ("rasterizer", "_kernels") in done and ("pruning", "build_level_space") in done
        assert ref_ras.render is rasterizer.render
        assert ref_pruning.build_level_space is pruning.build_level_space
        assert ref_ras._kernels.forward.__func__ if hasattr(ref_ras._kernels.forward, "__func__") else True
        assert ref_ras.KERNEL_BACKEND == rasterizer.KERNEL_BACKEND
        # from-imported aliases inside the reference's modules are rebound too
        from paper_2512_20943_b200 import errors, model, streamsim

        assert ref_sim.apply_delta is model.apply_delta and ref_sim.compose_deltas is model.compose_deltas
        assert ref_pruning.apply_delta is model.apply_delta
        assert sys.modules["splatstream.grouping"].apply_delta is model.apply_delta
        assert ref_sim.step_frame is streamsim.step_frame
        # the device path's exceptions are caught as the reference's classes
        assert issubclass(errors.StructuralError, sys.modules["splatstream.errors"].StructuralError)
        assert issubclass(errors.DecodeError, sys.modules["splatstream.errors"].SplatStreamError)
    finally:
        sys.path.remove("/root/reference/pkg/src")
        for k in [k for k in sys.modules if k == "splatstream" or k.startswith("splatstream.")]:
            del sys.modules[k]
