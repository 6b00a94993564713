"""On-disk formats: the GSSC scene container and the
trained-stream .npz, read and written byte-compatibly with the reference
(tests/golden/io_* written by the reference's own save_scene / save_stream)."""

import os

import numpy as np
import pytest

from conftest import load_golden

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_load_reference_scene_host():
    from paper_2512_20943_b200.model import load_scene

    v = load_golden("io_values.npz")
    frames = load_scene(os.path.join(HERE, "io_scene.gssc"))
    assert [f.frame_index for f in frames] == [0, 1]
    np.testing.assert_array_equal(frames[0].params, v["f0"])
    np.testing.assert_array_equal(frames[1].params, v["f1"])


def test_save_scene_is_byte_identical(tmp_path):
    from paper_2512_20943_b200.model import load_scene, save_scene

    frames = load_scene(os.path.join(HERE, "io_scene.gssc"))
    out = tmp_path / "s.gssc"
    save_scene(out, frames)
    assert out.read_bytes() == open(os.path.join(HERE, "io_scene.gssc"), "rb").read()


def test_scene_errors(tmp_path):
    from paper_2512_20943_b200.errors import ValidationError
    from paper_2512_20943_b200.model import load_scene

    data = open(os.path.join(HERE, "io_scene.gssc"), "rb").read()
    for bad, name in ((b"XXXX" + data[4:], "magic"), (data[:-3], "trunc"), (data[:4] + b"\x02" + data[5:], "ver")):
        p = tmp_path / f"{name}.gssc"
        p.write_bytes(bad)
        with pytest.raises(ValidationError):
            load_scene(p)


def test_save_stream_matches_reference_arrays(tmp_path):
    from paper_2512_20943_b200 import grouping
    from paper_2512_20943_b200.model import CanonicalSpace, DeltaTensor, GaussianFrame

    v = load_golden("io_values.npz")

    def host_delta(dense):
        return DeltaTensor(30, 17, {int(i): dense[i].copy() for i in np.nonzero(np.any(dense != 0, axis=1))[0]})

    space = CanonicalSpace(GaussianFrame(params=v["base"], frame_index=0, group_key=0), capacity_U=32)
    recs = [grouping.FrameRecord(t, 0, t == 0, host_delta(v[f"step{t}"]), host_delta(v[f"cum{t}"]), 40.0 - t)
            for t in range(3)]
    plan = grouping.GroupPlan(30.0, (grouping.GroupSpan(0, 0, 2),))
    out = tmp_path / "s.npz"
    grouping.save_stream(out, grouping.TrainedStream(plan=plan, spaces={0: space}, records=recs))
    with np.load(out) as a, np.load(os.path.join(HERE, "io_stream.npz")) as b:
        assert sorted(a.files) == sorted(b.files)
        for k in b.files:
            np.testing.assert_array_equal(a[k], b[k])


@pytest.mark.gpu
def test_load_scene_to_device_and_stream():
    from paper_2512_20943_b200 import grouping
    from paper_2512_20943_b200.model import load_scene

    v = load_golden("io_values.npz")
    frames = load_scene(os.path.join(HERE, "io_scene.gssc"), to_device=True)
    assert all(f.on_device for f in frames)
    np.testing.assert_array_equal(frames[0].params, v["f0"])  # downloaded from the device planes
    np.testing.assert_array_equal(frames[1].params, v["f1"])
    st = grouping.load_stream(os.path.join(HERE, "io_stream.npz"))
    np.testing.assert_array_equal(st.spaces[0].frame.params, v["base"])
    for t in range(3):
        np.testing.assert_array_equal(st.records[t].cumulative_delta.dense(), v[f"cum{t}"])
        np.testing.assert_array_equal(st.records[t].step_delta.dense(), v[f"step{t}"])
    assert st.plan.tau_db == 30.0 and [r.is_keyframe for r in st.records] == [True, False, False]
