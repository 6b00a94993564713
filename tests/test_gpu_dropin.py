"""Drop-in acceptance on the B200: the reference's
OWN hot-path test modules -- unchanged, from the vendored reference package
(baseline/_ref, see baseline/Makefile) -- run with dropin.install applied, so
every render, render_with_usage, psnr, decode/encode, compose/apply, prune,
level sweep, probe and session step they exercise goes through
libairgs_b200.so.  The reference's pluggable-kernel parity checks
(_kernels_py vs its compiled _composite) and its trainer still run on the
host, as in the reference."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref", "pkg")

# the reference's hot-path suites: rasterizer, pruning, codec,
# metrics, model (delta algebra), grouping (probes), streamsim (sessions), and
# the acceptance tests of the evaluation path (tests/test_acceptance.py:91-467)
MODULES = ["test_rasterizer.py", "test_pruning.py", "test_codec.py", "test_metrics.py", "test_model.py",
           "test_grouping.py", "test_streamsim.py"]
ACCEPTANCE = ("test_level_selection_matches_linear_scan_and_optimum or test_per_frame_argmax_equals_joint_enumeration"
              " or test_client_quality_recovers_after_bandwidth_starvation"
              " or test_grouping_bounds_quality_through_appearance_event"
              " or test_delta_sparsity_tracks_movers_and_payload_scales_linearly"
              " or test_pruning_quality_curve_weakly_decreases_with_a_cliff"
              " or test_codec_round_trips_and_exact_sizes")


def _run(args, tmp_path, name):
    report = str(tmp_path / f"{name}.json")
    env = dict(os.environ, AIRGS_DROPIN_REPORT=report,
               PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, os.path.join(REF, "src")]))
    proc = subprocess.run([sys.executable, "-m", "pytest", "-p", "dropin_plugin", "-q", "-p", "no:cacheprovider",
                           "--rootdir", REF, *args], cwd=os.path.join(REF, "tests"), env=env,
                          capture_output=True, text=True, timeout=1800)
    tail = "\n".join((proc.stdout + proc.stderr).strip().splitlines()[-40:])
    assert proc.returncode == 0, tail
    with open(report) as fh:
        rep = json.load(fh)
    assert rep["device_launches"] > 0, rep
    assert any(p.endswith("libairgs_b200.so") for p in rep["mapped"]), rep
    return rep, tail


@pytest.fixture(scope="module")
def vendored():
    if not os.path.isdir(os.path.join(REF, "tests")):
        pytest.skip("vendored reference missing: run `make -C baseline` where /root/reference exists")


def test_reference_hot_path_suites_pass_on_the_device(vendored, tmp_path):
    rep, tail = _run(MODULES, tmp_path, "suites")
    patched = {tuple(p) for p in rep["patched"]}
    assert ("rasterizer", "render") in patched and ("pruning", "build_level_space") in patched
    assert ("streamsim", "apply_delta") in patched  # the from-imported alias, rebound
    assert " passed" in tail and " failed" not in tail


def test_reference_acceptance_tests_pass_on_the_device(vendored, tmp_path):
    _, tail = _run(["test_acceptance.py", "-k", ACCEPTANCE], tmp_path, "acceptance")
    assert " passed" in tail and " failed" not in tail
