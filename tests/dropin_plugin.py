"""pytest plugin: run the REFERENCE's own test modules with this package's
device path installed (``paper_2512_20943_b200.dropin.install``).

Loaded with ``-p dropin_plugin`` before the reference's test modules are
collected, so their ``from splatstream.x import f`` bindings already see the
replacements.  The reference package comes from the vendored copy
``baseline/_ref/pkg/src`` (git-ignored, shipped to the GPU box; built by
``make -C baseline``).  At the end it writes a JSON report
(``$AIRGS_DROPIN_REPORT``): what was patched, how many kernels the device
path launched during the run, and which airgs libraries the process mapped.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = os.path.join(ROOT, "baseline", "_ref", "pkg", "src")

_STATE = {}


def pytest_configure(config):
    for p in (ROOT, REF_SRC):
        if p not in sys.path:
            sys.path.insert(0, p)
    import splatstream

    from paper_2512_20943_b200 import _lib, dropin

    _STATE["patched"] = dropin.install(splatstream)
    _STATE["launches0"] = _lib.engine().launches


def pytest_unconfigure(config):
    path = os.environ.get("AIRGS_DROPIN_REPORT")
    if not path or "launches0" not in _STATE:
        return
    from paper_2512_20943_b200 import _lib

    maps = []
    try:
        with open("/proc/self/maps") as fh:
            maps = sorted({line.split()[-1] for line in fh if "airgs" in line or "_composite" in line})
    except OSError:
        pass
    with open(path, "w") as fh:
        json.dump({"patched": [list(p) for p in _STATE["patched"]],
                   "device_launches": _lib.engine().launches - _STATE["launches0"],
                   "mapped": maps}, fh)
