"""Shared test setup.

* registers the `gpu` marker (tests that need a B200; run with -m gpu);
* puts the reference package (baseline/_ref, this container only) on sys.path
  BEFORE our package is imported, so `ecsr.errors` classes are shared;
* loads the golden fixtures made from the reference by tests/golden/make_golden.py.
"""

import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = os.path.join(ROOT, "baseline", "_ref", "pkg", "src")
if os.path.isdir(REF_SRC) and REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: minutes of CPU; runs with ECSR_RUN_SLOW=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("ECSR_RUN_SLOW"):
        return
    skip = pytest.mark.skip(reason="slow (set ECSR_RUN_SLOW=1)")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


def have_reference() -> bool:
    try:
        import ecsr  # noqa: F401
        from ecsr import _speedups  # noqa: F401
    except ImportError:
        return False
    return True


needs_reference = pytest.mark.skipif(not have_reference(),
                                     reason="reference package not importable here")


def golden_names():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return [c["name"] for c in json.load(fh)]


def golden_manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return {c["name"]: c for c in json.load(fh)}


def load_golden(name):
    from paper_2507_12205_b200.container import deserialize

    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    out = {k: z[k] for k in z.files}
    out["blob"] = out["blob"].tobytes()
    out["ec"] = deserialize(out["blob"])
    out["report"] = dict(zip([str(k) for k in out["report_keys"]],
                             [int(v) for v in out["report_vals"]]))
    return out


def rel_err(y, y_ref):
    """Infinity-norm error relative to max |y_ref| (pkg/tests/conftest.py:9-16)."""
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    if y_ref.size == 0:
        return 0.0
    scale = max(float(np.max(np.abs(y_ref))), 1e-30)
    return float(np.max(np.abs(y - y_ref))) / scale


def rel_l2(y, y_ref):
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    d = float(np.linalg.norm(y_ref))
    return float(np.linalg.norm(y - y_ref)) / max(d, 1e-30)
