"""The drop-in boundary, end to end: the reference's own registry and test suite.

* `backend.register(); _kernels.use_backend("b200")` then the reference's
  `executor.spmv_ec` (pkg/src/ecsr/executor.py:80-96) over every golden case: bitwise
  equal to the reference's compiled backend in f64 and f32 (y64, y32);
* the reference package's whole test suite (baseline/_ref/pkg/tests: executor, the
  200-matrix acceptance corpus C1-C8, storage, kernels, ...) run with "b200" active
  through tests/refsuite/ecsr_b200_plugin.py, every spmv_set call shadow-checked
  against the compiled kernel (bitwise).

Needs the reference package (baseline/_ref, built in place; it travels to the GPU box
with the repo snapshot) and a GPU.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import golden_names, have_reference, load_golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_reference(), reason="reference package (baseline/_ref) not built")]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "pkg")


@pytest.fixture
def b200_backend():
    from ecsr import _kernels

    from paper_2507_12205_b200 import backend

    backend.register()
    before = _kernels.active_backend()
    _kernels.use_backend("b200")
    assert _kernels.active_backend() == "b200"
    yield
    _kernels.use_backend(before)


@pytest.mark.parametrize("name", golden_names())
def test_reference_executor_through_b200_backend(name, b200_backend):
    from ecsr import executor, storage

    g = load_golden(name)
    ec = storage.deserialize(g["blob"])  # the reference's own container type
    y64 = executor.spmv_ec(ec, g["x"])
    assert y64.dtype == np.float64 and np.array_equal(y64, g["y64"])
    y32 = executor.spmv_ec(ec.astype(np.float32), g["x"].astype(np.float32))
    assert y32.dtype == np.float32 and np.array_equal(y32, g["y32"])


def test_reference_suite_with_b200_backend(tmp_path):
    stats = tmp_path / "stats.json"
    env = dict(os.environ, ECSR_B200_PLUGIN_STATS=str(stats),
               PYTHONPATH=os.pathsep.join([os.path.join(REF_PKG, "src"), ROOT,
                                           os.path.join(ROOT, "tests", "refsuite")]))
    out = subprocess.run([sys.executable, "-m", "pytest", "tests", "-q", "-x", "-p", "ecsr_b200_plugin",
                          "-p", "no:cacheprovider"],
                         cwd=REF_PKG, env=env, capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    s = json.loads(stats.read_text())
    assert s["mismatches"] == 0 and s["calls"] > 1000, s
    print(out.stdout.strip().splitlines()[-1], s)
