"""pytest plugin: run the REFERENCE package's own test suite with backend "b200" active.

    cd baseline/_ref/pkg && PYTHONPATH=<repo>:<repo>/tests/refsuite \\
        python -m pytest tests -p ecsr_b200_plugin

At configure time the plugin registers this repo's backend module in the reference's
registry (`ecsr._kernels._BACKENDS["b200"]`, pkg/src/ecsr/_kernels.py:17-43) and makes
it the active backend, so every `executor.spmv_ec` of the reference suite
(test_executor.py, test_acceptance.py C1/C7/C8, test_storage.py, ...) runs its block
sets on the GPU through libecsr_b200.so. Shadow check: every call is also run by the
reference's compiled kernel (`_speedups.spmv_set`) on a copy of y, and the two y must be
equal (np.array_equal, NaN == NaN) -- bitwise parity over the whole reference suite.
Tests that switch backends explicitly (test_kernels.py) restore "b200" afterwards.
Call counts go to $ECSR_B200_PLUGIN_STATS (JSON) at session end.
"""

import json
import os
import types

import numpy as np

STATS = {"calls": 0, "mismatches": 0, "first_mismatch": None}


def pytest_configure(config):
    from ecsr import _kernels, _speedups

    from paper_2507_12205_b200 import backend

    def spmv_set(g, warp_size, vector_size, row_ids, block_indptr, base_indices, delta_indices,
                 block_values, x, y):
        y_ref = y.copy()
        _speedups.spmv_set(g, warp_size, vector_size, row_ids, block_indptr, base_indices,
                           delta_indices, block_values, x, y_ref)
        backend.spmv_set(g, warp_size, vector_size, row_ids, block_indptr, base_indices,
                         delta_indices, block_values, x, y)
        STATS["calls"] += 1
        if not np.array_equal(y, y_ref, equal_nan=True):
            STATS["mismatches"] += 1
            if STATS["first_mismatch"] is None:
                STATS["first_mismatch"] = {"g": int(g), "warp": int(warp_size), "v": int(vector_size),
                                           "dtype": str(y.dtype)}
            raise AssertionError("b200 spmv_set differs from the reference's compiled kernel")

    shim = types.SimpleNamespace(NAME=backend.NAME, spmv_set=spmv_set,
                                 overlap_counts=backend.overlap_counts)
    _kernels._BACKENDS[backend.NAME] = shim
    _kernels.use_backend(backend.NAME)


def pytest_unconfigure(config):
    path = os.environ.get("ECSR_B200_PLUGIN_STATS")
    if path:
        with open(path, "w") as fh:
            json.dump(STATS, fh)
