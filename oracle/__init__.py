"""CPU oracle for the EC-CSR SpMV hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package. It is the checker, never the product: the package
`paper_2507_12205_b200` never imports it and has no CPU fallback.

* `spmv_ec_oracle(ec, x)` -- `executor.spmv_ec` (`pkg/src/ecsr/executor.py:80-96`)
  over the plain-C restatement `liboracle.so` of `_speedups._spmv_set_impl`
  (`pkg/src/ecsr/_speedups.pyx:81-129`).
* `load_reference_speedups()` -- the reference's own compiled kernel, built from
  /root/reference/pkg/src/ecsr/_speedups.pyx into oracle/_ref/ by `make ref`
  (kind "reference" for the CPU baseline).
* `spmv_oracle_f64(csr, x)` -- `core.spmv_oracle` (`pkg/src/ecsr/core.py:223-235`).

Pinning: tests/test_oracle.py checks liboracle bit-for-bit against the reference's
compiled backend and against the golden vectors in tests/golden/ (made from the
reference by tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> None:
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        _LIB = ctypes.CDLL(path)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        for name in ("oracle_spmv_set_f32", "oracle_spmv_set_f64"):
            fn = getattr(_LIB, name)
            fn.restype = i32
            fn.argtypes = [i32, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp]
    return _LIB


def _p(a):
    return a.ctypes.data if a.size else None


def spmv_set(g, warp_size, vector_size, row_ids, block_indptr, base_indices, delta_indices,
             block_values, x, y) -> None:
    """Same protocol as `_speedups.spmv_set` (`_speedups.pyx:55-78`), y updated in place."""
    dt = np.float64 if y.dtype == np.float64 else np.float32
    assert y.dtype == dt and y.flags.c_contiguous
    rows = np.ascontiguousarray(row_ids, dtype=np.uint32)
    indptr = np.ascontiguousarray(block_indptr, dtype=np.int64)
    bases = np.ascontiguousarray(base_indices, dtype=np.uint32)
    deltas = np.ascontiguousarray(delta_indices, dtype=np.uint32)
    vals = np.ascontiguousarray(block_values, dtype=dt)
    xx = np.ascontiguousarray(x, dtype=dt)
    fn = lib().oracle_spmv_set_f64 if dt == np.float64 else lib().oracle_spmv_set_f32
    rc = fn(int(g), int(warp_size), int(vector_size), max(len(indptr) - 1, 0), _p(rows),
            _p(indptr), _p(bases), _p(deltas), _p(vals), _p(xx), _p(y))
    if rc:
        raise MemoryError("oracle allocation failed")


def spmv_ec_oracle(ec, x, dtype=None, set_fn=None) -> np.ndarray:
    """`executor.spmv_ec(ec, x, validate=False)` on the C oracle (or `set_fn`)."""
    dtype = np.dtype(dtype or ec.dtype)
    x = np.ascontiguousarray(x, dtype=dtype)
    y = np.zeros(ec.num_rows, dtype=dtype)
    fn = set_fn or spmv_set
    for s in ec.sets:
        fn(s.granularity, ec.warp_size, s.vector_size, s.row_indices, s.block_indptr,
           s.base_indices, s.delta_indices, np.asarray(s.block_values, dtype=dtype), x, y)
    return y


def spmv_oracle_f64(csr, x) -> np.ndarray:
    """f64 y accumulated in row order (`core.py:223-235`)."""
    x = np.asarray(x)
    prod = csr.values.astype(np.float64) * x.astype(np.float64)[csr.col_idx]
    rows = np.repeat(np.arange(csr.num_rows), np.diff(csr.row_ptr))
    return np.bincount(rows, weights=prod, minlength=csr.num_rows)


def load_reference_speedups():
    """Import oracle/_ref/_speedups*.so (the reference's Cython kernel) or None."""
    hits = glob.glob(os.path.join(HERE, "_ref", "_speedups*.so"))
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_speedups", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
