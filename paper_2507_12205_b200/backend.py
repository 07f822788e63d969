"""The reference's kernel-backend protocol, implemented on the B200 (drop-in module).

`pkg/src/ecsr/_kernels.py:17-71` selects a backend module exposing NAME,
overlap_counts(...) and spmv_set(...). `register()` adds this module as
`ecsr._kernels._BACKENDS["b200"]` -- no reference edits -- after which
`ecsr._kernels.use_backend("b200")` routes every `executor.spmv_ec` set through
libecsr_b200.so. The name is not "gpu": the reference's own test
`tests/test_kernels.py:33-35` requires "gpu" to stay unknown.
"""

from __future__ import annotations

import numpy as np

from . import _lib

NAME = "b200"


def spmv_set(g, warp_size, vector_size, row_ids, block_indptr, base_indices,
             delta_indices, block_values, x, y):
    """Accumulate one block set into y in place (`_speedups.pyx:55-78` semantics).

    Precision follows y.dtype (f64, else f32); inputs are coerced with
    np.ascontiguousarray like the reference. Computed on the GPU by the generic
    kernel in the canonical order (lane-sequential, fixed lane tree, container-order
    y updates), so results are bitwise equal to the compiled reference backend.
    """
    if y.dtype == np.float64:
        dt, code = np.float64, _lib.F64
    else:
        dt, code = np.float32, _lib.F32
    if not (isinstance(y, np.ndarray) and y.dtype == dt and y.flags.c_contiguous):
        raise ValueError("y must be a contiguous float32/float64 array (updated in place)")
    rows = np.ascontiguousarray(row_ids, dtype=np.uint32)
    indptr = np.ascontiguousarray(block_indptr, dtype=np.int64)
    bases = np.ascontiguousarray(base_indices, dtype=np.uint32)
    deltas = np.ascontiguousarray(delta_indices, dtype=np.uint32)
    vals = np.ascontiguousarray(block_values, dtype=dt)
    xx = np.ascontiguousarray(x, dtype=dt)
    nb = max(len(indptr) - 1, 0)
    rc = _lib.lib().ecsr_b200_spmv_set(
        int(g), int(warp_size), int(vector_size), nb, _lib.ptr(rows), _lib.ptr(indptr),
        _lib.ptr(bases), _lib.ptr(deltas), _lib.ptr(vals), _lib.ptr(xx), xx.size,
        _lib.ptr(y), y.size, code)
    _lib.check(rc, "ecsr_b200_spmv_set")


def overlap_counts(row_ptr, col_idx, num_rows, num_cols):
    """Pairwise shared-column counts, diagonal zeroed (`_speedups.pyx:24-52`).

    Offline extraction only (not the SpMV hot path): exact integer counts from a
    0/1 pattern product, identical to both reference backends.
    """
    counts = np.zeros((num_rows, num_rows), dtype=np.int32)
    col_idx = np.asarray(col_idx)
    if num_rows == 0 or col_idx.size == 0:
        return counts
    rows = np.repeat(np.arange(num_rows), np.diff(np.asarray(row_ptr)))
    dense = np.zeros((num_rows, num_cols), dtype=np.float32)
    dense[rows, col_idx] = 1.0
    counts = (dense @ dense.T).astype(np.int32)
    np.fill_diagonal(counts, 0)
    return counts


def register() -> None:
    """Insert this module into the reference's backend registry."""
    import sys

    from ecsr import _kernels  # the reference package (tests / host integration)

    _kernels._BACKENDS[NAME] = sys.modules[__name__]
