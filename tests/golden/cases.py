"""Inputs of the golden fixtures, reconstructible without the reference installed.

`golden_matrix(case)` rebuilds the CSR a golden case was encoded from (the manifest
entry written by make_golden.py): the reference's generate_uniform (restated
draw-for-draw in paper_2507_12205_b200.generators), our magnitude / planted
generators, and the three hand-written KATs (pkg/tests/test_storage.py:30-42, 112-132,
162-166 and pkg/tests/test_executor.py:28-31).
"""

import numpy as np

from paper_2507_12205_b200.generators import CsrMatrix, generate_uniform, make_matrix


def corpus_params(i):
    """The reference acceptance corpus mix (pkg/tests/test_acceptance.py:51-67)."""
    rng = np.random.default_rng(1000 + i)
    sparsity = (0.5, 0.7, 0.8, 0.9)[i % 4]
    bits = (8, 4)[i % 2]
    if i % 10 == 9:
        lo, hi, wv = 192, 512, (32, 4)
    elif i % 10 in (7, 8):
        lo, hi, wv = 64, 192, (8, 2)
    else:
        lo, hi = 8, 64
        wv = [(2, 2), (4, 1), (2, 1), (4, 2)][i % 4]
    m = int(rng.integers(lo, hi + 1))
    k = int(rng.integers(lo, hi + 1))
    return m, k, sparsity, bits, wv


def _coo(m, k, rows, cols, vals):
    rows, cols, vals = np.asarray(rows), np.asarray(cols), np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=m), out=row_ptr[1:])
    return CsrMatrix(m, k, row_ptr, cols.astype(np.int64), vals)


def golden_matrix(case):
    name, kind = case["name"], case["kind"]
    if name == "kat_two_row_block":
        return _coo(2, 7, [0] * 4 + [1] * 4, [2, 4, 5, 6] * 2, [1.0] * 8)
    if name == "kat_identity6":
        return _coo(6, 6, range(6), range(6), [1.0] * 6)
    if name == "kat_explicit_zero":
        return _coo(2, 4, [0, 0, 1], [0, 2, 1], [0.0, 3.0, 4.0])
    if kind == "corpus":
        i = case["index"]
        m, k, s, _, _ = corpus_params(i)
        return generate_uniform(m, k, s, seed=i)
    return make_matrix(kind, case["m"], case["k"], case["s"], case["seed"], dtype=np.float64)
