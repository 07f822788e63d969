"""Native EC-CSR encoder: `convert_csr` of the reference, in C++ (libecsr_b200.so).

`convert_csr(matrix, warp_size=32, vector_size=4, delta_bits=8, ...)` returns the same
container as `ecsr.storage.convert_csr(matrix, ExtractionConfig(warp_size, vector_size,
delta_bits, max_levels), clip_limit, dtype)` (`pkg/src/ecsr/storage.py:700-708`), array
for array and byte for byte after `serialize` -- tests/test_encoder.py checks that
against the reference's own encodings (golden fixtures) and, in the dev container,
against the live reference. It is the offline producer of the hot path's input and
makes the 70B / OPT-30B shapes encodable in seconds instead of hours.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .container import EcCsrMatrix, EcCsrSet
from .errors import ContainerError


def convert_csr(matrix, warp_size: int = 32, vector_size: int = 4, delta_bits: int = 8,
                max_levels: int | None = None, clip_limit: int | None = None, dtype=None,
                value_bits: int | None = None, threads: int = 0) -> EcCsrMatrix:
    """`storage.convert_csr` (`storage.py:700-708`) natively; `matrix` is any CSR with
    num_rows, num_cols, row_ptr, col_idx, values (`core.CsrMatrix` or ours)."""
    lib = _lib.lib()
    row_ptr = np.ascontiguousarray(matrix.row_ptr, dtype=np.int64)
    col_idx = np.ascontiguousarray(matrix.col_idx, dtype=np.int64)
    values = np.ascontiguousarray(matrix.values)
    if values.dtype not in (np.float32, np.float64):
        values = values.astype(np.float64)
    dtype = np.dtype(dtype if dtype is not None else values.dtype)
    if dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError("container values must be float32 or float64")
    if value_bits is None:
        value_bits = dtype.itemsize * 8
    out = ctypes.c_void_p()
    rc = lib.ecsr_b200_encode(int(matrix.num_rows), int(matrix.num_cols), _lib.ptr(row_ptr),
                              _lib.ptr(col_idx), _lib.ptr(values), _lib.dtype_code(values.dtype),
                              int(warp_size), int(vector_size), int(delta_bits),
                              -1 if max_levels is None else int(max_levels),
                              -1 if clip_limit is None else int(clip_limit), int(threads),
                              ctypes.byref(out))
    if rc != _lib.OK:
        msg = (lib.ecsr_b200_enc_last_error() or b"").decode()
        if rc == _lib.ERR_CONTAINER:
            raise ContainerError(msg)
        raise ValueError(msg)
    try:
        sets = []
        for i in range(lib.ecsr_b200_enc_nsets(out)):
            info = _lib.SetInfo()
            _lib.check(lib.ecsr_b200_enc_set_info(out, i, ctypes.byref(info)), "enc_set_info")
            g, nb, st = info.granularity, info.num_blocks, info.stored_cols
            s = EcCsrSet(g, info.vector_size, nb, st, info.real_nnz,
                         np.zeros(g * nb, np.uint32), np.zeros(nb + 1, np.int64),
                         np.zeros(warp_size * nb, np.uint32), np.zeros(st, np.uint32),
                         np.zeros(st, np.bool_), np.zeros(g * st, dtype))
            o = _lib.OutSet(_lib.ptr(s.row_indices), s.block_indptr.ctypes.data,
                            _lib.ptr(s.base_indices), _lib.ptr(s.delta_indices),
                            _lib.ptr(s.pad_mask.view(np.uint8)), _lib.ptr(s.block_values))
            _lib.check(lib.ecsr_b200_enc_copy_set(out, i, ctypes.byref(o), _lib.dtype_code(dtype)),
                       "enc_copy_set")
            sets.append(s)
    finally:
        lib.ecsr_b200_enc_free(out)
    return EcCsrMatrix(int(matrix.num_rows), int(matrix.num_cols), int(value_bits), int(delta_bits),
                       int(warp_size), sets)
