"""ctypes binding of libecsr_b200.so (include/ecsr_b200.h).

This is the exact binding a maintainer would add to the reference:
plain pointers and sizes, no torch types. Loading fails loudly -- there is no CPU
fallback anywhere on the product path.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ContainerError, DeviceError, EcsrError

LIB_NAME = "libecsr_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

OK, ERR_CONTAINER, ERR_VALUE, ERR_CUDA = 0, 1, 2, 3
F16, F32, F64 = 1, 2, 3
PACK_DEFAULT, PACK_FORCE_GENERIC = 0, 1
SPMV_OVERWRITE, SPMV_ACCUMULATE, SPMV_ORDERED, SPMV_MEMSET_Y = 0, 1, 2, 4
IO_AFTER_PREDECESSOR = 1  # include/ecsr_b200.h ECSR_IO_AFTER_PREDECESSOR

_DTYPE_CODE = {np.dtype(np.float16): F16, np.dtype(np.float32): F32, np.dtype(np.float64): F64}

c_i32, c_i64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p


class HostSet(ctypes.Structure):
    _fields_ = [("granularity", c_i32), ("vector_size", c_i32), ("num_blocks", c_i64),
                ("stored_cols", c_i64), ("real_nnz", c_i64), ("row_indices", c_vp),
                ("block_indptr", c_vp), ("base_indices", c_vp), ("delta_indices", c_vp),
                ("pad_mask", c_vp), ("block_values", c_vp)]


class OutSet(ctypes.Structure):
    _fields_ = [("row_indices", c_vp), ("block_indptr", c_vp), ("base_indices", c_vp),
                ("delta_indices", c_vp), ("pad_mask", c_vp), ("block_values", c_vp)]


class SetInfo(ctypes.Structure):
    _fields_ = [("granularity", c_i32), ("vector_size", c_i32), ("num_blocks", c_i64),
                ("stored_cols", c_i64), ("real_nnz", c_i64)]


class BlobInfo(ctypes.Structure):
    _fields_ = [("num_rows", c_i64), ("num_cols", c_i64), ("nsets", c_i32), ("warp_size", c_i32),
                ("delta_bits", c_i32), ("value_bits", c_i32), ("value_bytes", c_i32),
                ("num_blocks", c_i64), ("stored_cols", c_i64), ("real_nnz", c_i64)]

    def to_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class Bytes(ctypes.Structure):
    _fields_ = [("row_indices", c_i64), ("block_indptr", c_i64), ("base_indices", c_i64),
                ("delta_indices", c_i64), ("pad_mask", c_i64), ("block_values", c_i64),
                ("desc", c_i64), ("model_kernel_bytes", c_i64),
                ("device_arena_bytes", c_i64), ("device_total_bytes", c_i64),
                ("layout", c_i32), ("grid", c_i32), ("stages", c_i32),
                ("stage_bytes", c_i32), ("tiles", c_i64), ("queue_tiles", c_i64)]

    def to_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# name -> (restype, argtypes); every symbol include/ecsr_b200.h declares.
SIGNATURES = {
    "ecsr_b200_pack": (c_i32, [ctypes.POINTER(HostSet), c_i32, c_i64, c_i64, c_i32, c_i32, c_i32,
                               c_i32, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "ecsr_b200_spmv": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_vp]),
    "ecsr_b200_parse": (c_i32, [c_vp, c_i64, ctypes.POINTER(BlobInfo)]),
    "ecsr_b200_load": (c_i32, [c_vp, c_i64, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "ecsr_b200_info": (c_i32, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                               ctypes.POINTER(c_i32), ctypes.POINTER(c_i32),
                               ctypes.POINTER(c_i32), ctypes.POINTER(c_i32),
                               ctypes.POINTER(c_i32)]),
    "ecsr_b200_set_info": (c_i32, [c_vp, c_i32, ctypes.POINTER(SetInfo)]),
    "ecsr_b200_unpack": (c_i32, [c_vp, ctypes.POINTER(OutSet), c_i32, c_i32]),
    "ecsr_b200_bytes": (c_i32, [c_vp, ctypes.POINTER(Bytes)]),
    "ecsr_b200_free": (None, [c_vp]),
    "ecsr_b200_blob_open": (c_i32, [c_vp, c_i64, ctypes.POINTER(c_vp)]),
    "ecsr_b200_blob_header": (c_i32, [c_vp, ctypes.POINTER(BlobInfo)]),
    "ecsr_b200_blob_set_info": (c_i32, [c_vp, c_i32, ctypes.POINTER(SetInfo)]),
    "ecsr_b200_blob_copy_set": (c_i32, [c_vp, c_i32, ctypes.POINTER(OutSet)]),
    "ecsr_b200_blob_free": (None, [c_vp]),
    "ecsr_b200_serialize": (c_i32, [ctypes.POINTER(HostSet), c_i32, c_i64, c_i64, c_i32, c_i32, c_i32, c_i32,
                                    c_vp, c_i64, ctypes.POINTER(c_i64)]),
    "ecsr_b200_group_create": (c_i32, [ctypes.POINTER(c_vp), c_i32, ctypes.POINTER(c_vp)]),
    "ecsr_b200_group_spmv": (c_i32, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i32, c_vp]),
    "ecsr_b200_group_info": (c_i32, [c_vp, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32),
                                     ctypes.POINTER(c_i32), c_i32]),
    "ecsr_b200_group_free": (None, [c_vp]),
    "ecsr_b200_xchg_create": (c_i32, [c_i64, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "ecsr_b200_xchg_handle": (c_i32, [c_vp, c_vp]),
    "ecsr_b200_xchg_open": (c_i32, [c_vp, c_vp]),
    "ecsr_b200_xchg_plan": (c_i32, [c_vp, c_vp, c_i32]),
    "ecsr_b200_xchg_run": (c_i32, [c_vp, c_vp, c_vp]),
    "ecsr_b200_xchg_y": (c_vp, [c_vp]),
    "ecsr_b200_xchg_free": (None, [c_vp]),
    "ecsr_b200_host_io": (c_i32, [c_vp, c_i32, c_i32, c_vp]),
    "ecsr_b200_trace": (c_i32, [c_vp, c_vp, c_i64, ctypes.POINTER(c_i64)]),
    "ecsr_b200_spmv_set": (c_i32, [c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_i64, c_vp, c_i64, c_i32]),
    "ecsr_b200_to_f16": (c_i32, [c_vp, c_i32, c_vp, c_i64]),
    "ecsr_b200_encode": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32,
                                 c_i64, c_i32, ctypes.POINTER(c_vp)]),
    "ecsr_b200_enc_nsets": (c_i32, [c_vp]),
    "ecsr_b200_enc_set_info": (c_i32, [c_vp, c_i32, ctypes.POINTER(SetInfo)]),
    "ecsr_b200_enc_copy_set": (c_i32, [c_vp, c_i32, ctypes.POINTER(OutSet), c_i32]),
    "ecsr_b200_enc_free": (None, [c_vp]),
    "ecsr_b200_enc_last_error": (ctypes.c_char_p, []),
    "ecsr_b200_last_error": (ctypes.c_char_p, []),
    "ecsr_b200_version": (ctypes.c_char_p, []),
    "ecsr_b200_device_count": (c_i32, []),
}

_lib = None


def lib():
    """Load the in-tree library once; raise (never fall back) when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the EC-CSR SpMV has no CPU fallback)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().ecsr_b200_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc == OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == ERR_CONTAINER:
        raise ContainerError(msg)
    if rc == ERR_VALUE:
        raise ValueError(msg)
    if rc == ERR_CUDA:
        raise DeviceError(msg)
    raise EcsrError(msg)


def ptr(a: np.ndarray) -> int | None:
    return a.ctypes.data if a.size else None


def dtype_code(dtype) -> int:
    try:
        return _DTYPE_CODE[np.dtype(dtype)]
    except KeyError:
        raise ValueError(f"unsupported dtype {dtype}") from None
