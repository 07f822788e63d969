"""The EC-CSR container on the host: types, wire format, byte model, validation.

Mirrors `pkg/src/ecsr/storage.py` for the parts the hot path consumes, so the
GPU box needs no reference install:

* `EcCsrSet` / `EcCsrMatrix` -- same fields, dtypes and meaning as
  `storage.py:50-96` (duck-type compatible: the packer accepts either class).
* `serialize` / `deserialize` -- the `.ecsr` format of `storage.py:16-31`,
  `389-483`, byte-identical (tests check `serialize` equality both ways); the bytes are
  written and parsed by the native library (`ecsr_b200_serialize`, `ecsr_b200_blob_*`).
* `storage_report` components and `kernel_model_bytes` -- the byte model of
  `storage.py:579-649`; the roofline numerator of SURVEY.md §8(d) is
  `kernel_model_bytes` (components minus pad_mask and desc, plus x and y).
* `validate_container` -- the checks of `executor.py:50-77` and
  `storage.py:312-329`, vectorised so it runs once at pack time in
  milliseconds instead of per call.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import ContainerError

MAGIC = b"ECSR"
VERSION = 1
_HEADER_FMT = "<BBBBHQQL"
_DESC_FMT = "<LLQQQ"
HEADER_BYTES = 4 + struct.calcsize(_HEADER_FMT)
DESC_BYTES = struct.calcsize(_DESC_FMT)


@dataclass
class EcCsrSet:
    """One block set (`storage.py:50-62`)."""

    granularity: int
    vector_size: int
    num_blocks: int
    stored_cols: int
    real_nnz: int
    row_indices: np.ndarray   # u32[g * num_blocks]
    block_indptr: np.ndarray  # i64[num_blocks + 1], stored columns incl. padding
    base_indices: np.ndarray  # u32[warp * num_blocks]
    delta_indices: np.ndarray  # u32[stored_cols], chunk-permuted
    pad_mask: np.ndarray      # bool[stored_cols], chunk-permuted
    block_values: np.ndarray  # f32/f64[g * stored_cols], chunk-permuted


@dataclass
class EcCsrMatrix:
    """The container (`storage.py:65-96`)."""

    num_rows: int
    num_cols: int
    value_bits: int
    delta_bits: int
    warp_size: int
    sets: list

    @property
    def dtype(self):
        for s in self.sets:
            return s.block_values.dtype
        return np.dtype(np.float64)

    @property
    def nnz(self) -> int:
        return sum(s.real_nnz for s in self.sets)

    def astype(self, dtype) -> "EcCsrMatrix":
        """Cast values only; index arrays are shared (`storage.py:84-96`)."""
        sets = [
            EcCsrSet(s.granularity, s.vector_size, s.num_blocks, s.stored_cols,
                     s.real_nnz, s.row_indices, s.block_indptr, s.base_indices,
                     s.delta_indices, s.pad_mask, s.block_values.astype(dtype))
            for s in self.sets
        ]
        return EcCsrMatrix(self.num_rows, self.num_cols, self.value_bits,
                           self.delta_bits, self.warp_size, sets)


# --- wire format (storage.py:389-483): native, libecsr_b200.so -----------------------


def _delta_bytes(count: int, bits: int) -> int:
    """Packed size of `count` deltas of `bits` bits (4-bit deltas share bytes)."""
    return (count * bits + 7) // 8


def host_sets(ec, check_shapes: bool = True):
    """Coerce a container's sets to the C-ABI dtypes (copies only on mismatch, like
    np.ascontiguousarray in `_speedups.pyx:62-77`). Returns (HostSet array, keepalive,
    value dtype). Array lengths are checked against the declared sizes first
    (`storage.py:312-329`): the native side trusts num_blocks / stored_cols."""
    from . import _lib

    dtype = np.dtype(ec.dtype)
    if dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError("container values must be float32 or float64")
    keep = []
    arr = (_lib.HostSet * max(len(ec.sets), 1))()
    for s in ec.sets if check_shapes else ():
        check_set_shapes(s, int(ec.warp_size))
    for i, s in enumerate(ec.sets):
        rows = np.ascontiguousarray(s.row_indices, dtype=np.uint32)
        indptr = np.ascontiguousarray(s.block_indptr, dtype=np.int64)
        bases = np.ascontiguousarray(s.base_indices, dtype=np.uint32)
        deltas = np.ascontiguousarray(s.delta_indices, dtype=np.uint32)
        mask = np.ascontiguousarray(s.pad_mask, dtype=np.bool_).view(np.uint8)
        vals = np.ascontiguousarray(s.block_values, dtype=dtype)
        keep += [rows, indptr, bases, deltas, mask, vals]
        arr[i] = _lib.HostSet(int(s.granularity), int(s.vector_size), int(s.num_blocks),
                              int(s.stored_cols), int(s.real_nnz), _lib.ptr(rows),
                              _lib.ptr(indptr), _lib.ptr(bases), _lib.ptr(deltas),
                              _lib.ptr(mask), _lib.ptr(vals))
    return arr, keep, dtype


def serialize(ec) -> bytes:
    """Byte-identical to `ecsr.storage.serialize` (`storage.py:389-428`), written by
    `ecsr_b200_serialize`."""
    import ctypes

    from . import _lib

    arr, keep, dtype = host_sets(ec)
    args = (arr, len(ec.sets), int(ec.num_rows), int(ec.num_cols), int(ec.warp_size), int(ec.delta_bits),
            int(ec.value_bits), _lib.dtype_code(dtype))
    n = ctypes.c_int64(0)
    _lib.check(_lib.lib().ecsr_b200_serialize(*args, None, 0, ctypes.byref(n)), "ecsr_b200_serialize")
    buf = ctypes.create_string_buffer(max(n.value, 1))
    _lib.check(_lib.lib().ecsr_b200_serialize(*args, buf, n.value, ctypes.byref(n)), "ecsr_b200_serialize")
    del keep
    return buf.raw[:n.value]


def deserialize(data: bytes) -> EcCsrMatrix:
    """Parse and reject corruption exactly as `storage.py:431-483` does (the native
    parser `ecsr_b200_blob_open`: same checks, same ContainerError messages)."""
    import ctypes

    from . import _lib

    lib = _lib.lib()
    data = bytes(data)
    buf = ctypes.create_string_buffer(data, len(data))
    h = ctypes.c_void_p()
    rc = lib.ecsr_b200_blob_open(buf, len(data), ctypes.byref(h))
    if rc == _lib.ERR_CONTAINER:  # the reference's message, unprefixed (storage.py:431-483)
        raise ContainerError(_lib.last_error())
    _lib.check(rc, "deserialize")
    try:
        info = _lib.BlobInfo()
        _lib.check(lib.ecsr_b200_blob_header(h, ctypes.byref(info)), "deserialize")
        dtype = np.dtype(np.float32 if info.value_bytes == 4 else np.float64)
        warp = int(info.warp_size)
        sets = []
        for i in range(info.nsets):
            si = _lib.SetInfo()
            _lib.check(lib.ecsr_b200_blob_set_info(h, i, ctypes.byref(si)), "deserialize")
            g, nb, st = int(si.granularity), int(si.num_blocks), int(si.stored_cols)
            arrs = [np.empty(nb * g, np.uint32), np.empty(max(nb + 1, 1), np.int64),
                    np.empty(nb * warp, np.uint32), np.empty(st, np.uint32), np.empty(st, np.uint8),
                    np.empty(st * g, dtype)]
            out = _lib.OutSet(*[a.ctypes.data for a in arrs])
            _lib.check(lib.ecsr_b200_blob_copy_set(h, i, ctypes.byref(out)), "deserialize")
            rows, indptr, bases, deltas, mask, vals = arrs
            sets.append(EcCsrSet(g, int(si.vector_size), nb, st, int(si.real_nnz), rows, indptr, bases,
                                 deltas, mask.astype(bool), vals))
    finally:
        lib.ecsr_b200_blob_free(h)
    return EcCsrMatrix(int(info.num_rows), int(info.num_cols), int(info.value_bits), int(info.delta_bits),
                       warp, sets)


def save_container(ec, path) -> None:
    with open(path, "wb") as fh:
        fh.write(serialize(ec))


def load_container(path) -> EcCsrMatrix:
    with open(path, "rb") as fh:
        return deserialize(fh.read())


# --- validation (executor.py:50-77, storage.py:312-329) ----------------------


def check_set_shapes(s, warp: int) -> None:
    """Array shapes against the set's declared sizes (`storage.py:312-329`): the same
    checks in the same order, so the same ContainerError message comes first."""
    nb, stored, g = int(s.num_blocks), int(s.stored_cols), int(s.granularity)
    indptr = np.asarray(s.block_indptr)
    rules = (
        (lambda: len(indptr) == nb + 1, "block_indptr length mismatch"),
        (lambda: indptr[0] == 0 and not np.any(np.diff(indptr) < 0),
         "block_indptr must start at 0 and be non-decreasing"),
        (lambda: int(indptr[-1]) == stored, "block_indptr does not cover stored columns"),
        (lambda: len(s.delta_indices) == stored and len(s.pad_mask) == stored,
         "delta or mask array length mismatch"),
        (lambda: len(s.block_values) == stored * g, "block_values length mismatch"),
        (lambda: len(s.row_indices) == nb * g, "row_indices length mismatch"),
        (lambda: len(s.base_indices) == nb * warp, "base_indices length mismatch"),
        (lambda: not np.any(np.diff(indptr) % (warp * int(s.vector_size))),
         "block widths must be multiples of warp_size * vector_size"),
    )
    for ok, message in rules:
        if not ok():
            raise ContainerError(message)


def lane_tops(s, warp: int) -> np.ndarray:
    """Per (block, lane) last decoded column: base + sum of the lane's deltas.

    Vectorised form of the per-block loop in `executor.py:62-76`. Chunk-permuted
    position p of block b belongs to lane ((p - start_b) // v) % warp.
    """
    nb = s.num_blocks
    if nb == 0:
        return np.zeros((0, warp), dtype=np.int64)
    starts = np.asarray(s.block_indptr[:-1], dtype=np.int64)
    widths = np.diff(np.asarray(s.block_indptr, dtype=np.int64))
    block_of = np.repeat(np.arange(nb, dtype=np.int64), widths)
    local = np.arange(s.stored_cols, dtype=np.int64) - starts[block_of]
    lane = (local // s.vector_size) % warp
    adv = np.zeros(nb * warp, dtype=np.int64)
    np.add.at(adv, block_of * warp + lane, np.asarray(s.delta_indices, dtype=np.int64))
    return np.asarray(s.base_indices, dtype=np.int64).reshape(nb, warp) + adv.reshape(nb, warp)


def validate_container(ec) -> None:
    """Structural and range checks; raises ContainerError on any violation."""
    limit = 1 << ec.delta_bits
    for s in ec.sets:
        check_set_shapes(s, ec.warp_size)
        if s.delta_indices.size and int(np.max(s.delta_indices)) >= limit:
            raise ContainerError(
                f"delta {int(np.max(s.delta_indices))} exceeds {ec.delta_bits}-bit range")
        if s.base_indices.size and int(np.max(s.base_indices)) >= max(ec.num_cols, 1):
            raise ContainerError("base index out of range")
        if s.row_indices.size and int(np.max(s.row_indices)) >= max(ec.num_rows, 1):
            raise ContainerError("row index out of range")
        widths = np.diff(np.asarray(s.block_indptr, dtype=np.int64))
        tops = lane_tops(s, ec.warp_size)
        live = widths > 0
        if live.any():
            top = int(tops[live].max())
            if top >= ec.num_cols:
                raise ContainerError(f"decoded column {top} out of range {ec.num_cols}")


# --- byte model (storage.py:579-649) -----------------------------------------


def storage_components(ec, value_bits: int = 16) -> dict:
    """`storage_report(ec, value_bits).components` (`storage.py:592-613`)."""
    comp = {"desc": HEADER_BYTES + DESC_BYTES * len(ec.sets), "row_indices": 0,
            "block_indptr": 0, "base_indices": 0, "delta_indices": 0, "pad_mask": 0,
            "block_values": 0}
    for s in ec.sets:
        comp["row_indices"] += 4 * s.num_blocks * s.granularity
        comp["block_indptr"] += 8 * (s.num_blocks + 1)
        comp["base_indices"] += 4 * s.num_blocks * ec.warp_size
        comp["delta_indices"] += _delta_bytes(s.stored_cols, ec.delta_bits)
        comp["pad_mask"] += (s.stored_cols + 7) // 8
        comp["block_values"] += s.stored_cols * s.granularity * value_bits // 8
    return comp


def kernel_model_bytes(ec, value_bits: int = 16, x_bytes: int = 2, y_bytes: int = 4) -> int:
    """Algorithmic bytes of one SpMV.

    storage_report components minus pad_mask and desc (the kernel needs
    neither) + K x-elements + M y-elements.
    """
    comp = storage_components(ec, value_bits)
    arrays = sum(v for k, v in comp.items() if k not in ("pad_mask", "desc"))
    return arrays + x_bytes * ec.num_cols + y_bytes * ec.num_rows


def csr32_bytes(ec, value_bits: int = 16) -> int:
    """CSR-32 baseline of `storage.py:633`."""
    nnz = ec.nnz
    return nnz * value_bits // 8 + nnz * 4 + 4 * (ec.num_rows + 1)


def from_reference(ec) -> EcCsrMatrix:
    """Copy a reference `ecsr.storage.EcCsrMatrix` (or any duck-typed one)."""
    sets = [EcCsrSet(s.granularity, s.vector_size, s.num_blocks, s.stored_cols, s.real_nnz,
                     np.asarray(s.row_indices), np.asarray(s.block_indptr),
                     np.asarray(s.base_indices), np.asarray(s.delta_indices),
                     np.asarray(s.pad_mask), np.asarray(s.block_values)) for s in ec.sets]
    return EcCsrMatrix(ec.num_rows, ec.num_cols, ec.value_bits, ec.delta_bits,
                       ec.warp_size, sets)


# --- decode (storage.py:260-309) ---------------------------------------------


def decode_ec_csr(ec):
    """Scatter every stored entry back into CSR, dropping padding and gap-bridging
    columns (`pad_mask`), exactly like `storage.decode_ec_csr` (`storage.py:260-309`):
    the round trip `decode_ec_csr(convert_csr(A)) == A` holds bit for bit."""
    from .generators import CsrMatrix

    warp = ec.warp_size
    rows_l, cols_l, vals_l = [], [], []
    for s in ec.sets:
        check_set_shapes(s, warp)
        g, v = s.granularity, s.vector_size
        for b in range(s.num_blocks):
            st, en = int(s.block_indptr[b]), int(s.block_indptr[b + 1])
            n = en - st
            if n == 0:
                continue
            ch = n // (warp * v)
            d = np.asarray(s.delta_indices[st:en]).reshape(ch, warp, v).transpose(1, 0, 2)
            d = d.reshape(warp, -1).astype(np.int64)
            cols = (np.asarray(s.base_indices[b * warp:(b + 1) * warp], np.int64)[:, None]
                    + np.cumsum(d, axis=1)).reshape(-1)
            if cols.size and int(cols.max()) >= ec.num_cols:
                raise ContainerError(f"decoded column {int(cols.max())} out of range {ec.num_cols}")
            vals = np.asarray(s.block_values[st * g:en * g]).reshape(ch, warp, v * g)
            vals = vals.transpose(1, 0, 2).reshape(n, g)
            mask = np.asarray(s.pad_mask[st:en]).reshape(ch, warp, v).transpose(1, 0, 2).reshape(-1)
            keep = ~mask
            block_rows = np.asarray(s.row_indices[b * g:(b + 1) * g], np.int64)
            kc = cols[keep]
            rows_l.append(np.repeat(block_rows[None, :], kc.size, axis=0).reshape(-1))
            cols_l.append(np.repeat(kc, g))
            vals_l.append(vals[keep].reshape(-1))
    if rows_l:
        rows, cols, vals = np.concatenate(rows_l), np.concatenate(cols_l), np.concatenate(vals_l)
    else:
        rows = cols = np.empty(0, np.int64)
        vals = np.empty(0, ec.dtype)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size > 1 and np.any((np.diff(rows) == 0) & (np.diff(cols) == 0)):
        raise ContainerError("duplicate entries while decoding; container is inconsistent")
    if rows.size and (int(rows.max()) >= ec.num_rows or int(rows.min()) < 0):
        raise ContainerError("row index out of range while decoding")
    row_ptr = np.zeros(ec.num_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=ec.num_rows), out=row_ptr[1:])
    return CsrMatrix(ec.num_rows, ec.num_cols, row_ptr, cols, vals)
