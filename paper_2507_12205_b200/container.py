"""The EC-CSR container on the host: types, wire format, byte model, validation.

Mirrors `pkg/src/ecsr/storage.py` for the parts the hot path consumes, so the
GPU box needs no reference install:

* `EcCsrSet` / `EcCsrMatrix` -- same fields, dtypes and meaning as
  `storage.py:50-96` (duck-type compatible: the packer accepts either class).
* `serialize` / `deserialize` -- the `.ecsr` format of `storage.py:16-31`,
  `389-483`, byte-identical (tests check `serialize` equality both ways).
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


# --- wire format (storage.py:335-483) ---------------------------------------


def _delta_bytes(count: int, bits: int) -> int:
    if bits == 4:
        return (count + 1) // 2
    return count * (bits // 8)


def _pack_deltas(deltas: np.ndarray, bits: int) -> bytes:
    if deltas.size and int(deltas.max()) >= (1 << bits):
        raise ContainerError(f"delta exceeds {bits}-bit range")
    if bits == 4:
        d = deltas.astype(np.uint8)
        if d.size % 2:
            d = np.concatenate((d, np.zeros(1, dtype=np.uint8)))
        return (d[0::2] | (d[1::2] << 4)).tobytes()
    if bits == 8:
        return deltas.astype(np.uint8).tobytes()
    return deltas.astype("<u2").tobytes()


def _unpack_deltas(buf: bytes, count: int, bits: int) -> np.ndarray:
    raw = np.frombuffer(buf, dtype=np.uint8)
    if bits == 4:
        out = np.empty(raw.size * 2, dtype=np.uint32)
        out[0::2] = raw & 0x0F
        out[1::2] = raw >> 4
        return out[:count].copy()
    if bits == 8:
        return raw.astype(np.uint32)
    return np.frombuffer(buf, dtype="<u2").astype(np.uint32)


def serialize(ec) -> bytes:
    """Byte-identical to `ecsr.storage.serialize` (`storage.py:389-428`)."""
    dtype = np.dtype(ec.dtype)
    parts = [MAGIC, struct.pack(_HEADER_FMT, VERSION, dtype.itemsize, ec.value_bits,
                                ec.delta_bits, ec.warp_size, ec.num_rows, ec.num_cols,
                                len(ec.sets))]
    for s in ec.sets:
        parts.append(struct.pack(_DESC_FMT, s.granularity, s.vector_size, s.num_blocks,
                                 s.stored_cols, s.real_nnz))
        for arr, dt in ((s.row_indices, "<u4"), (s.block_indptr, "<u8"),
                        (s.base_indices, "<u4")):
            a = np.ascontiguousarray(arr).astype(dt)
            parts.append(struct.pack("<Q", a.size))
            parts.append(a.tobytes())
        parts.append(struct.pack("<Q", s.delta_indices.size))
        parts.append(_pack_deltas(np.asarray(s.delta_indices), ec.delta_bits))
        parts.append(struct.pack("<Q", s.pad_mask.size))
        parts.append(np.packbits(np.asarray(s.pad_mask).astype(np.uint8),
                                 bitorder="little").tobytes())
        vals = np.ascontiguousarray(s.block_values, dtype=dtype.newbyteorder("<"))
        parts.append(struct.pack("<Q", vals.size))
        parts.append(vals.tobytes())
    return b"".join(parts)


class _Reader:
    def __init__(self, data: bytes):
        self.data = memoryview(data)
        self.pos = 0

    def take(self, n: int, what: str) -> bytes:
        if self.pos + n > len(self.data):
            raise ContainerError(
                f"truncated container: needed {n} bytes for {what} at offset {self.pos}")
        out = self.data[self.pos:self.pos + n]
        self.pos += n
        return out

    def unpack(self, fmt: str, what: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt), what))

    def array(self, dtype, what: str) -> np.ndarray:
        (count,) = self.unpack("<Q", what + " length")
        dt = np.dtype(dtype)
        return np.frombuffer(self.take(count * dt.itemsize, what), dtype=dt).copy()


def deserialize(data: bytes) -> EcCsrMatrix:
    """Parse and reject corruption exactly as `storage.py:431-483` does."""
    rd = _Reader(data)
    if bytes(rd.take(4, "magic")) != MAGIC:
        raise ContainerError("bad magic: not an ECSR container")
    version, vsize, vbits, dbits, warp, rows, cols, nsets = rd.unpack(_HEADER_FMT, "header")
    if version != VERSION:
        raise ContainerError(f"unsupported container version {version}")
    if vsize not in (4, 8):
        raise ContainerError(f"unsupported value width {vsize}")
    if vbits not in (16, 32, 64):
        raise ContainerError(f"unsupported value precision tag {vbits}")
    if dbits not in (4, 8, 16):
        raise ContainerError(f"unsupported delta precision {dbits}")
    if warp < 1:
        raise ContainerError("warp size must be positive")
    dtype = np.dtype(np.float32 if vsize == 4 else np.float64)
    sets = []
    for _ in range(nsets):
        g, v, num_blocks, stored, real = rd.unpack(_DESC_FMT, "set descriptor")
        if g < 1 or v < 1:
            raise ContainerError("set granularity and vector size must be positive")
        row_indices = rd.array("<u4", "row_indices")
        block_indptr = rd.array("<u8", "block_indptr").astype(np.int64)
        base_indices = rd.array("<u4", "base_indices")
        (dcount,) = rd.unpack("<Q", "delta_indices length")
        deltas = _unpack_deltas(rd.take(_delta_bytes(dcount, dbits), "delta_indices"),
                                dcount, dbits)
        (mcount,) = rd.unpack("<Q", "pad_mask length")
        mask_bytes = rd.take((mcount + 7) // 8, "pad_mask")
        mask = np.unpackbits(np.frombuffer(mask_bytes, dtype=np.uint8), count=mcount,
                             bitorder="little").astype(bool)
        values = rd.array(dtype.newbyteorder("<"), "block_values").astype(dtype)
        s = EcCsrSet(int(g), int(v), int(num_blocks), int(stored), int(real), row_indices,
                     block_indptr, base_indices, deltas, mask, values)
        check_set_shapes(s, warp)
        sets.append(s)
    if rd.pos != len(data):
        raise ContainerError(f"{len(data) - rd.pos} trailing bytes after container")
    return EcCsrMatrix(int(rows), int(cols), vbits, dbits, warp, sets)


def save_container(ec, path) -> None:
    with open(path, "wb") as fh:
        fh.write(serialize(ec))


def load_container(path) -> EcCsrMatrix:
    with open(path, "rb") as fh:
        return deserialize(fh.read())


# --- validation (executor.py:50-77, storage.py:312-329) ----------------------


def check_set_shapes(s, warp: int) -> None:
    if len(s.block_indptr) != s.num_blocks + 1:
        raise ContainerError("block_indptr length mismatch")
    if s.block_indptr[0] != 0 or np.any(np.diff(s.block_indptr) < 0):
        raise ContainerError("block_indptr must start at 0 and be non-decreasing")
    if int(s.block_indptr[-1]) != s.stored_cols:
        raise ContainerError("block_indptr does not cover stored columns")
    if len(s.delta_indices) != s.stored_cols or len(s.pad_mask) != s.stored_cols:
        raise ContainerError("delta or mask array length mismatch")
    if len(s.block_values) != s.stored_cols * s.granularity:
        raise ContainerError("block_values length mismatch")
    if len(s.row_indices) != s.num_blocks * s.granularity:
        raise ContainerError("row_indices length mismatch")
    if len(s.base_indices) != s.num_blocks * warp:
        raise ContainerError("base_indices length mismatch")
    widths = np.diff(s.block_indptr)
    if np.any(widths % (warp * s.vector_size)):
        raise ContainerError("block widths must be multiples of warp_size * vector_size")


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
