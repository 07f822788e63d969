"""Device-resident EC-CSR matrices and the SpMV call (torch-facing API).

`to_device(ec)` validates and packs a container once (`ecsr_b200_pack`); `spmv(W, x)`
is the reference's `executor.spmv_ec(ec, x)` (`pkg/src/ecsr/executor.py:80-96`) on
device tensors: x fp16 [K] -> y fp32 [M], stream-ordered, no host sync. PyTorch only
supplies device memory and streams; all compute is in libecsr_b200.so.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .container import EcCsrMatrix, EcCsrSet, host_sets

_DEVICE_DTYPES = {"f16": _lib.F16, "f32": _lib.F32, "f64": _lib.F64}


def _torch():
    import torch

    return torch


def _host_sets(ec, check_shapes: bool = True):
    return host_sets(ec, check_shapes)


class DeviceMatrix:
    """Opaque handle to a packed container.

    The packed layout is read-only after pack. Each launch also writes a small
    workspace (the overwrite mode's grid-gate counter, the ordered mode's block
    partials); the handle keeps one per CUDA stream (up to 4 streams), so launches
    from different streams may overlap, and launches from one stream are ordered.
    """

    def __init__(self, handle: int, num_rows: int, num_cols: int, device_dtype: str,
                 device_index: int):
        self._handle = ctypes.c_void_p(handle)
        self.num_rows = num_rows
        self.num_cols = num_cols
        self.device_dtype = device_dtype
        self.device_index = device_index

    @property
    def handle(self) -> ctypes.c_void_p:
        if not self._handle:
            raise ValueError("DeviceMatrix was freed")
        return self._handle

    def free(self) -> None:
        if self._handle:
            _lib.lib().ecsr_b200_free(self._handle)
            self._handle = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:  # interpreter shutdown
            pass

    @property
    def x_dtype(self):
        torch = _torch()
        return {"f16": torch.float16, "f32": torch.float32, "f64": torch.float64}[self.device_dtype]

    @property
    def y_dtype(self):
        torch = _torch()
        return torch.float64 if self.device_dtype == "f64" else torch.float32

    def bytes(self) -> dict:
        out = _lib.Bytes()
        _lib.check(_lib.lib().ecsr_b200_bytes(self.handle, ctypes.byref(out)), "ecsr_b200_bytes")
        return out.to_dict()

    @property
    def layout(self) -> str:
        return {1: "tiled", 2: "generic"}[self.bytes()["layout"]]

    def spmv(self, x, y=None, accumulate: bool = False, ordered: bool = False, stream=None):
        return spmv(self, x, y=y, accumulate=accumulate, ordered=ordered, stream=stream)

    def unpack(self, value_dtype=np.float32) -> EcCsrMatrix:
        return unpack(self, value_dtype)


def to_device(ec, device_dtype: str = "f16", force_generic: bool = False,
              device=None, tile_kb: int | None = None, queue_pct: int | None = None) -> DeviceMatrix:
    """Validate once and upload (replaces the per-call `validate_container`,
    `executor.py:85-86`). Raises ContainerError exactly where the reference would.
    Tiled-layout options: `tile_kb` overrides the tile size (1..64 KB), `queue_pct` the
    cost share (0..100 %) of each CTA's tiles drawn from the launch's tail queue."""
    torch = _torch()
    if device_dtype not in _DEVICE_DTYPES:
        raise ValueError(f"device_dtype must be one of {sorted(_DEVICE_DTYPES)}")
    dev = torch.device("cuda" if device is None else device)
    index = dev.index if dev.index is not None else torch.cuda.current_device()
    arr, keep, dtype = _host_sets(ec)
    out = ctypes.c_void_p()
    flags = _lib.PACK_FORCE_GENERIC if force_generic else _lib.PACK_DEFAULT
    if tile_kb is not None:
        if not 1 <= int(tile_kb) <= 64:
            raise ValueError("tile_kb must be in [1, 64]")
        flags |= int(tile_kb) << 8
    if queue_pct is not None:
        if not 0 <= int(queue_pct) <= 100:
            raise ValueError("queue_pct must be in [0, 100]")
        flags |= ((int(queue_pct) & 0x7F) | 0x80) << 16
    with torch.cuda.device(index):
        rc = _lib.lib().ecsr_b200_pack(arr, len(ec.sets), int(ec.num_rows), int(ec.num_cols),
                                       int(ec.warp_size), int(ec.delta_bits), int(ec.value_bits),
                                       _lib.dtype_code(dtype), _DEVICE_DTYPES[device_dtype],
                                       flags, ctypes.byref(out))
    _lib.check(rc, "ecsr_b200_pack")
    del keep
    return DeviceMatrix(out.value, int(ec.num_rows), int(ec.num_cols), device_dtype, index)


def _blob(blob_or_path):
    if isinstance(blob_or_path, (bytes, bytearray, memoryview)):
        return bytes(blob_or_path)
    with open(blob_or_path, "rb") as fh:
        return fh.read()


def parse_blob(blob_or_path) -> dict:
    """Host-only parse + shape check of a `.ecsr` blob by the native loader; raises
    ContainerError with the reference's message on corruption (`storage.py:431-483`)."""
    data = _blob(blob_or_path)
    info = _lib.BlobInfo()
    buf = ctypes.create_string_buffer(data, len(data))
    _lib.check(_lib.lib().ecsr_b200_parse(buf, len(data), ctypes.byref(info)), "ecsr_b200_parse")
    return info.to_dict()


def load_device(blob_or_path, device_dtype: str = "f16", force_generic: bool = False,
                device=None) -> DeviceMatrix:
    """`.ecsr` blob (bytes or path) straight to a device handle: the native loader parses
    the wire format and packs without building numpy sets (`load_container` + `to_device`
    in one C call, same rejection rules)."""
    torch = _torch()
    if device_dtype not in _DEVICE_DTYPES:
        raise ValueError(f"device_dtype must be one of {sorted(_DEVICE_DTYPES)}")
    data = _blob(blob_or_path)
    info = parse_blob(data)
    dev = torch.device("cuda" if device is None else device)
    index = dev.index if dev.index is not None else torch.cuda.current_device()
    out = ctypes.c_void_p()
    flags = _lib.PACK_FORCE_GENERIC if force_generic else _lib.PACK_DEFAULT
    buf = ctypes.create_string_buffer(data, len(data))
    with torch.cuda.device(index):
        rc = _lib.lib().ecsr_b200_load(buf, len(data), _DEVICE_DTYPES[device_dtype], flags,
                                       ctypes.byref(out))
    _lib.check(rc, "ecsr_b200_load")
    return DeviceMatrix(out.value, int(info["num_rows"]), int(info["num_cols"]), device_dtype, index)


def spmv(W: DeviceMatrix, x, y=None, accumulate: bool = False, ordered: bool = False,
         stream=None, memset_y: bool = False):
    """y = W x (y += W x with accumulate). x: device tensor [K] of W.x_dtype.

    ordered=True selects the bitwise-reproducible reduction (per-block partials summed
    per row in container order, exactly the reference's y order); the default uses
    red.global.add.f32 and is the fast path. memset_y makes the overwrite mode clear y
    with a memset before an ungated launch (the path taken automatically when the whole
    grid cannot be resident, e.g. under an MPS thread limit).
    """
    torch = _torch()
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError("x must be a CUDA tensor (use spmv_host for host buffers)")
    if x.shape != (W.num_cols,):
        raise ValueError(f"x has shape {tuple(x.shape)}, expected ({W.num_cols},)")
    if x.dtype != W.x_dtype:
        raise ValueError(f"x must be {W.x_dtype}, got {x.dtype}")
    if x.device.index != W.device_index:
        raise ValueError(f"x is on cuda:{x.device.index}, the matrix on cuda:{W.device_index}")
    x = x.contiguous()
    if y is None:
        y = torch.empty(W.num_rows, dtype=W.y_dtype, device=x.device)
        if accumulate:
            y.zero_()
    elif y.shape != (W.num_rows,) or y.dtype != W.y_dtype or not y.is_contiguous():
        raise ValueError("y must be a contiguous device tensor of shape (num_rows,) and y dtype")
    elif not y.is_cuda or y.device.index != W.device_index:
        raise ValueError(f"y must be on cuda:{W.device_index}")
    mode = (_lib.SPMV_ACCUMULATE if accumulate else _lib.SPMV_OVERWRITE) | (
        _lib.SPMV_ORDERED if ordered else 0) | (_lib.SPMV_MEMSET_Y if memset_y else 0)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    rc = _lib.lib().ecsr_b200_spmv(W.handle, ctypes.c_void_p(x.data_ptr()),
                                   ctypes.c_void_p(y.data_ptr()), mode,
                                   ctypes.c_void_p(s.cuda_stream))
    _lib.check(rc, "ecsr_b200_spmv")
    return y


class SpmvGroup:
    """Several independent products y_i = W_i x_i in ONE launch (`ecsr_b200_group_*`).

    The members' CTAs run side by side, so the group pays one launch ramp and one tail
    instead of one per matrix -- e.g. the projections of a decoder layer whose inputs are
    all ready. Every member must use the tiled layout; the group keeps references to its
    matrices (they must outlive it)."""

    def __init__(self, mats):
        mats = list(mats)
        if not mats:
            raise ValueError("empty group")
        if len({W.device_index for W in mats}) != 1:
            raise ValueError("group members must be on one device")
        self.mats = mats
        self.device_index = mats[0].device_index
        arr = (ctypes.c_void_p * len(mats))(*[W.handle.value for W in mats])
        out = ctypes.c_void_p()
        _lib.check(_lib.lib().ecsr_b200_group_create(arr, len(mats), ctypes.byref(out)),
                   "ecsr_b200_group_create")
        self._handle = out

    def __len__(self):
        return len(self.mats)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h:
            try:
                _lib.lib().ecsr_b200_group_free(h)
            except Exception:  # noqa: BLE001 -- interpreter shutdown
                pass
            self._handle = None

    def info(self) -> dict:
        launches, grid = ctypes.c_int32(), ctypes.c_int32()
        ctas = (ctypes.c_int32 * len(self.mats))()
        _lib.check(_lib.lib().ecsr_b200_group_info(self._handle, ctypes.byref(launches), ctypes.byref(grid),
                                                   ctas, len(self.mats)), "ecsr_b200_group_info")
        return {"launches": launches.value, "grid": grid.value, "ctas": list(ctas)}

    def spmv(self, xs, ys=None, accumulate: bool = False, ordered: bool = False, stream=None,
             memset_y: bool = False):
        """ys[i] = W_i xs[i] (+= with accumulate) for every member, one launch."""
        torch = _torch()
        if len(xs) != len(self.mats):
            raise ValueError(f"expected {len(self.mats)} inputs, got {len(xs)}")
        if ys is None:
            ys = [None] * len(self.mats)
        outs = []
        for W, x, y in zip(self.mats, xs, ys):
            if not isinstance(x, torch.Tensor) or not x.is_cuda or x.shape != (W.num_cols,) \
                    or x.dtype != W.x_dtype or x.device.index != W.device_index or not x.is_contiguous():
                raise ValueError(f"each x must be a contiguous {W.x_dtype} CUDA tensor of shape ({W.num_cols},) "
                                 f"on cuda:{W.device_index}")
            if y is None:
                y = torch.empty(W.num_rows, dtype=W.y_dtype, device=x.device)
                if accumulate:
                    y.zero_()
            elif y.shape != (W.num_rows,) or y.dtype != W.y_dtype or not y.is_contiguous() \
                    or not y.is_cuda or y.device.index != W.device_index:
                raise ValueError(f"each y must be a contiguous {W.y_dtype} tensor of shape ({W.num_rows},) "
                                 f"on cuda:{W.device_index}")
            outs.append(y)
        xa = (ctypes.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
        ya = (ctypes.c_void_p * len(outs))(*[y.data_ptr() for y in outs])
        mode = (_lib.SPMV_ACCUMULATE if accumulate else _lib.SPMV_OVERWRITE) | (
            _lib.SPMV_ORDERED if ordered else 0) | (_lib.SPMV_MEMSET_Y if memset_y else 0)
        s = stream if stream is not None else torch.cuda.current_stream(xs[0].device)
        _lib.check(_lib.lib().ecsr_b200_group_spmv(self._handle, xa, ya, mode, ctypes.c_void_p(s.cuda_stream)),
                   "ecsr_b200_group_spmv")
        return outs


class _IoSpan(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("bytes", ctypes.c_int64)]


def host_io(pairs, stream=None, after_predecessor: bool = False) -> None:
    """A step's host traffic as one kernel in the stream's launch chain
    (`ecsr_b200_host_io`, csrc/ecsr_hostio.cu): copies every (src, dst) tensor pair --
    CUDA tensors of the current device or pinned host tensors, same byte size, 16-B
    aligned starts, contiguous -- without a copy stream, so the next SpMV keeps its PDL edge.
    The copies overlap the preceding launch unless `after_predecessor` (then they read
    what it wrote); the caller keeps the preceding launch off the spans."""
    torch = _torch()
    spans = []
    for src, dst in pairs:
        for t in (src, dst):
            if not isinstance(t, torch.Tensor) or not t.is_contiguous():
                raise ValueError("host_io: contiguous tensors required")
            if not t.is_cuda and not t.is_pinned():
                raise ValueError("host_io: host tensors must be pinned")
        nb = src.numel() * src.element_size()
        if nb != dst.numel() * dst.element_size():
            raise ValueError(f"host_io: src has {nb} bytes, dst {dst.numel() * dst.element_size()}")
        spans.append(_IoSpan(src.data_ptr(), dst.data_ptr(), nb))
    devs = {t.device.index for p in pairs for t in p if t.is_cuda}
    if len(devs) > 1:
        raise ValueError(f"host_io: tensors on several devices {sorted(devs)}")
    dev = torch.device("cuda", devs.pop()) if devs else (stream.device if stream is not None
                                                         else torch.device("cuda", torch.cuda.current_device()))
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    arr = (_IoSpan * max(1, len(spans)))(*spans)
    with torch.cuda.device(dev):  # the C-ABI checks device pointers against the current device
        _lib.check(_lib.lib().ecsr_b200_host_io(arr, len(spans), _lib.IO_AFTER_PREDECESSOR if after_predecessor
                                                else 0, ctypes.c_void_p(s.cuda_stream)), "ecsr_b200_host_io")


def spmv_host(W: DeviceMatrix, x: np.ndarray, ordered: bool = False) -> np.ndarray:
    """End-to-end call with host buffers: H2D x, SpMV, D2H y (synchronous)."""
    torch = _torch()
    xt = torch.from_numpy(np.ascontiguousarray(x).astype(
        {"f16": np.float16, "f32": np.float32, "f64": np.float64}[W.device_dtype]))
    xd = xt.to(f"cuda:{W.device_index}", non_blocking=False)
    y = spmv(W, xd, ordered=ordered)
    return y.cpu().numpy()


def unpack(W: DeviceMatrix, value_dtype=np.float32) -> EcCsrMatrix:
    """Read the device layout back into reference set arrays (`storage.py:50-62`)."""
    lib = _lib.lib()
    M, K = ctypes.c_int64(), ctypes.c_int64()
    nsets, warp, dbits, vbits, ddt = (ctypes.c_int32() for _ in range(5))
    _lib.check(lib.ecsr_b200_info(W.handle, ctypes.byref(M), ctypes.byref(K), ctypes.byref(nsets),
                                  ctypes.byref(warp), ctypes.byref(dbits), ctypes.byref(vbits),
                                  ctypes.byref(ddt)), "ecsr_b200_info")
    vdt = np.dtype(value_dtype)
    sets, outs = [], (_lib.OutSet * max(nsets.value, 1))()
    for i in range(nsets.value):
        info = _lib.SetInfo()
        _lib.check(lib.ecsr_b200_set_info(W.handle, i, ctypes.byref(info)), "ecsr_b200_set_info")
        g, nb, st = info.granularity, info.num_blocks, info.stored_cols
        s = EcCsrSet(info.granularity, info.vector_size, nb, st, info.real_nnz,
                     np.zeros(g * nb, np.uint32), np.zeros(nb + 1, np.int64),
                     np.zeros(warp.value * nb, np.uint32), np.zeros(st, np.uint32),
                     np.zeros(st, np.bool_), np.zeros(g * st, vdt))
        sets.append(s)
        outs[i] = _lib.OutSet(_lib.ptr(s.row_indices), s.block_indptr.ctypes.data,
                              _lib.ptr(s.base_indices), _lib.ptr(s.delta_indices),
                              _lib.ptr(s.pad_mask.view(np.uint8)), _lib.ptr(s.block_values))
    _lib.check(lib.ecsr_b200_unpack(W.handle, outs, nsets.value, _lib.dtype_code(vdt)),
               "ecsr_b200_unpack")
    return EcCsrMatrix(M.value, K.value, vbits.value, dbits.value, warp.value, sets)


def vstack(ecs) -> EcCsrMatrix:
    """Stack containers by rows into one (fused QKV / gate-up): y = [A_0 x; A_1 x; ...].

    The sets are concatenated in order with row ids offset, which is a valid
    container for spmv_ec semantics (any set order is; executor.py:90-95).
    """
    ecs = list(ecs)
    if not ecs:
        raise ValueError("nothing to stack")
    k = ecs[0].num_cols
    w, b = ecs[0].warp_size, ecs[0].delta_bits
    sets, off = [], 0
    dtype = np.result_type(*[np.dtype(e.dtype) for e in ecs])
    for e in ecs:
        if e.num_cols != k or e.warp_size != w or e.delta_bits != b:
            raise ValueError("stacked containers must share num_cols, warp_size and delta_bits")
        for s in e.sets:
            sets.append(EcCsrSet(s.granularity, s.vector_size, s.num_blocks, s.stored_cols,
                                 s.real_nnz, np.asarray(s.row_indices, np.uint32) + np.uint32(off),
                                 s.block_indptr, s.base_indices, s.delta_indices, s.pad_mask,
                                 np.asarray(s.block_values, dtype)))
        off += e.num_rows
    return EcCsrMatrix(off, k, ecs[0].value_bits, b, w, sets)


def to_f16(values: np.ndarray) -> np.ndarray:
    """The packer's f32/f64 -> f16 rounding (IEEE RNE), for host-side parity checks."""
    v = np.ascontiguousarray(values)
    out = np.empty(v.shape, dtype=np.uint16)
    _lib.check(_lib.lib().ecsr_b200_to_f16(v.ctypes.data, _lib.dtype_code(v.dtype),
                                           out.ctypes.data, v.size), "ecsr_b200_to_f16")
    return out.view(np.float16)
