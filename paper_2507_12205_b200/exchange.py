"""Row-sharded y exchange over NVLink peer memory (`ecsr_b200_xchg_*`, csrc/ecsr_xchg.cu).

Every rank owns a `y_full` buffer (all ranks' output rows in their final layout) that the
peers map through CUDA IPC. `PeerExchange.run(src)` is ONE kernel, PDL-chained behind the
rank's shard SpMV: it stores this rank's segments of `src` into every rank's `y_full`,
signals each peer and waits for every peer's push -- the all-gather and the assembly of
the sharded step in one launch, over peer stores instead of NCCL.

    ex = PeerExchange(y_full_floats, rank, world)       # torch.distributed initialised
    ex.plan(segments)                                   # [(src_off, dst_off, n)] floats
    ex.run(y_shard, stream)                             # -> ex.y (torch view of y_full)

`ex.y` holds the step's rows until this rank's next `run` (stream order): a peer pushes
its next step into it only after that call has passed its griddepcontrol.wait (the
kernel's ready handshake), however far ahead the peer runs.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


class _Seg(ctypes.Structure):
    _fields_ = [("src_off", ctypes.c_int64), ("dst_off", ctypes.c_int64), ("bytes", ctypes.c_int64)]


class _DeviceArray:
    """__cuda_array_interface__ over the library-owned y_full (float32)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


def shard_segments(bounds_per_launch, slot_offsets, y_offsets, rank: int):
    """Segments (floats) of this rank's rows: for every launch (matrices stacked in one
    handle, each row-sharded by `bounds`), its shard output sits at `slot_offsets[l]` of
    the SpMV output (matrices back to back), and matrix i's rows belong at
    `y_offsets[l] + sum(M_j, j < i) + bounds_i[rank]` of y_full."""
    segs = []
    for bounds, so, yo in zip(bounds_per_launch, slot_offsets, y_offsets):
        within, rows_before = 0, 0
        for b in bounds:
            n = b[rank + 1] - b[rank]
            if n:
                segs.append((so + within, yo + rows_before + b[rank], n))
            within += n
            rows_before += b[-1]
    return segs


class PeerExchange:
    def __init__(self, y_full_floats: int, rank: int, world: int, group=None):
        import torch
        import torch.distributed as dist

        self.rank, self.world, self.n = int(rank), int(world), int(y_full_floats)
        lib = _lib.lib()
        h = ctypes.c_void_p()
        self._h = h
        mine, err = None, None
        try:  # a failing rank still takes part in the handle all-gather below
            _lib.check(lib.ecsr_b200_xchg_create(4 * self.n, self.rank, self.world, ctypes.byref(h)),
                       "ecsr_b200_xchg_create")
            self._h = h
            buf = (ctypes.c_uint8 * 64)()
            _lib.check(lib.ecsr_b200_xchg_handle(h, buf), "ecsr_b200_xchg_handle")
            mine = bytes(buf)
        except Exception as exc:  # noqa: BLE001
            err = exc
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, mine, group=group)
        else:
            handles = [mine]
        if err is not None:
            raise err
        if any(x is None for x in handles):
            raise RuntimeError("peer exchange: another rank could not create its buffer")
        allh = (ctypes.c_uint8 * (64 * self.world)).from_buffer_copy(b"".join(handles))
        _lib.check(lib.ecsr_b200_xchg_open(h, allh), "ecsr_b200_xchg_open")
        ptr = lib.ecsr_b200_xchg_y(h)
        self.y = torch.as_tensor(_DeviceArray(ptr, self.n), device=torch.device("cuda", torch.cuda.current_device()))
        self.segments = []

    def plan(self, segments):
        """segments: (src_off, dst_off, count) in float32 elements."""
        self.segments = [tuple(int(v) for v in s) for s in segments]
        arr = (_Seg * max(len(self.segments), 1))(*[_Seg(4 * a, 4 * b, 4 * n) for a, b, n in self.segments])
        _lib.check(_lib.lib().ecsr_b200_xchg_plan(self._h, arr, len(self.segments)), "ecsr_b200_xchg_plan")

    def run(self, src, stream=None):
        import torch

        if not isinstance(src, torch.Tensor) or not src.is_cuda or src.dtype != torch.float32:
            raise ValueError("src must be a float32 CUDA tensor")
        need = max((a + n for a, _, n in self.segments), default=0)
        if src.numel() < need or not src.is_contiguous():
            raise ValueError(f"src must be contiguous with at least {need} elements")
        s = stream if stream is not None else torch.cuda.current_stream(src.device)
        _lib.check(_lib.lib().ecsr_b200_xchg_run(self._h, ctypes.c_void_p(src.data_ptr()),
                                                 ctypes.c_void_p(s.cuda_stream)), "ecsr_b200_xchg_run")
        return self.y

    def free(self):
        if self._h:
            _lib.lib().ecsr_b200_xchg_free(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def reference_layout(ys_per_launch) -> np.ndarray:
    """The y_full a step must produce: every launch's full y, launches back to back."""
    return np.concatenate([np.asarray(y, np.float32) for y in ys_per_launch])
