"""Access trace of the device layout and its coalescing audit.

The reference traces its canonical walk (`spmv_ec_traced`, `pkg/src/ecsr/executor.py:
106-168`) and audits it with `check_coalescing` (`executor.py:171-221`): every warp step
reads one contiguous span of exactly W*v deltas / W*v*g values, aligned to its own
width, and a warp's spans tile its block exactly. `device_trace(W)` produces the same
records for what the B200 kernel reads (`ecsr_b200_trace`: the tiled kernel's own
pointer arithmetic replayed over the device arena), so the reference's auditor can be
run on them unchanged; `check_device_coalescing` restates that audit and adds the
device-side rules of the tiled layout: every span starts 16-B aligned in the arena
(whole bulk-copied 16-B chunks; each lane's `lane_bytes` load is naturally aligned) and
is exactly one reference chunk (32v delta bytes, 64vg fp16 value bytes).
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple

import numpy as np

from . import _lib

ARRAYS = ("deltas", "values")


class TraceRecord(NamedTuple):
    """Field-compatible with the reference's TraceRecord (executor.py:26-34), plus
    where the span sits in device memory."""

    warp: int
    step: int
    array: str
    set_index: int
    start: int
    span: int
    dev_offset: int = 0
    dev_bytes: int = 0
    lane_bytes: int = 0


class _Rec(ctypes.Structure):
    _fields_ = [("warp", ctypes.c_int64), ("step", ctypes.c_int32), ("array", ctypes.c_int32),
                ("set_index", ctypes.c_int32), ("lane_bytes", ctypes.c_int32),
                ("start", ctypes.c_int64), ("span", ctypes.c_int64),
                ("dev_offset", ctypes.c_int64), ("dev_bytes", ctypes.c_int64)]


_DTYPE = np.dtype([(name, np.int64 if ctype is ctypes.c_int64 else np.int32)
                   for name, ctype in _Rec._fields_])
assert _DTYPE.itemsize == ctypes.sizeof(_Rec)


def device_trace_array(W) -> np.ndarray:
    """The raw trace of a DeviceMatrix as a structured numpy array (fields of
    ecsr_trace_rec, include/ecsr_b200.h)."""
    lib = _lib.lib()
    n = ctypes.c_int64(0)
    _lib.check(lib.ecsr_b200_trace(W.handle, None, 0, ctypes.byref(n)), "ecsr_b200_trace")
    out = np.zeros(n.value, dtype=_DTYPE)
    if n.value:
        _lib.check(lib.ecsr_b200_trace(W.handle, out.ctypes.data, n.value, ctypes.byref(n)),
                   "ecsr_b200_trace")
    return out


def device_trace(W) -> list[TraceRecord]:
    """Trace records in the reference's shape (warp, step, array, set_index, start,
    span), in the order the kernel reads them."""
    a = device_trace_array(W)
    return [TraceRecord(int(r["warp"]), int(r["step"]), ARRAYS[int(r["array"])], int(r["set_index"]),
                        int(r["start"]), int(r["span"]), int(r["dev_offset"]), int(r["dev_bytes"]),
                        int(r["lane_bytes"])) for r in a]


def check_device_coalescing(ec, trace, tiled: bool = True) -> list[str]:
    """The reference's audit (executor.py:171-221) restated over `trace`, plus the tiled
    layout's device rules. Returns a list of violations (empty = clean)."""
    violations: list[str] = []
    blocks = []
    for si, s in enumerate(ec.sets):
        for b in range(int(s.num_blocks)):
            blocks.append((si, int(s.block_indptr[b]), int(s.block_indptr[b + 1]),
                           int(s.granularity), int(s.vector_size)))
    seen: dict = {}
    for rec in trace:
        if rec.array not in ARRAYS:
            continue
        if rec.warp >= len(blocks):
            violations.append(f"warp {rec.warp} beyond container blocks")
            continue
        si, start, stop, g, v = blocks[rec.warp]
        mult = g if rec.array == "values" else 1
        width = ec.warp_size * v * mult
        lo, hi = start * mult, stop * mult
        if rec.set_index != si:
            violations.append(f"warp {rec.warp}: read from set {rec.set_index}, expected {si}")
        if rec.span != width:
            violations.append(f"warp {rec.warp}: {rec.array} span {rec.span}, expected {width}")
        if rec.start % width:
            violations.append(f"warp {rec.warp}: {rec.array} read at {rec.start} not {width}-aligned")
        if not (lo <= rec.start and rec.start + rec.span <= hi):
            violations.append(f"warp {rec.warp}: {rec.array} read [{rec.start}, {rec.start + rec.span}) "
                              f"outside block range [{lo}, {hi})")
        if tiled:
            want = 32 * v if rec.array == "deltas" else 64 * v * g
            if rec.dev_bytes != want:
                violations.append(f"warp {rec.warp}: device {rec.array} span {rec.dev_bytes} B, expected {want}")
            if rec.dev_offset % 16:
                violations.append(f"warp {rec.warp}: device {rec.array} span at byte {rec.dev_offset} "
                                  "not 16-B aligned")
            if rec.lane_bytes <= 0 or (rec.dev_offset % min(rec.lane_bytes, 16)):
                violations.append(f"warp {rec.warp}: lane load of {rec.lane_bytes} B misaligned")
        seen.setdefault((rec.warp, rec.array), []).append(rec.start)
    for (w, array), starts in seen.items():
        si, start, stop, g, v = blocks[w]
        mult = g if array == "values" else 1
        width = ec.warp_size * v * mult
        if sorted(starts) != list(range(start * mult, stop * mult, width)):
            violations.append(f"warp {w}: {array} steps do not tile the block exactly")
    for w, (si, start, stop, g, v) in enumerate(blocks):
        if stop > start and (w, "deltas") not in seen:
            violations.append(f"warp {w}: block of {stop - start} stored columns never read")
    return violations


def as_reference_trace(trace, executor_module):
    """Wrap our records in the reference's AccessTrace (executor.py:37-47) so its own
    check_coalescing can audit them."""
    tr = executor_module.AccessTrace()
    for r in trace:
        tr.add(r.warp, r.step, r.array, r.set_index, r.start, r.span)
    return tr
