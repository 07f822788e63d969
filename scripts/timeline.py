"""Where an isolated launch's time goes (tuning build: scripts/build_exp.sh tune
-DECSR_B200_TUNING; run with ECSR_B200_TRACE=2).

Per launch kind of the bench layer, after an L2 flush: the CUDA-event time of the
launch alone, and from the per-CTA globaltimer stamps (relative to the first CTA
start): CTA start spread, consumer past griddepcontrol.wait, x landed, first tile
landed, last warp end. The gap event-time minus (last end - first start) is launch
latency + teardown, which no kernel change can remove."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_12205_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "build", "libtune.so")  # ECSR_B200_PRE etc. apply
import bench  # noqa: E402
from paper_2507_12205_b200.device import spmv, to_device, vstack  # noqa: E402

lib = _lib.lib()
lib.ecsr_b200_debug_trace.restype = ctypes.c_int32
lib.ecsr_b200_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
lib.ecsr_b200_debug_trace_reset.restype = ctypes.c_int32
lib.ecsr_b200_debug_trace_reset.argtypes = [ctypes.c_void_p]

wl = sys.argv[1] if len(sys.argv) > 1 else bench.HEADLINE
ecs, _ = bench.load_workload(wl)
flush = torch.empty(1 << 29, dtype=torch.uint8, device="cuda")
for ln, names in bench.WORKLOADS[wl]["launches"]:
    W = to_device(vstack([ecs[n] for n in names]))
    x = torch.randn(W.num_cols, device="cuda").half()
    y = torch.empty(W.num_rows, device="cuda")
    for _ in range(3):
        spmv(W, x, y=y)
    torch.cuda.synchronize()
    grid = W.bytes()["grid"]
    evs, rows = [], []
    for rep in range(8):
        _lib.check(lib.ecsr_b200_debug_trace_reset(W.handle), "reset")
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        spmv(W, x, y=y)
        b.record()
        torch.cuda.synchronize()
        evs.append(a.elapsed_time(b) * 1e3)
        out = np.zeros(16 * grid, dtype=np.uint64)
        _lib.check(lib.ecsr_b200_debug_trace(W.handle, out.ctypes.data, out.size), "trace")
        t = out.reshape(grid, 16).astype(np.int64)
        t0 = t[:, 0].min()
        rel = lambda i: (t[:, i] - t0) / 1e3  # noqa: E731
        rows.append([np.median(rel(0)), rel(0).max(), np.median(rel(1)), np.median(rel(2)),
                     np.median(rel(3)), np.median(rel(6)), rel(6).min(), rel(6).max()])
    r = np.median(np.array(rows), axis=0)
    ev = float(np.median(evs))
    mb = sum(bench.model_bytes(ecs[n]) for n in names) / 1e6
    print(f"{ln:8s} {mb:6.1f} MB  event {ev:6.2f} us | start med {r[0]:5.2f} max {r[1]:5.2f} | "
          f"pdl {r[2]:5.2f} x {r[3]:5.2f} tile0 {r[4]:5.2f} | end min {r[6]:6.2f} med {r[5]:6.2f} "
          f"max {r[7]:6.2f} | outside kernel {ev - r[7]:5.2f} | stream {mb / 1e3 / 6.5e-3:5.2f} us @6.5TB/s",
          flush=True)
    W.free()
