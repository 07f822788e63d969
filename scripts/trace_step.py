"""Timeline of one bench step (launches back to back in one CUDA graph, PDL-chained, no
host syncs): per launch, CTA start / past griddepcontrol.wait / x landed / zero-y gate
open / last warp end, relative to the step's first CTA start. Tuning builds only:

    ECSR_B200_TRACE=2 python scripts/trace_step.py build/libNAME.so [workload] [grouped]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2507_12205_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
_h = ctypes.CDLL(_lib.LIB_PATH)
for _name in list(_lib.SIGNATURES):
    if not hasattr(_h, _name):
        del _lib.SIGNATURES[_name]
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_12205_b200.device import spmv, to_device, vstack  # noqa: E402

lib = _lib.lib()
lib.ecsr_b200_debug_trace.restype = ctypes.c_int32
lib.ecsr_b200_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
lib.ecsr_b200_debug_trace_reset.restype = ctypes.c_int32
lib.ecsr_b200_debug_trace_reset.argtypes = [ctypes.c_void_p]
name = sys.argv[2] if len(sys.argv) > 2 else bench.HEADLINE
launches = bench.WORKLOADS[name]["launches"]
ecs, _ = bench.load_workload(name)
Ws, xs, ys = {}, {}, {}
for ln, names in launches:
    Ws[ln] = to_device(vstack([ecs[n] for n in names]))
    xs[ln] = torch.randn(Ws[ln].num_cols, device="cuda").half()
    ys[ln] = torch.empty(Ws[ln].num_rows, device="cuda")
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    for _ in range(3):
        for ln, _ in launches:
            spmv(Ws[ln], xs[ln], y=ys[ln], stream=stream)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=stream):
    for ln, _ in launches:
        spmv(Ws[ln], xs[ln], y=ys[ln], stream=stream)
for rep in range(3):
    for ln in Ws:
        _lib.check(lib.ecsr_b200_debug_trace_reset(Ws[ln].handle), "reset")
    with torch.cuda.stream(stream):
        graph.replay()  # the step before streams the same weights: warm like the bench
        graph.replay()
    torch.cuda.synchronize()
    tr = {}
    for ln in Ws:
        g = Ws[ln].bytes()["grid"]
        out = np.zeros(16 * g, np.uint64)
        _lib.check(lib.ecsr_b200_debug_trace(Ws[ln].handle, out.ctypes.data, out.size), "trace")
        tr[ln] = out.reshape(g, 16).astype(np.int64)
    t0 = min(t[:, 0].min() for t in tr.values())
    print(f"{os.path.basename(sys.argv[1])} rep {rep}: us from the step's first CTA start")
    for ln, t in tr.items():
        f = lambda i: (t[:, i] - t0) / 1e3  # noqa: E731
        gate = f"gate {np.median(f(14)):6.2f} (max {f(14).max():6.2f})" if t[:, 14].any() else "gate    n/a"
        if t[:, 9].any():
            gate += f" | prod pdl {np.median(f(8)):6.2f} (max {f(8).max():6.2f}) zeroed {np.median(f(9)):6.2f} (max {f(9).max():6.2f})"
        print(f"  {ln:8s} start {f(0).min():6.2f}..{f(0).max():6.2f} pdl {np.median(f(1)):6.2f} "
              f"x {np.median(f(2)):6.2f} (max {f(2).max():6.2f}) {gate} "
              f"end {np.percentile(f(6), 10):6.2f} / {np.median(f(6)):6.2f} / {f(6).max():6.2f}", flush=True)
