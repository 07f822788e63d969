"""Per-CTA timeline of the grouped bench step (tuning build, ECSR_B200_TRACE=2):
per member, CTA start / x landed / gate open / last warp end, relative to the step's
first CTA start, and the CTA end spread that the tail queue has to absorb.

    ECSR_B200_TRACE=2 python scripts/trace_group.py build/libNAME.so [workload]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2507_12205_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_12205_b200.device import SpmvGroup, to_device, vstack  # noqa: E402

lib = _lib.lib()
fn = lib.ecsr_b200_debug_group_trace
fn.restype = ctypes.c_int32
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32]
name = sys.argv[2] if len(sys.argv) > 2 else bench.HEADLINE
launches = bench.WORKLOADS[name]["launches"]
ecs, _ = bench.load_workload(name)
Ws = [to_device(vstack([ecs[n] for n in names])) for _, names in launches]
g = SpmvGroup(Ws)
info = g.info()
xs = [torch.randn(W.num_cols, device="cuda").half() for W in Ws]
ys = [torch.empty(W.num_rows, device="cuda") for W in Ws]
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    for _ in range(3):
        g.spmv(xs, ys, stream=stream)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=stream):
    g.spmv(xs, ys, stream=stream)
grid = info["grid"]
bounds = np.cumsum([0] + info["ctas"])
for rep in range(3):
    _lib.check(fn(g._handle, None, 0, 1), "reset")
    with torch.cuda.stream(stream):
        graph.replay()
        graph.replay()  # traced: the second (warm, after a step like the bench's)
    torch.cuda.synchronize()
    out = np.zeros(16 * grid, np.uint64)
    _lib.check(fn(g._handle, out.ctypes.data, out.size, 0), "trace")
    t = out.reshape(grid, 16).astype(np.int64)
    t0 = t[:, 0].min()
    f = lambda i: (t[:, i] - t0) / 1e3  # noqa: E731
    end = f(6)
    print(f"rep {rep}: start {f(0).min():.2f}..{f(0).max():.2f} x med {np.median(f(2)):.2f} "
          f"gate med {np.median(f(14)):.2f} max {f(14).max():.2f} | end p10 {np.percentile(end, 10):.2f} "
          f"med {np.median(end):.2f} max {end.max():.2f} us", flush=True)
