"""A/B timing of the bench step with a given library build (tuning knobs via env).

    python scripts/step_ab.py build/libtune.so [workload]

Prints the step time (graph of 5 consecutive steps, CUDA events) and each launch kind
alone (graph of one launch, after the whole step streamed through L2), like bench.py."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_12205_b200 import _lib  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    import ctypes

    _lib.LIB_PATH = os.path.abspath(sys.argv.pop(1))
    _h = ctypes.CDLL(_lib.LIB_PATH)  # an older build may lack newer entry points
    for _name in list(_lib.SIGNATURES):
        if not hasattr(_h, _name):
            del _lib.SIGNATURES[_name]
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_12205_b200.device import spmv  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.HEADLINE
dev = torch.device("cuda", 0)
if "ecsr_b200_group_create" not in _lib.SIGNATURES:
    class _NoGroup:
        def __init__(self, *a):
            pass
    import paper_2507_12205_b200.device as _dev
    _dev.SpmvGroup = _NoGroup
wl = bench.Workload(name, dev)
stream = torch.cuda.Stream(dev)
spg = 5
g = wl.graph(stream, spg, chained=True)
ms, _ = bench.time_graph(g, 20, 3, stream)
ms /= spg
res = {}
for ln, _ in wl.launches:
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=stream):
        spmv(wl.handles[ln], wl.xs[ln], y=wl.ys[ln], stream=stream)
    tot, n = 0.0, 20
    with torch.cuda.stream(stream):
        for _ in range(3):
            g.replay()
            g1.replay()
        for _ in range(n):
            g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g1.replay()
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
    res[ln] = tot / n * 1e3
if "ecsr_b200_group_create" in _lib.SIGNATURES:
    gg = wl.graph(stream, spg)
    mg, _ = bench.time_graph(gg, 20, 3, stream)
    res["GROUPED-step"] = mg / spg * 1e3
env = {k: v for k, v in os.environ.items() if k.startswith("ECSR_")}
print(f"{name} {env} step {ms * 1e3:.2f} us = {wl.step_bytes / (ms * 1e-3) / 1e9:.1f} GB/s | "
      + " ".join(f"{k} {v:.2f}" for k, v in res.items()), flush=True)
