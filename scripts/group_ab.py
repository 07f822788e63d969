"""Step time of a bench workload: 4 chained launches vs one grouped launch (graphs of
5 consecutive steps, CUDA events).  python scripts/group_ab.py [lib.so] [workload]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_12205_b200 import _lib  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    _lib.LIB_PATH = os.path.abspath(sys.argv.pop(1))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_12205_b200.device import SpmvGroup  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.HEADLINE
dev = torch.device("cuda", 0)
wl = bench.Workload(name, dev)
stream = torch.cuda.Stream(dev)
lns = [ln for ln, _ in wl.launches]
grp = SpmvGroup([wl.handles[ln] for ln in lns])
xs = [wl.xs[ln] for ln in lns]
ys = [wl.ys[ln] for ln in lns]


def graph(body, n):
    with torch.cuda.stream(stream):
        body()
        body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(n):
            body()
    return g


for rep in range(2):
    gc = graph(lambda: wl.step_chained(stream), 5)
    gg = graph(lambda: grp.spmv(xs, ys, stream=stream), 5)
    mc, _ = bench.time_graph(gc, 20, 3, stream)
    mg, _ = bench.time_graph(gg, 20, 3, stream)
    g1 = graph(lambda: grp.spmv(xs, ys, stream=stream), 1)
    m1, _ = bench.time_graph(g1, 50, 3, stream)
    f = lambda ms: wl.step_bytes / (ms * 1e-3) / 1e9  # noqa: E731
    print(f"{name}: chained {mc / 5 * 1e3:.2f} us ({f(mc / 5):.0f} GB/s) | grouped {mg / 5 * 1e3:.2f} us "
          f"({f(mg / 5):.0f} GB/s) | grouped, 1 per graph {m1 * 1e3:.2f} us ({f(m1):.0f} GB/s) | {grp.info()}",
          flush=True)
