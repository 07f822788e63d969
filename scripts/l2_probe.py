"""L2-resident vs HBM-streamed time of each bench launch (tuning aid): one handle
replayed back to back (its arena stays in the 126 MB L2 when small enough) vs rotating
copies whose arenas together exceed L2. The gap says how much of a launch is the HBM
stream and how much is on-chip work (consumer decode, ramp, tail)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2507_12205_b200.device import spmv, to_device, vstack
from probe import timed_graph

ecs, _ = bench.load_workload()
for ln, names in bench.LAUNCHES:
    ec = vstack([ecs[n] for n in names])
    W = to_device(ec)
    arena = W.bytes()["device_arena_bytes"]
    n = max(2, int(2 * 126e6 / arena) + 1)
    Ws = [W] + [to_device(ec) for _ in range(n - 1)]
    x = torch.randn(ec.num_cols, device="cuda").half()
    ys = [torch.zeros(ec.num_rows, device="cuda") for _ in range(n)]
    hot = timed_graph(lambda: [spmv(W, x, y=ys[0]) for _ in range(n)], reps=20) / n
    cold = timed_graph(lambda: [spmv(Ws[i], x, y=ys[i]) for i in range(n)], reps=20) / n
    print(f"{ln:8s} arena {arena/1e6:6.1f} MB  L2-hot {hot:6.2f} us ({arena/hot/1e3:6.0f} GB/s)  "
          f"streamed {cold:6.2f} us ({arena/cold/1e3:6.0f} GB/s)", flush=True)
