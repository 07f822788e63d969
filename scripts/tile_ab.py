"""Grouped step time of a bench workload at several tile sizes, interleaved in ONE
process (A, B, C, A, B, C, ...) so clock / power drift hits every arm alike.
python scripts/tile_ab.py WORKLOAD [tile_kb ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_12205_b200.device import SpmvGroup, to_device, vstack  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.HEADLINE
kbs = [int(v) for v in sys.argv[2:]] or [0, 24]  # 0: the packer's default
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
ecs, _ = bench.load_workload(name)
launches = bench.WORKLOADS[name]["launches"]
stacked = [vstack([ecs[n] for n in names]) for _, names in launches]
step_bytes = sum(bench.model_bytes(ecs[n]) for _, names in launches for n in names)
rng = np.random.default_rng(1)
xs = [torch.from_numpy(rng.uniform(-1, 1, e.num_cols).astype(np.float16)).cuda() for e in stacked]
ys = [torch.empty(e.num_rows, device=dev) for e in stacked]
arms = {}
for kb in kbs:
    g = SpmvGroup([to_device(e, tile_kb=kb or None) for e in stacked])
    with torch.cuda.stream(stream):
        g.spmv(xs, ys, stream=stream)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=stream):
        for _ in range(5):
            g.spmv(xs, ys, stream=stream)
    arms[kb] = (g, gr, [])
for rep in range(8):
    for kb, (_, gr, ts) in arms.items():
        ms, _ = bench.time_graph(gr, 10, 2, stream)
        ts.append(ms / 5 * 1e3)
for kb, (g, _, ts) in arms.items():
    med = float(np.median(ts))
    print(f"{name} tile {kb} KB: median {med:.2f} us ({step_bytes / med / 1e3:.0f} GB/s), "
          f"min {min(ts):.2f} max {max(ts):.2f} | {g.info()}", flush=True)
