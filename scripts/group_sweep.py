"""Sweep the grouped step over packing / launch knobs (tuning build): tile size,
tail-queue share, tiles streamed before griddepcontrol.wait. Encodes once.

    python scripts/group_sweep.py build/libNAME.so [workload]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_12205_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_12205_b200.device import SpmvGroup, spmv, to_device, vstack  # noqa: E402

name = sys.argv[2] if len(sys.argv) > 2 else bench.HEADLINE
ecs, _ = bench.load_workload(name)
launches = bench.WORKLOADS[name]["launches"]
stacked = {ln: vstack([ecs[n] for n in names]) for ln, names in launches}
step_bytes = sum(bench.model_bytes(e) for e in ecs.values())
stream = torch.cuda.Stream()
xs = [torch.randn(stacked[ln].num_cols, device="cuda").half() for ln, _ in launches]
ys = [torch.empty(stacked[ln].num_rows, device="cuda") for ln, _ in launches]


def run(tile_kb=None, queue_pct=None, pre=None, chained=False):
    if pre is None:
        os.environ.pop("ECSR_B200_PRE", None)
    else:
        os.environ["ECSR_B200_PRE"] = str(pre)
    Ws = [to_device(stacked[ln], tile_kb=tile_kb, queue_pct=queue_pct) for ln, _ in launches]
    g = SpmvGroup(Ws)

    def body():
        if chained:
            for W, x, y in zip(Ws, xs, ys):
                spmv(W, x, y=y, stream=stream)
        else:
            g.spmv(xs, ys, stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(3):
            body()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=stream):
        for _ in range(5):
            body()
    ms, _ = bench.time_graph(gr, 20, 3, stream)
    ms /= 5
    print(f"{name} {'chained' if chained else 'grouped'} tile_kb={tile_kb} queue_pct={queue_pct} pre={pre}: "
          f"{ms * 1e3:.2f} us {step_bytes / (ms * 1e-3) / 1e9:.0f} GB/s", flush=True)
    del g, Ws


qs = [int(v) for v in os.environ.get("QS", "5,30,40,50,60,75,90,100").split(",")]
for chained in (False, True):
    for q in qs:
        run(queue_pct=q, chained=chained)
