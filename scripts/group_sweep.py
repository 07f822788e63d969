"""Sweep the tail-queue share of the grouped step (ECSR_B200_GROUP_QPCT) and of the
chained step (the handles' pack-time share), tuning build. Encodes once.

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


def run(queue_pct=None, chained=False):
    if chained:
        Ws = [to_device(stacked[ln], queue_pct=queue_pct) for ln, _ in launches]
    else:
        os.environ["ECSR_B200_GROUP_QPCT"] = str(queue_pct)
        Ws = [to_device(stacked[ln]) for ln, _ in launches]
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
    print(f"{name} {'chained, handle' if chained else 'grouped, group'} queue_pct={queue_pct}: "
          f"{ms * 1e3:.2f} us {step_bytes / (ms * 1e-3) / 1e9:.0f} GB/s", flush=True)
    del g, Ws


for q in [int(v) for v in os.environ.get("QG", "20,25,30,35").split(",")]:
    run(queue_pct=q)
for q in [int(v) for v in os.environ.get("QC", "5,15,30").split(",")]:
    run(queue_pct=q, chained=True)
