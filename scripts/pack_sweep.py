"""Grouped-step time vs packing knobs (tuning build): tile size (ECSR_B200_TILE bytes)
and the average-record cap (ECSR_B200_RECCAP bytes). Encodes once.

    python scripts/pack_sweep.py build/libNAME.so [workload]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_12205_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_12205_b200.device import SpmvGroup, to_device, vstack  # noqa: E402

name = sys.argv[2] if len(sys.argv) > 2 else bench.HEADLINE
ecs, _ = bench.load_workload(name)
launches = bench.WORKLOADS[name]["launches"]
stacked = [vstack([ecs[n] for n in names]) for _, names in launches]
step_bytes = sum(bench.model_bytes(e) for e in ecs.values())
stream = torch.cuda.Stream()
xs = [torch.randn(e.num_cols, device="cuda").half() for e in stacked]
ys = [torch.empty(e.num_rows, device="cuda") for e in stacked]


def run(env):
    for k in ("ECSR_B200_TILE", "ECSR_B200_RECCAP", "ECSR_B200_RECMAX"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    Ws = [to_device(e) for e in stacked]
    g = SpmvGroup(Ws)
    with torch.cuda.stream(stream):
        for _ in range(3):
            g.spmv(xs, ys, stream=stream)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=stream):
        for _ in range(5):
            g.spmv(xs, ys, stream=stream)
    ms, _ = bench.time_graph(gr, 20, 3, stream)
    ms /= 5
    b = Ws[0].bytes()
    print(f"{name} {env or 'default'}: {ms * 1e3:.2f} us {step_bytes / (ms * 1e-3) / 1e9:.0f} GB/s "
          f"(stage {b['stage_bytes']} x {b['stages']})", flush=True)


run({})
for env in [{"ECSR_B200_TILE": 11000, "ECSR_B200_RECCAP": 8600, "ECSR_B200_RECMAX": 11000},
            {"ECSR_B200_TILE": 13000, "ECSR_B200_RECCAP": 8600, "ECSR_B200_RECMAX": 13000},
            {"ECSR_B200_TILE": 8600, "ECSR_B200_RECCAP": 8600, "ECSR_B200_RECMAX": 8600},
            {"ECSR_B200_TILE": 12500, "ECSR_B200_RECCAP": 6000, "ECSR_B200_RECMAX": 12500},
            {"ECSR_B200_TILE": 20500}]:
    run(env)
run({})
