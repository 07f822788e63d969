"""Tail-queue share sweep on the bench layer: step time (graph of 5 layers) and the
isolated o-launch latency per queue_pct (pack option ECSR_PACK_QUEUE_PCT)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2507_12205_b200 import _lib

args = sys.argv[1:]
tag = "product"
if args and args[0] == "--lib":  # A/B against another build (e.g. build/libhead.so)
    _lib.LIB_PATH, tag, args = os.path.abspath(args[1]), os.path.basename(args[1]), args[2:]
from paper_2507_12205_b200.device import spmv, to_device, vstack

pcts = [int(a) for a in args] or [0, 10, 20, 30, 50]
ecs, _ = bench.load_workload(bench.HEADLINE)
launches = bench.LAUNCHES
stacked = {ln: vstack([ecs[n] for n in names]) for ln, names in launches}
xs16 = bench.launch_inputs(bench.HEADLINE)
xs = {ln: torch.from_numpy(xs16[ln]).cuda() for ln, _ in launches}
step_bytes = sum(bench.model_bytes(e) for e in ecs.values())
stream = torch.cuda.Stream()
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
for pct in pcts:
    Ws = {ln: to_device(stacked[ln], queue_pct=pct) for ln, _ in launches}
    ys = {ln: torch.empty(Ws[ln].num_rows, device="cuda") for ln, _ in launches}
    def step():
        for ln, _ in launches:
            spmv(Ws[ln], xs[ln], y=ys[ln], stream=stream)
    with torch.cuda.stream(stream):
        step(); step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(5):
            step()
    res = []
    for rep in range(3):
        ms, _ = bench.time_graph(g, 10, 2, stream)
        res.append(ms / 5)
    lat = {}
    for ln, _ in launches:
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, stream=stream):
            spmv(Ws[ln], xs[ln], y=ys[ln], stream=stream)
        m, _ = bench.time_graph(g1, 20, 3, stream, flush=flush)
        lat[ln] = round(m * 1e3, 2)
    q = {ln: Ws[ln].bytes().get("queue_tiles") if tag == "product" else None for ln in Ws}
    t = {ln: Ws[ln].bytes()["tiles"] for ln in Ws}
    ms = min(res)
    print(json.dumps({"lib": tag, "queue_pct": pct, "step_us": round(ms * 1e3, 2), "reps_us": [round(r * 1e3, 2) for r in res],
                      "GBps": round(step_bytes / (ms * 1e-3) / 1e9, 1), "lat_us": lat, "queue_tiles": q, "tiles": t}), flush=True)
    del Ws, g
    torch.cuda.synchronize()
