"""Timeline of one whole bench step (qkv, o, gate_up, down launched back to back, PDL
chained, no syncs): per launch, CTA start / x ready / first tile / producer done / last
warp end relative to the step's first CTA start. Run with ECSR_B200_DEBUG=12 (trace,
caller-reset)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2507_12205_b200 import _lib
from paper_2507_12205_b200.device import spmv, to_device, vstack

lib = _lib.lib()
lib.ecsr_b200_debug_trace.restype = ctypes.c_int32
lib.ecsr_b200_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
lib.ecsr_b200_debug_trace_reset.restype = ctypes.c_int32
lib.ecsr_b200_debug_trace_reset.argtypes = [ctypes.c_void_p]
LAUNCHES = bench.WORKLOADS[bench.HEADLINE]["launches"]
ecs, _ = bench.load_workload(bench.HEADLINE)
Ws, xs, ys = {}, {}, {}
for ln, names in LAUNCHES:
    Ws[ln] = to_device(vstack([ecs[n] for n in names]), queue_pct=QPCT)
    xs[ln] = torch.randn(Ws[ln].num_cols, device="cuda").half()
    ys[ln] = torch.empty(Ws[ln].num_rows, device="cuda")
for _ in range(3):
    for ln, _ in LAUNCHES:
        spmv(Ws[ln], xs[ln], y=ys[ln])
torch.cuda.synchronize()
stream = torch.cuda.Stream()
graph = torch.cuda.CUDAGraph()  # the step as the bench runs it: no host in the loop
with torch.cuda.graph(graph, stream=stream):
    for ln, _ in LAUNCHES:
        spmv(Ws[ln], xs[ln], y=ys[ln], stream=stream)
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for rep in range(3):
    for ln in Ws:
        _lib.check(lib.ecsr_b200_debug_trace_reset(Ws[ln].handle), "reset")
    with torch.cuda.stream(stream):
        flush.zero_()
        graph.replay()
    torch.cuda.synchronize()
    tr = {}
    for ln in Ws:
        g = Ws[ln].bytes()["grid"]
        out = np.zeros(16 * g, np.uint64)
        _lib.check(lib.ecsr_b200_debug_trace(Ws[ln].handle, out.ctypes.data, out.size), "trace")
        tr[ln] = out.reshape(g, 16).astype(np.int64)
    t0 = min(t[:, 0].min() for t in tr.values())
    np.savez(os.path.join(ROOT, "gpurun_out", f"step_trace_q{QPCT}_{rep}.npz"), **tr)
    print(f"rep {rep}: times in us from the step's first CTA start")
    for ln, t in tr.items():
        f = lambda i: (t[:, i] - t0) / 1e3
        mb = Ws[ln].bytes()["device_arena_bytes"] / 1e6
        print(f"  {ln:8s} {mb:6.1f} MB start {f(0).min():6.2f}..{f(0).max():6.2f}  pdl {np.median(f(1)):6.2f} "
              f" x_ready {np.median(f(2)):6.2f} (max {f(2).max():6.2f})  "
              f"prod_done {np.median(f(5)):6.2f}  end {np.percentile(f(6), 10):6.2f} / {np.median(f(6)):6.2f} / {f(6).max():6.2f}")
