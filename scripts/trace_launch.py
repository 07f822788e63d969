"""CTA timeline of one bench launch kind (ECSR_B200_DEBUG=4): start / x ready / end spread."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2507_12205_b200 import _lib
from paper_2507_12205_b200.device import spmv, to_device, vstack

ecs, _ = bench.load_workload()
ln = sys.argv[1] if len(sys.argv) > 1 else "gate_up"
names = dict(bench.LAUNCHES)[ln]
W = to_device(vstack([ecs[n] for n in names]))
x = torch.randn(W.num_cols, device="cuda").half()
y = torch.empty(W.num_rows, device="cuda")
for _ in range(5):
    spmv(W, x, y=y)
torch.cuda.synchronize()
grid = W.bytes()["grid"]
out = np.zeros(16 * grid, dtype=np.uint64)
fn = _lib.lib().ecsr_b200_debug_trace
fn.restype = ctypes.c_int32
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
_lib.check(fn(W.handle, out.ctypes.data, out.size), "trace")
t = out.reshape(grid, 16).astype(np.int64)
t0 = t[:, 0].min()
for i, n in [(0, "start"), (2, "x_ready"), (5, "prod_done"), (6, "last_warp_end")]:
    v = (t[:, i] - t0) / 1e3
    print(f"{ln} {n:14s} min {v.min():7.2f} p10 {np.percentile(v,10):7.2f} med {np.median(v):7.2f} p90 {np.percentile(v,90):7.2f} max {v.max():7.2f} us")
end = (t[:, 6] - t0) / 1e3
print("CTA end by index (8 per row):")
for c in range(0, grid, 16):
    print("  ", " ".join(f"{e:5.1f}" for e in end[c:c + 16]))

sm = t[:, 12]
per_sm = {}
for c in range(grid):
    per_sm.setdefault(int(sm[c]), []).append(end[c])
sms = sorted(per_sm)
sm_end = np.array([max(per_sm[s]) for s in sms])
print("SM end (max over its CTAs) by smid (16 per row):")
for i in range(0, len(sms), 16):
    print("  ", " ".join(f"{sm_end[j]:5.1f}" for j in range(i, min(i + 16, len(sms)))))
# does the slowness follow the SM or the work? correlate with per-CTA tile count
nt = t[:, 11]
print("corr(end, ntiles) =", float(np.corrcoef(end, nt)[0, 1]))
if t[:, 10].sum() > 0:  # ECSR_TRACE_CYCLES build: consumer wait vs work cycles
    wait, work, nrec = t[:, 8].sum(), t[:, 9].sum(), t[:, 10].sum()
    print(f"consumer cycles: wait {wait / (wait + work):.1%} of wait+work; "
          f"work per record {work / nrec:.0f}, wait per record {wait / nrec:.0f} cycles "
          f"(tile not yet issued: {t[:, 13].sum() / nrec:.0f}); records {nrec}")
