"""Fit the packer's per-record cost model from measured per-CTA times (tuning aid).

For each bench launch kind: trace one launch (ECSR_B200_DEBUG=4) and read each CTA's
static work features (records and block-chunk steps per g class, bytes); fit
  t_cta(work) = sum_g a_g * records_g + b_g * steps_g + c * bytes
by least squares on (end - x_ready). Prints the coefficients in cycles at 1.965 GHz.
"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2507_12205_b200 import _lib
from paper_2507_12205_b200.device import spmv, to_device, vstack

lib = _lib.lib()
for name in ("ecsr_b200_debug_trace", "ecsr_b200_debug_ctafeat"):
    getattr(lib, name).restype = ctypes.c_int32
    getattr(lib, name).argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
ecs, _ = bench.load_workload()
X, Y = [], []
for ln, names in bench.LAUNCHES:
    W = to_device(vstack([ecs[n] for n in names]))
    x = torch.randn(W.num_cols, device="cuda").half()
    y = torch.empty(W.num_rows, device="cuda")
    for _ in range(5):
        spmv(W, x, y=y)
    torch.cuda.synchronize()
    grid = W.bytes()["grid"]
    tr = np.zeros(16 * grid, np.uint64)
    _lib.check(lib.ecsr_b200_debug_trace(W.handle, tr.ctypes.data, tr.size), "trace")
    ft = np.zeros(9 * grid)
    _lib.check(lib.ecsr_b200_debug_ctafeat(W.handle, ft.ctypes.data, ft.size), "feat")
    t = tr.reshape(grid, 16).astype(np.int64)
    work = (t[:, 6] - t[:, 2]) / 1e3 * 1965.0  # cycles from x ready to the CTA's last warp
    X.append(ft.reshape(grid, 9))
    Y.append(work)
    if os.environ.get("ECSR_CAL_DUMP"):
        np.savez(os.path.join(os.environ["ECSR_CAL_DUMP"], f"cal_{ln}.npz"), trace=t, feat=ft.reshape(grid, 9))
    print(ln, "CTA work cycles: min %.0f med %.0f max %.0f" % (work.min(), np.median(work), work.max()))
X = np.concatenate(X)
Y = np.concatenate(Y)
coef, *_ = np.linalg.lstsq(X, Y, rcond=None)
names = ["rec_g1", "steps_g1", "rec_g2", "steps_g2", "rec_g4", "steps_g4", "rec_g8", "steps_g8", "bytes"]
for n, c in zip(names, coef):
    print(f"  {n:9s} {c:10.3f} cycles")
pred = X @ coef
print("fit rel err: med %.3f max %.3f" % (np.median(np.abs(pred - Y) / Y), np.max(np.abs(pred - Y) / Y)))
