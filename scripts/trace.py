"""Per-CTA timeline of one tiled-kernel launch (tuning aid; needs ECSR_B200_DEBUG=4)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_12205_b200 import _lib  # noqa: E402
from paper_2507_12205_b200.container import load_container  # noqa: E402
from paper_2507_12205_b200.device import spmv, to_device  # noqa: E402

NAMES = ["start", "pdl_wait", "x_staged", "tile0", "loop_done", "prod_done", "last_warp", "first_warp"]


def main():
    ec = load_container(sys.argv[1])
    mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
    W = to_device(ec)
    x = torch.randn(ec.num_cols, device="cuda").half()
    y = torch.zeros(ec.num_rows, device="cuda")
    for _ in range(5):
        spmv(W, x, y=y, accumulate=(mode == "acc"))
    torch.cuda.synchronize()
    grid = W.bytes()["grid"]
    out = np.zeros(16 * grid, dtype=np.uint64)
    fn = _lib.lib().ecsr_b200_debug_trace
    fn.restype = ctypes.c_int32
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    _lib.check(fn(W.handle, out.ctypes.data, out.size), "trace")
    t = out.reshape(grid, 16).astype(np.int64)
    t0 = t[:, 0].min()
    print(f"grid {grid}; times in us relative to first CTA start")
    for i, n in enumerate(NAMES):
        v = (t[:, i] - t0) / 1e3
        print(f"  {n:11s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")
    w = t[:, 8] / 16 / 1.9e3
    k = t[:, 9] / 16 / 1.9e3
    print(f"  per-warp wait us: med {np.median(w):.2f} max {w.max():.2f}; work us: med {np.median(k):.2f} "
          f"max {k.max():.2f}; work-tiles/warp med {np.median(t[:, 10] / 16):.1f}; tiles/CTA {np.median(t[:, 11] / 16):.1f}")
    print(f"  records/CTA (from tiles) n/a; work cycles per CTA-sum med {np.median(t[:, 9]):.0f}")
    n = t[:, 15] % 1000000
    ch = t[:, 15] // 1000000
    ok = n > 0
    print(f"  per pair (cycles): header {np.sum(t[ok, 12]) / n[ok].sum():.0f}  loop {np.sum(t[ok, 13]) / n[ok].sum():.0f}"
          f" (chunk-steps/pair {ch[ok].sum() / n[ok].sum():.2f})  reduce+emit {np.sum(t[ok, 14]) / n[ok].sum():.0f}; pairs/CTA {np.median(n):.0f}")
    if os.environ.get("TRACE_PER_CTA"):
        ld = (t[:, 4] - t0) / 1e3
        for c0 in range(0, grid, 8):
            print("   cta", c0, " ".join(f"{v:5.2f}" for v in ld[c0:c0 + 8]), " tiles", t[c0:c0 + 8, 11] // 16)
    hot = np.argsort(-t[:, 9])[:5]
    print("  slowest CTAs (work us):", [(int(c), round(float(k[c]), 2)) for c in hot])


if __name__ == "__main__":
    main()
