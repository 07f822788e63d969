"""Run each bench launch alone with a sync and a parity check (debug aid)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2507_12205_b200.device import spmv, to_device, vstack
import oracle

ecs, _ = bench.load_workload()
only = sys.argv[1:] or [ln for ln, _ in bench.LAUNCHES]
for ln, names in bench.LAUNCHES:
    if ln not in only:
        continue
    ec = vstack([ecs[n] for n in names])
    W = to_device(ec)
    b = W.bytes()
    print(ln, "stage", b["stage_bytes"], "stages", b["stages"], "tiles", b["tiles"], flush=True)
    x = np.random.default_rng(1).uniform(-1, 1, ec.num_cols)
    y = spmv(W, torch.from_numpy(x.astype(np.float16)).cuda())
    torch.cuda.synchronize()
    ref = oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32),
                                x.astype(np.float16).astype(np.float32), np.float32)
    err = float(np.max(np.abs(y.cpu().numpy() - ref)) / np.max(np.abs(ref)))
    print(ln, "ok rel-inf", err, flush=True)
