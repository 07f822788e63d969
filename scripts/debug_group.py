"""One grouped launch of a bench workload (the bench step), checked against the oracle
-- the target of `ncu --set full -k regex:ecsr_tiled -c 1` (its first tiled launch)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
from paper_2507_12205_b200.device import SpmvGroup, to_device, vstack  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.HEADLINE
ecs, _ = bench.load_workload(name)
launches = bench.WORKLOADS[name]["launches"]
stacked = [vstack([ecs[n] for n in names]) for _, names in launches]
g = SpmvGroup([to_device(e) for e in stacked])
rng = np.random.default_rng(1)
xs = [rng.uniform(-1, 1, e.num_cols) for e in stacked]
ys = g.spmv([torch.from_numpy(x.astype(np.float16)).cuda() for x in xs])
torch.cuda.synchronize()
for (ln, _), e, x, y in zip(launches, stacked, xs, ys):
    ref = oracle.spmv_ec_oracle(e.astype(np.float16).astype(np.float32), x.astype(np.float16).astype(np.float32),
                                np.float32)
    err = float(np.max(np.abs(y.cpu().numpy() - ref)) / np.max(np.abs(ref)))
    print(ln, "rel-inf", err, flush=True)
    assert err <= 1e-5
print(g.info())
