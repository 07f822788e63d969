"""Workload for compute-sanitizer (racecheck / synccheck / memcheck / initcheck) of the
tiled kernel: small containers, every launch mode, checked against the oracle.

    compute-sanitizer --tool racecheck python scripts/sanitize.py

Covers: the smoke container (one tile per CTA), a 1024x4096 matrix packed with 1 KB
tiles (many tiles per CTA: the stage pool, the tile->stage map and the tail queue
wrap), the u32-base (K > 65535) variant, two streams sharing one handle, overwrite /
accumulate / ordered modes, a grouped launch (gated and memset overwrite), and the
host-io chain around it (ecsr_b200_host_io)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2507_12205_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:  # a tuning build (scripts/build_exp.sh) instead of the product library
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2507_12205_b200.container import deserialize  # noqa: E402
from paper_2507_12205_b200.device import spmv, to_device  # noqa: E402
from paper_2507_12205_b200.encoder import convert_csr  # noqa: E402
from paper_2507_12205_b200.generators import make_matrix  # noqa: E402


def ref16(ec, x):
    return oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32),
                                 x.astype(np.float16).astype(np.float32), np.float32)


def check(ec, W, x, label):
    xd = torch.from_numpy(x.astype(np.float16)).cuda()
    r = ref16(ec, x)
    y = spmv(W, xd, ordered=True).cpu().numpy()
    assert np.array_equal(y, r), label + ": ordered"
    yf = torch.empty(W.num_rows, device="cuda")
    for _ in range(3):
        spmv(W, xd, y=yf)
    e = np.max(np.abs(yf.cpu().numpy() - r)) / max(np.max(np.abs(r)), 1e-30)
    assert e <= 1e-5, (label, e)
    spmv(W, xd, y=yf, accumulate=True)
    e = np.max(np.abs(yf.cpu().numpy() - 2 * r)) / max(np.max(np.abs(r)), 1e-30)
    assert e <= 1e-5, (label, "accumulate", e)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ya, yb = torch.empty_like(yf), torch.empty_like(yf)
    torch.cuda.synchronize()
    for _ in range(2):
        spmv(W, xd, y=ya, stream=s1)
        spmv(W, xd, y=yb, stream=s2)
    torch.cuda.synchronize()
    for v in (ya, yb):
        e = np.max(np.abs(v.cpu().numpy() - r)) / max(np.max(np.abs(r)), 1e-30)
        assert e <= 1e-5, (label, "two streams", e)
    print(f"{label}: ok", flush=True)


z = np.load(os.path.join(ROOT, "tests", "golden", "planted_512x384_s0.5_b8_seed15.npz"))
ec = deserialize(z["blob"].tobytes())
check(ec, to_device(ec), z["x"], "smoke 512x384")
ec = convert_csr(make_matrix("magnitude", 1024, 4096, 0.5, 7, dtype=np.float32))
W = to_device(ec, tile_kb=1)
print("tiles", W.bytes()["tiles"], "grid", W.bytes()["grid"], "queue", W.bytes()["queue_tiles"])
check(ec, W, np.random.default_rng(1).uniform(-1, 1, 4096), "1024x4096 1 KB tiles")
ec = convert_csr(make_matrix("magnitude", 256, 70000, 0.995, 9, dtype=np.float32))
check(ec, to_device(ec), np.random.default_rng(2).uniform(-1, 1, 70000), "256x70000 wide bases")
# a grouped launch of three matrices (x of 8 KB and 22 KB side by side), gated and memset
from paper_2507_12205_b200.device import SpmvGroup  # noqa: E402

ecs = [convert_csr(make_matrix("magnitude", m, k, 0.5, 11 + i, dtype=np.float32))
       for i, (m, k) in enumerate([(512, 4096), (256, 4096), (256, 11008)])]
g = SpmvGroup([to_device(e) for e in ecs])
xs = [np.random.default_rng(3 + i).uniform(-1, 1, e.num_cols) for i, e in enumerate(ecs)]
xd = [torch.from_numpy(x.astype(np.float16)).cuda() for x in xs]
for memset_y in (False, True, False):
    ys = g.spmv(xd, memset_y=memset_y)
    for e, x, y in zip(ecs, xs, ys):
        r = ref16(e, x)
        err = np.max(np.abs(y.cpu().numpy() - r)) / max(np.max(np.abs(r)), 1e-30)
        assert err <= 1e-5, ("group", err)
print("group of 3: ok", flush=True)
# host-io chain: io(i) stages x(i) (pinned host -> device) and writes y(i-2) out while
# the previous grouped launch runs; the last two y after the last launch
from paper_2507_12205_b200.device import host_io  # noqa: E402

n = 4
xh = [torch.cat([torch.from_numpy(np.random.default_rng(20 + i).uniform(-1, 1, e.num_cols).astype(np.float16))
                 for e in ecs]).pin_memory() for i in range(n)]
kx = [e.num_cols for e in ecs]
xdev = [torch.zeros_like(xh[0], device="cuda") for _ in range(2)]
ydev = [torch.zeros(sum(e.num_rows for e in ecs), device="cuda") for _ in range(2)]
yh = [torch.zeros(ydev[0].numel()).pin_memory() for _ in range(n)]
xv = [list(torch.split(xdev[b], kx)) for b in range(2)]
yv = [list(torch.split(ydev[b], [e.num_rows for e in ecs])) for b in range(2)]
for i in range(n):
    b = i % 2
    host_io([(xh[i], xdev[b])] + ([(ydev[b], yh[i - 2])] if i >= 2 else []))
    g.spmv(xv[b], yv[b])
host_io([(ydev[(n - 2) % 2], yh[n - 2])])
host_io([(ydev[(n - 1) % 2], yh[n - 1])], after_predecessor=True)
torch.cuda.synchronize()
for i in range(n):
    got = torch.split(yh[i], [e.num_rows for e in ecs])
    for e, xs_i, y in zip(ecs, torch.split(xh[i], kx), got):
        r = ref16(e, xs_i.numpy().astype(np.float64))
        err = np.max(np.abs(y.numpy() - r)) / max(np.max(np.abs(r)), 1e-30)
        assert err <= 1e-5, ("host io", i, err)
print("host-io chain of 4: ok", flush=True)
print("sanitize workload done")
