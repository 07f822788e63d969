"""Time the peer exchange alone at world 1 (bench-sized segments) with a given build."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_12205_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

from paper_2507_12205_b200.exchange import PeerExchange  # noqa: E402

rows = [12288, 4096, 22016, 4096]
segs, o = [], 0
for r in rows:  # one matrix set per launch, offsets not 16-B aligned like real shards
    segs.append((o + 1, o + 1, r))
    o += r
src = torch.randn(o + 8, device="cuda")
ex = PeerExchange(o + 8, 0, 1)
ex.plan(segs)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        ex.run(src, s)
torch.cuda.synchronize()
assert torch.equal(ex.y[1:o + 1], src[1:o + 1])
for n in (1, 20):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            ex.run(src, s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    with torch.cuda.stream(s):
        for _ in range(10):
            g.replay()
    b.record(s)
    torch.cuda.synchronize()
    print(os.path.basename(sys.argv[1] if len(sys.argv) > 1 else "product"),
          f"{n} exchanges per graph: {a.elapsed_time(b) / 10 / n * 1e3:.2f} us per exchange", flush=True)
