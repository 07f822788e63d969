"""Record-size cap sweep (tuning aid): stream time of a few config shapes for several
ECSR_B200_RECCAP values (the packer reads it at every pack)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
from paper_2507_12205_b200.container import kernel_model_bytes
from paper_2507_12205_b200.device import spmv, to_device
from paper_2507_12205_b200.encoder import convert_csr
from paper_2507_12205_b200.generators import make_matrix
from probe import timed_graph

SHAPES = [("70B-up", 28672, 8192, 0.5, 501), ("70B-q", 8192, 8192, 0.5, 500), ("down", 4096, 11008, 0.5, 202),
          ("up@70", 11008, 4096, 0.7, 201)]
caps = [c for c in (sys.argv[1] if len(sys.argv) > 1 else "0,8192,12288,16384,24576").split(",")]
for name, m, k, s, seed in SHAPES:
    ec = convert_csr(make_matrix("magnitude", m, k, s, seed))
    mb = kernel_model_bytes(ec)
    x = torch.randn(k, device="cuda").half()
    for cap in caps:
        mean, _, hard = cap.partition("/")  # "mean[/hard]", 0 = default
        for key, val in (("ECSR_B200_RECCAP", mean), ("ECSR_B200_RECMAX", hard)):
            if val and val != "0":
                os.environ[key] = val
            else:
                os.environ.pop(key, None)
        n = max(2, int(2 * 126e6 / mb) + 1)
        Ws = [to_device(ec) for _ in range(n)]
        ys = [torch.zeros(m, device="cuda") for _ in range(n)]
        us = timed_graph(lambda: [spmv(Ws[i], x, y=ys[i]) for i in range(n)], reps=20) / n
        b = Ws[0].bytes()
        print(f"{name:7s} cap {cap:>12} stream {us:7.2f} us {mb / us / 1e3:7.1f} GB/s  stage {b['stage_bytes']} x {b['stages']}"
              f"  tiles {b['tiles']}", flush=True)
        del Ws, ys
        torch.cuda.empty_cache()
