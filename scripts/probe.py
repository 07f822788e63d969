"""Kernel probe (tuning aid): pack a .ecsr blob, time the SpMV over rotating copies (> 2x L2)
with CUDA-graph replay. Env knobs of libecsr_b200 (ECSR_B200_TILE / ECSR_B200_DEBUG) apply."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2507_12205_b200.container import kernel_model_bytes, load_container  # noqa: E402
from paper_2507_12205_b200.device import spmv, to_device  # noqa: E402


def timed_graph(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    path = sys.argv[1]
    ncopy = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["fast", "ordered"]
    t0 = time.time()
    ec = load_container(path)
    Ws = [to_device(ec) for _ in range(ncopy)]
    info = Ws[0].bytes()
    mb = kernel_model_bytes(ec)
    x = torch.randn(ec.num_cols, device="cuda").half()
    ys = [torch.zeros(ec.num_rows, device="cuda") for _ in range(ncopy)]
    res = {"env": {k: v for k, v in os.environ.items() if k.startswith("ECSR_B200")},
           "pack_s": round(time.time() - t0, 2), "tiles": info["tiles"],
           "stages": info["stages"], "stage_bytes": info["stage_bytes"], "model_bytes": mb}
    for mode in modes:
        us = timed_graph(lambda: [spmv(Ws[i], x, y=ys[i], ordered=(mode == "ordered"),
                                       accumulate=(mode == "acc")) for i in range(ncopy)])
        res[mode] = {"us": round(us / ncopy, 3), "GBps": round(mb / (us / ncopy) / 1e3, 1)}
    if "copy" in modes:
        a = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
        b = torch.empty_like(a)
        us = timed_graph(lambda: b.copy_(a), reps=10)
        res["copy_GBps"] = round(2 * a.numel() * 4 / us / 1e3, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
