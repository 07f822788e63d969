"""Quick kernel probe: pack a .ecsr blob, time the tiled kernel over rotating copies (> 2x L2)."""
import json
import sys
import os
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2507_12205_b200.container import load_container, kernel_model_bytes
from paper_2507_12205_b200.device import spmv, to_device


def main():
    path = sys.argv[1]
    ncopy = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    t0 = time.time()
    ec = load_container(path)
    Ws = [to_device(ec) for _ in range(ncopy)]
    print("pack s", time.time() - t0, Ws[0].bytes())
    mb = kernel_model_bytes(ec)
    x = torch.randn(ec.num_cols, device="cuda").half()
    ys = [torch.empty(ec.num_rows, device="cuda") for _ in range(ncopy)]
    for ordered in (False, True):
        for _ in range(3):
            for i in range(ncopy):
                spmv(Ws[i], x, y=ys[i], ordered=ordered)
        torch.cuda.synchronize()
        # graph of ncopy launches
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            spmv(Ws[0], x, y=ys[0], ordered=ordered)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(ncopy):
                spmv(Ws[i], x, y=ys[i], ordered=ordered)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * ncopy)
        print(json.dumps({"ordered": ordered, "us_per_spmv": round(us, 3),
                          "model_GBps": round(mb / us / 1e3, 1), "model_bytes": mb}))


if __name__ == "__main__":
    main()
