"""Where the end-to-end step loses time against the device-resident step (bench headline
workload, graphs of 5 steps): variants of the copy arrangement around the grouped launch.

  none      no copies (the device-resident headline step)
  y_out     every step's y -> pinned host on a copy stream (outgoing edge only)
  x_in      every step's x <- pinned host on a copy stream, the launch waits on it
  x_early   all steps' x copied up front into per-step buffers, launch i waits on copy i
  x_inline  the x copy on the launch stream itself, between the launches
  both      x_in + y_out (the copy-stream pipeline)
  io_x      x(i) in by the host-io kernel chained before launch i (device.host_io)
  io        x(i) in and y(i-2) out by the host-io kernel, the last two y by a tail one
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

SPG = 5
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
copy = torch.cuda.Stream(dev)
wl = bench.Workload(bench.HEADLINE, dev)
nbuf = SPG
x_dev = [wl.x_all] + [torch.empty_like(wl.x_all) for _ in range(nbuf - 1)]
y_dev = [wl.y_all] + [torch.empty_like(wl.y_all) for _ in range(nbuf - 1)]
y_host = [wl.y_host_all] + [torch.empty_like(wl.y_host_all).pin_memory() for _ in range(nbuf - 1)]


def views(buf, like, base):
    return [buf[(t.data_ptr() - base.data_ptr()) // t.element_size():][:t.numel()] for t in like]


x_lists = [views(x, wl.x_list, wl.x_all) for x in x_dev]
y_lists = [views(y, wl.y_list, wl.y_all) for y in y_dev]


def body(kind):
    if kind.startswith("io"):
        from paper_2507_12205_b200.device import host_io

        for i in range(SPG):
            b = i % 2
            pairs = [(wl.x_host_all, x_dev[b])]
            if kind == "io" and i >= 2:
                pairs.append((y_dev[b], y_host[b]))
            host_io(pairs, stream)
            wl.group.spmv(x_lists[b], y_lists[b], stream=stream)
        if kind == "io":
            host_io([(y_dev[(SPG - 2) % 2], y_host[(SPG - 2) % 2]), (y_dev[(SPG - 1) % 2], y_host[(SPG - 1) % 2])],
                    stream, after_predecessor=True)
        return
    start = torch.cuda.Event()
    start.record(stream)
    copy.wait_event(start)
    x_ev = []
    if kind == "x_early":
        with torch.cuda.stream(copy):
            for i in range(SPG):
                x_dev[i].copy_(wl.x_host_all, non_blocking=True)
                e = torch.cuda.Event()
                e.record(copy)
                x_ev.append(e)
    for i in range(SPG):
        b = i % 2 if kind != "x_early" else i
        if kind in ("x_in", "both"):
            with torch.cuda.stream(copy):
                x_dev[b].copy_(wl.x_host_all, non_blocking=True)
                e = torch.cuda.Event()
                e.record(copy)
            stream.wait_event(e)
        elif kind == "x_early":
            stream.wait_event(x_ev[i])
        elif kind == "x_inline":
            with torch.cuda.stream(stream):
                x_dev[b].copy_(wl.x_host_all, non_blocking=True)
        wl.group.spmv(x_lists[b], y_lists[b], stream=stream)
        if kind in ("y_out", "both"):
            e = torch.cuda.Event()
            e.record(stream)
            with torch.cuda.stream(copy):
                copy.wait_event(e)
                y_host[b].copy_(y_dev[b], non_blocking=True)
    done = torch.cuda.Event()
    done.record(copy)
    stream.wait_event(done)


for rep in range(2):
    for kind in ("none", "y_out", "x_in", "x_early", "x_inline", "both", "io_x", "io"):
        with torch.cuda.stream(stream):
            body(kind)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            body(kind)
        ms, _ = bench.time_graph(g, 40, 5, stream)
        print(f"{kind:9s} {ms / SPG * 1e3:6.2f} us/step", flush=True)

# the io pipeline really moved the bytes
for b in range(2):
    assert torch.equal(x_dev[b].cpu(), wl.x_host_all), "x not copied in"
    assert torch.equal(y_host[b], y_dev[b].cpu()), "y not copied out"
print("io copies verified", flush=True)
