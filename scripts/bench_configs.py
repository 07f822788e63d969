"""Per-config SpMV measurements for BASELINE.json configs 1-5 (writes one JSON line each).

    python scripts/bench_configs.py [--out profiles/round1/configs.jsonl] [--only 1,3]

Inputs: seeded synthetic matrices (magnitude-pruned N(0, 1/K) or planted blocks),
encoded by the native encoder (byte-identical to the reference convert_csr). For each
matrix: `stream_us` = average device time per SpMV when launched back to back (CUDA
graph over rotating copies whose total exceeds 2x L2, as in a layer sequence),
`single_us` = one launch after a 256 MB L2 flush, GB/s = model bytes / time (stream:
mean of 40 back-to-back graph replays; p10/p50/p90 from a second pass with an event
between replays, which costs them their overlap), frac vs
the 6.65 TB/s fallback HBM peak. Parity: fast-mode y vs the C oracle on fp16-rounded
inputs (rel-inf). Config 5 reports the per-GPU shard SpMV of an N-way row split
(the NCCL all-gather needs more than the one GPU available here).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2507_12205_b200.container import kernel_model_bytes  # noqa: E402
from paper_2507_12205_b200.device import spmv, to_device  # noqa: E402
from paper_2507_12205_b200.encoder import convert_csr  # noqa: E402
from paper_2507_12205_b200.generators import make_matrix  # noqa: E402
from paper_2507_12205_b200.sharded import row_slice, shard_bounds  # noqa: E402

PEAK = 6650.0
L2 = 126 << 20

CONFIGS = {
    1: [("4096x4096@50%", "magnitude", 4096, 4096, 0.5, 1, None)],
    2: [(f"{n}@{int(s * 100)}%", "magnitude", m, k, s, 200 + i, None)
        for s in (0.5, 0.6, 0.7)
        for i, (n, m, k) in enumerate((("q 4096x4096", 4096, 4096), ("up 11008x4096", 11008, 4096),
                                       ("down 4096x11008", 4096, 11008)))],
    3: [("13B-q 5120x5120 planted@50%", "planted", 5120, 5120, 0.5, 301, None),
        ("13B-up 13824x5120 planted@50%", "planted", 13824, 5120, 0.5, 302, None),
        ("13B-q 5120x5120 planted@70%", "planted", 5120, 5120, 0.7, 303, None)],
    4: [("OPT30B-q 7168x7168@70%", "magnitude", 7168, 7168, 0.7, 401, None),
        ("OPT30B-fc1 28672x7168@70%", "magnitude", 28672, 7168, 0.7, 402, None),
        ("OPT30B-fc2 7168x28672@70%", "magnitude", 7168, 28672, 0.7, 403, None)],
    5: [(f"70B-{n} shard 0/{p}", "magnitude", m, 8192, 0.5, 500 + j, p)
        for j, (n, m) in enumerate((("q 8192x8192", 8192), ("up 28672x8192", 28672)))
        for p in (1, 2, 4, 8)],
}


def time_graph(fn, reps):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        # per-replay spread from a second pass with an event between replays (the events
        # cost the replays their back-to-back overlap, so the mean comes from the first)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        ev[0].record(s)
        for i in range(reps):
            g.replay()
            ev[i + 1].record(s)
    torch.cuda.synchronize()
    per = np.array([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(reps)])
    time_graph.spread = (float(np.percentile(per, 10)), float(np.median(per)), float(np.percentile(per, 90)))
    return e0.elapsed_time(e1) * 1e3 / reps


def measure(label, kind, m, k, s, seed, shards):
    t0 = time.time()
    a = make_matrix(kind, m, k, s, seed, dtype=np.float32)
    if shards:
        b = shard_bounds(a.row_ptr, shards)
        a = row_slice(a, b[0], b[1])
    ec = convert_csr(a)
    enc_s = time.time() - t0
    mb = kernel_model_bytes(ec)
    ncopy = max(1, int(np.ceil(2.2 * L2 / mb)))
    Ws = [to_device(ec) for _ in range(ncopy)]
    x = np.random.default_rng(seed).uniform(-1, 1, k).astype(np.float16)
    xd = torch.from_numpy(x).cuda()
    ys = [torch.empty(ec.num_rows, device="cuda") for _ in range(ncopy)]
    y = spmv(Ws[0], xd, y=ys[0]).cpu().numpy()
    ref = oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32), x.astype(np.float32), np.float32)
    rel = float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))
    stream_us = time_graph(lambda: [spmv(Ws[i], xd, y=ys[i]) for i in range(ncopy)], 40) / ncopy
    p10, p50, p90 = (v / ncopy for v in time_graph.spread)
    flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
    singles = []
    for _ in range(10):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        spmv(Ws[0], xd, y=ys[0])
        e1.record()
        torch.cuda.synchronize()
        singles.append(e0.elapsed_time(e1) * 1e3)
    single_us = float(np.median(singles))
    return {"matrix": label, "rows": ec.num_rows, "cols": k, "nnz": ec.nnz,
            "shards": shards, "model_bytes": mb, "layout": Ws[0].layout,
            "stream_us": round(stream_us, 2), "stream_us_p10_p50_p90": [round(p10, 2), round(p50, 2), round(p90, 2)],
            "stream_GBps": round(mb / stream_us / 1e3, 1),
            "stream_frac": round(mb / stream_us / 1e3 / PEAK, 3),
            "single_us": round(single_us, 2), "single_GBps": round(mb / single_us / 1e3, 1),
            "parity_rel_inf": rel, "encode_s": round(enc_s, 1),
            "sets": [(st.granularity, st.vector_size, st.num_blocks) for st in ec.sets]}


def measure_sequence():
    """Config 4 as a decoder-layer sequence: q|k|v row-stacked into
    one launch sharing x, then o, fc1, fc2, PDL-chained in one CUDA graph; per-layer
    time over a > L2 working set (one layer is ~590 MB)."""
    from paper_2507_12205_b200.device import vstack

    t0 = time.time()
    mats = {}
    for name, m, k, seed in (("q", 7168, 7168, 401), ("k", 7168, 7168, 404), ("v", 7168, 7168, 405),
                             ("o", 7168, 7168, 406), ("fc1", 28672, 7168, 402), ("fc2", 7168, 28672, 403)):
        mats[name] = convert_csr(make_matrix("magnitude", m, k, 0.7, seed, dtype=np.float32))
    enc_s = time.time() - t0
    launches = [("qkv", ["q", "k", "v"]), ("o", ["o"]), ("fc1", ["fc1"]), ("fc2", ["fc2"])]
    ecs = {ln: vstack([mats[n] for n in names]) for ln, names in launches}
    Ws = {ln: to_device(ec) for ln, ec in ecs.items()}
    mb = sum(kernel_model_bytes(ec) for ec in ecs.values())
    xs, ys, rel = {}, {}, 0.0
    for i, (ln, _) in enumerate(launches):
        x = np.random.default_rng(4000 + i).uniform(-1, 1, ecs[ln].num_cols).astype(np.float16)
        xs[ln] = torch.from_numpy(x).cuda()
        ys[ln] = torch.empty(ecs[ln].num_rows, device="cuda")
        y = spmv(Ws[ln], xs[ln], y=ys[ln]).cpu().numpy()
        ref = oracle.spmv_ec_oracle(ecs[ln].astype(np.float16).astype(np.float32), x.astype(np.float32),
                                    np.float32)
        rel = max(rel, float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30)))
    layer_us = time_graph(lambda: [spmv(Ws[ln], xs[ln], y=ys[ln]) for ln, _ in launches], 200)
    return {"matrix": "OPT30B decoder layer @70% (q|k|v, o, fc1, fc2 in one graph)", "model_bytes": mb,
            "layer_us": round(layer_us, 2), "stream_us": round(layer_us, 2),
            "stream_us_p10_p50_p90": [round(v, 2) for v in time_graph.spread],
            "stream_GBps": round(mb / layer_us / 1e3, 1), "stream_frac": round(mb / layer_us / 1e3 / PEAK, 3),
            "target_us_70pct": round(mb / (0.7 * PEAK) / 1e3, 1), "parity_rel_inf": rel,
            "encode_s": round(enc_s, 1), "launches": [ln for ln, _ in launches]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.jsonl"))
    ap.add_argument("--only", default="1,2,3,4,5")
    args = ap.parse_args()
    with open(args.out, "w") as fh:
        for c in [int(v) for v in args.only.split(",")]:
            cases = [lambda case=case: measure(*case) for case in CONFIGS[c]]
            if c == 4:
                cases.append(measure_sequence)
            for run in cases:
                r = run()
                r["config"] = c
                line = json.dumps(r)
                print(line, flush=True)
                fh.write(line + "\n")
                fh.flush()


if __name__ == "__main__":
    main()
