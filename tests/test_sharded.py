"""Row-sharded SpMV host logic on CPU, world_size 2 over gloo.

Each rank encodes its row shard (shard-first, native encoder), computes its y rows
with the CPU oracle, and one all-gather assembles y; the result must equal the
single-matrix product. The GPU/NCCL variant of the same code path runs in bench.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_12205_b200.encoder import convert_csr
from paper_2507_12205_b200.generators import make_matrix
from paper_2507_12205_b200.sharded import plan_shards, row_slice, shard_bounds


def test_shard_bounds_balance_nonzeros():
    a = make_matrix("uniform", 300, 200, 0.5, 3)
    # skew: make the first rows much denser
    rp = a.row_ptr.copy()
    b = shard_bounds(rp, 4)
    assert b[0] == 0 and b[-1] == 300 and all(x <= y for x, y in zip(b, b[1:]))
    counts = [rp[b[i + 1]] - rp[b[i]] for i in range(4)]
    assert max(counts) - min(counts) <= 2 * int(np.max(np.diff(rp)))
    assert shard_bounds(np.array([0, 5, 5, 5]), 2) in ([0, 1, 3], [0, 0, 3], [0, 1, 3])


def test_shard_bounds_uniform_rows_split_evenly():
    rp = np.arange(0, 8193, dtype=np.int64) * 10
    assert shard_bounds(rp, 8) == [i * 1024 for i in range(9)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mats = [make_matrix("planted", 256, 192, 0.5, 21, dtype=np.float32),
            make_matrix("magnitude", 160, 192, 0.6, 22, dtype=np.float32)]
    plan = plan_shards(mats, ["a", "b"], world)
    x = np.random.default_rng(7).uniform(-1, 1, 192).astype(np.float16).astype(np.float32)
    local = []
    for m, b in zip(mats, plan.bounds):
        ec = convert_csr(row_slice(m, b[rank], b[rank + 1]))
        ec16 = ec.astype(np.float16).astype(np.float32)
        local.append(oracle.spmv_ec_oracle(ec16, x, np.float32))
    buf = np.zeros(plan.max_rows(), np.float32)
    cat = np.concatenate(local)
    buf[:cat.size] = cat
    gathered = [torch.zeros(plan.max_rows()) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(buf))
    ys = plan.assemble(torch.stack(gathered).numpy())
    if rank == 0:
        res = []
        for m, y in zip(mats, ys):
            full = convert_csr(m).astype(np.float16).astype(np.float32)
            ref = oracle.spmv_ec_oracle(full, x, np.float32)
            res.append(float(np.max(np.abs(y - ref)) / np.max(np.abs(ref))))
        out.put(res)
    dist.destroy_process_group()


def test_row_sharded_spmv_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    out = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    errs = out.get()
    # shard encodings differ from the whole-matrix one (pairings are shard-local), so y
    # agrees up to fp32 summation order only
    assert all(e <= 1e-5 for e in errs), errs
