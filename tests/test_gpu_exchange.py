"""The sharded step's y exchange over peer memory (ecsr_b200_xchg_*), on the B200:

* world 1 (one process): the exchange writes the rank's grouped-SpMV output into y_full
  at its final offsets;
* world 2 as two processes sharing the one GPU of the pool (CUDA IPC between processes
  works on one device as across NVLink): each rank runs its shards of two matrix sets in
  one grouped launch, then the exchange; after every step (eager and CUDA-graph
  replays) both ranks' y_full must equal the oracle of every shard, concatenated;
* a lagging peer: rank 1 reads each step's y_full ~20 ms late while rank 0 runs ahead;
  no push of a later step may land in it first (the exchange's ready handshake).
"""

import os
import socket

import numpy as np
import pytest

import oracle
from conftest import rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

SETS = [[("magnitude", 300, 512, 0.5, 71), ("planted", 260, 512, 0.5, 72)],
        [("magnitude", 200, 768, 0.6, 73)]]


def _step_inputs(world, rank):
    from paper_2507_12205_b200.device import SpmvGroup, to_device, vstack
    from paper_2507_12205_b200.encoder import convert_csr
    from paper_2507_12205_b200.exchange import shard_segments
    from paper_2507_12205_b200.generators import make_matrix
    from paper_2507_12205_b200.sharded import row_slice, shard_bounds

    bounds, shard_ecs, refs = [], [], []
    rng = np.random.default_rng(5)
    xs = [rng.uniform(-1, 1, mats[0][2]).astype(np.float16) for mats in SETS]
    for mats, x in zip(SETS, xs):
        bl, ecs, ref = [], [], []
        for kind, m, k, s, seed in mats:
            a = make_matrix(kind, m, k, s, seed, dtype=np.float32)
            b = shard_bounds(a.row_ptr, world)
            bl.append(b)
            ecs.append(convert_csr(row_slice(a, b[rank], b[rank + 1])))
            for r in range(world):  # every rank's shard, for the expected y_full
                e = convert_csr(row_slice(a, b[r], b[r + 1]))
                ref.append((b[r], oracle.spmv_ec_oracle(e.astype(np.float16).astype(np.float32),
                                                        x.astype(np.float32), np.float32)))
        bounds.append(bl)
        shard_ecs.append(ecs)
        full = []
        for b, (kind, m, k, s, seed) in zip(bl, mats):
            y = np.zeros(m, np.float32)
            full.append(y)
        # scatter each shard's reference rows
        i = 0
        for mi, b in enumerate(bl):
            for r in range(world):
                lo, yr = ref[i]
                full[mi][lo:lo + len(yr)] = yr
                i += 1
        refs.append(np.concatenate(full))
    Ws = [to_device(vstack(ecs)) for ecs in shard_ecs]
    group = SpmvGroup(Ws)
    slot = [sum(bb[-1] for bb in bl) for bl in bounds]  # generous slots: full rows
    slot_off = np.concatenate([[0], np.cumsum(slot)[:-1]]).tolist()
    y_off = slot_off
    segs = shard_segments(bounds, slot_off, y_off, rank)
    send = torch.zeros(sum(slot), dtype=torch.float32, device="cuda")
    ys = [send[o:o + W.num_rows] for o, W in zip(slot_off, Ws)]
    xd = [torch.from_numpy(x).cuda() for x in xs]
    return group, xd, ys, send, segs, np.concatenate(refs)


def test_exchange_world_one():
    from paper_2507_12205_b200.exchange import PeerExchange

    group, xd, ys, send, segs, ref = _step_inputs(1, 0)
    ex = PeerExchange(ref.size, 0, 1)
    ex.plan(segs)
    for _ in range(3):
        ex.y.fill_(float("nan"))
        group.spmv(xd, ys)
        y = ex.run(send).cpu().numpy()
        assert rel_err(y, ref) <= 1e-5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_12205_b200.exchange import PeerExchange

        torch.cuda.set_device(0)
        group, xd, ys, send, segs, ref = _step_inputs(world, rank)
        ex = PeerExchange(ref.size, rank, world)
        ex.plan(segs)
        errs = []
        stream = torch.cuda.Stream()
        for _ in range(3):
            with torch.cuda.stream(stream):
                group.spmv(xd, ys, stream=stream)
                ex.run(send, stream)
            stream.synchronize()
            errs.append(rel_err(ex.y.cpu().numpy(), ref))
            dist.barrier()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            group.spmv(xd, ys, stream=stream)
            ex.run(send, stream)
        for _ in range(3):
            with torch.cuda.stream(stream):
                g.replay()
            stream.synchronize()
            errs.append(rel_err(ex.y.cpu().numpy(), ref))
            dist.barrier()
        q.put((rank, errs))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_exchange_two_processes_one_gpu():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(2))
    for r in range(2):
        assert len(res[r]) == 6 and max(res[r]) <= 1e-5, res


def _lag_worker(rank, world, port, q, steps, n):
    """Rank 1 holds every step's y_full for ~20 ms (a device sleep) before reading it,
    while rank 0 races ahead with the next steps' pushes."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_12205_b200.exchange import PeerExchange

        torch.cuda.set_device(0)
        ex = PeerExchange(world * n, rank, world)
        ex.plan([(0, rank * n, n)])
        src = torch.empty(n, device="cuda")
        snaps = [torch.empty(world * n).pin_memory() for _ in range(steps)]
        stream = torch.cuda.Stream()
        dist.barrier()
        with torch.cuda.stream(stream):
            for s in range(steps):
                src.fill_(float(1000 * rank + s))
                ex.run(src, stream)
                if rank == 1:
                    torch.cuda._sleep(40_000_000)  # ~20 ms at ~2 GHz, on the stream
                snaps[s].copy_(ex.y, non_blocking=True)
        stream.synchronize()
        bad = []
        for s in range(steps):
            want = np.concatenate([np.full(n, 1000 * r + s, np.float32) for r in range(world)])
            if not np.array_equal(snaps[s].numpy(), want):
                bad.append(s)
        q.put((rank, bad))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_exchange_lagging_peer_keeps_its_y_full():
    """A push of step s+1 never lands in a y_full its owner still reads (step s)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_lag_worker, args=(r, 2, port, q, 5, 4096)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(2))
    assert res == {0: [], 1: []}, res
