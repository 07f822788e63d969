"""Host-io kernel (ecsr_b200_host_io, csrc/ecsr_hostio.cu): a step's host traffic in the
launch chain. Copies are checked byte for byte; the pipelined decode-style chain
(io(i): x(i) in, y(i-2) out -> grouped SpMV(i)) is checked step by step against the C
oracle of the reference kernel (pkg/src/ecsr/_speedups.pyx:81-129) on fp16-rounded
inputs, with a different x every step, so a copy that raced its neighbouring launch
would show up as a wrong y."""

import numpy as np
import pytest

import oracle
from conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2507_12205_b200 import _lib  # noqa: E402
from paper_2507_12205_b200.device import SpmvGroup, _IoSpan, host_io, to_device  # noqa: E402
from paper_2507_12205_b200.encoder import convert_csr  # noqa: E402
from paper_2507_12205_b200.generators import make_matrix  # noqa: E402


def _pinned(n, dtype=torch.float32, seed=0):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(n, generator=g).to(dtype).pin_memory()


def test_copies_every_direction():
    h_in = _pinned(4096, seed=1)
    d_in = torch.randn(1000, device="cuda")
    h_out = torch.zeros(1000).pin_memory()
    d_dst = torch.zeros(4096, device="cuda")
    d_src2 = torch.randn(36, device="cuda")
    d_dst2 = torch.zeros(36, device="cuda")
    host_io([(h_in, d_dst), (d_in, h_out), (d_src2, d_dst2)])
    torch.cuda.synchronize()
    assert torch.equal(d_dst.cpu(), h_in)
    assert torch.equal(h_out, d_in.cpu())
    assert torch.equal(d_dst2, d_src2)


def test_many_spans_and_large_span():
    hs = [_pinned(4 * (k + 1), seed=k) for k in range(16)]
    ds = [torch.zeros(4 * (k + 1), device="cuda") for k in range(16)]
    host_io(list(zip(hs, ds)))
    big_h = _pinned(3 << 20, torch.float16, seed=7)
    big_d = torch.zeros(3 << 20, dtype=torch.float16, device="cuda")
    host_io([(big_h, big_d)])
    torch.cuda.synchronize()
    for h, d in zip(hs, ds):
        assert torch.equal(d.cpu(), h)
    assert torch.equal(big_d.cpu(), big_h)


def test_ragged_byte_counts():
    """Spans need 16-B aligned starts, not 16-B multiples: odd fp16 lengths, a 3-float
    span, a 1-byte span."""
    pairs, outs = [], []
    for n, dt in [(4097, torch.float16), (3, torch.float32), (1, torch.uint8), (33, torch.float16)]:
        h = (torch.arange(n) % 251).to(dt).pin_memory()
        d = torch.zeros(n, dtype=dt, device="cuda")
        pairs.append((h, d))
        outs.append((h, d))
    back = torch.zeros(4097, dtype=torch.float16).pin_memory()
    host_io(pairs)
    host_io([(outs[0][1], back)], after_predecessor=True)
    torch.cuda.synchronize()
    for h, d in outs:
        assert torch.equal(d.cpu(), h)
    assert torch.equal(back, outs[0][0])


def test_empty_call_keeps_the_chain():
    host_io([])
    host_io([], after_predecessor=True)
    torch.cuda.synchronize()


def test_rejects_bad_spans():
    d = torch.zeros(64, device="cuda")
    with pytest.raises(ValueError, match="pinned"):
        host_io([(torch.zeros(64), d)])
    with pytest.raises(ValueError, match="bytes"):
        host_io([(torch.zeros(32).pin_memory(), d)])
    h = torch.zeros(68).pin_memory()
    with pytest.raises(ValueError, match="16-B aligned"):
        host_io([(h[1:65], d)])
    with pytest.raises(ValueError, match="entries"):
        host_io([(torch.zeros(4, device="cuda"), torch.zeros(4, device="cuda"))] * 17)
    # the C-ABI itself rejects pageable host memory (no UVA mapping)
    pageable = np.zeros(64, np.float32)
    span = (_IoSpan * 1)(_IoSpan(pageable.ctypes.data, d.data_ptr(), 256))
    rc = _lib.lib().ecsr_b200_host_io(span, 1, 0, None)
    assert rc == 2 and "pinned" in _lib.last_error()


def test_pipelined_decode_chain_in_a_graph():
    """n steps, each with its own x: io(i) stages x(i) into buffer i%2 and writes y(i-2)
    out while SpMV(i-1) runs; the last two y follow the last launch."""
    ecs = [convert_csr(make_matrix("magnitude", 2048, 1536, 0.5, 3, dtype=np.float32)),
           load_golden("uniform_256x256_s0.5_b8_seed11")["ec"]]
    Ws = [to_device(ec) for ec in ecs]
    g = SpmvGroup(Ws)
    n = 6
    rng = np.random.default_rng(9)
    kx = [ec.num_cols for ec in ecs]
    my = [ec.num_rows for ec in ecs]
    pad = lambda v: (v + 7) // 8 * 8  # noqa: E731
    xoff = np.cumsum([0] + [pad(k) for k in kx])
    yoff = np.cumsum([0] + [pad(m) for m in my])
    xs_host = [torch.zeros(int(xoff[-1]), dtype=torch.float16).pin_memory() for _ in range(n)]
    xs_np = []
    for i in range(n):
        xi = [rng.uniform(-1, 1, k).astype(np.float16) for k in kx]
        xs_np.append(xi)
        for j, v in enumerate(xi):
            xs_host[i][xoff[j]:xoff[j] + kx[j]] = torch.from_numpy(v)
    ys_host = [torch.full((int(yoff[-1]),), float("nan")).pin_memory() for _ in range(n)]
    x_dev = [torch.zeros(int(xoff[-1]), dtype=torch.float16, device="cuda") for _ in range(2)]
    y_dev = [torch.zeros(int(yoff[-1]), device="cuda") for _ in range(2)]
    xv = [[x_dev[b][xoff[j]:xoff[j] + kx[j]] for j in range(len(ecs))] for b in range(2)]
    yv = [[y_dev[b][yoff[j]:yoff[j] + my[j]] for j in range(len(ecs))] for b in range(2)]
    s = torch.cuda.Stream()

    def steps():
        for i in range(n):
            b = i % 2
            pairs = [(xs_host[i], x_dev[b])]
            if i >= 2:
                pairs.append((y_dev[b], ys_host[i - 2]))
            host_io(pairs, s)
            g.spmv(xv[b], yv[b], stream=s)
        host_io([(y_dev[(n - 2) % 2], ys_host[n - 2])], s)
        host_io([(y_dev[(n - 1) % 2], ys_host[n - 1])], s, after_predecessor=True)

    with torch.cuda.stream(s):
        steps()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        steps()
    for yh in ys_host:
        yh.fill_(float("nan"))
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for i in range(n):
        for j, ec in enumerate(ecs):
            ref = oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32),
                                        xs_np[i][j].astype(np.float32), np.float32)
            got = ys_host[i][yoff[j]:yoff[j] + my[j]].numpy()
            assert rel_err(got, ref) <= 1e-5, (i, j)
