"""Grouped launch (ecsr_b200_group_*): several independent products in ONE launch, and
the overwrite mode's memset path (taken when the grid cannot be co-resident).

Every member's y is checked against the C oracle of the reference kernel on
fp16-rounded inputs (pkg/src/ecsr/_speedups.pyx:81-129): fast mode within rel-inf 1e-5
(the tolerance of the single-matrix tests), ordered mode bit for bit.
"""

import numpy as np
import pytest

import oracle
from conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2507_12205_b200.device import SpmvGroup, spmv, to_device, vstack  # noqa: E402
from paper_2507_12205_b200.encoder import convert_csr  # noqa: E402
from paper_2507_12205_b200.generators import make_matrix  # noqa: E402

TOL = 1e-5
NAMES = ["planted_512x384_s0.5_b8_seed15", "magnitude_256x512_s0.7_b8_seed14",
         "uniform_256x256_s0.5_b8_seed11", "uniform_200x300_s0.7_b8_seed12"]


def _ref16(ec, x):
    return oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32),
                                 x.astype(np.float16).astype(np.float32), np.float32)


def _members(names, seed=0):
    rng = np.random.default_rng(seed)
    ecs = [load_golden(n)["ec"] for n in names]
    xs = [rng.uniform(-1, 1, ec.num_cols) for ec in ecs]
    Ws = [to_device(ec) for ec in ecs]
    assert all(W.layout == "tiled" for W in Ws)
    return ecs, xs, Ws


def _x16(x):
    return torch.from_numpy(np.asarray(x).astype(np.float16)).cuda()


def test_group_matches_each_member():
    ecs, xs, Ws = _members(NAMES)
    g = SpmvGroup(Ws)
    info = g.info()
    assert info["launches"] == 1
    assert sum(info["ctas"]) == info["grid"] and min(info["ctas"]) >= 1
    xd = [_x16(x) for x in xs]
    refs = [_ref16(ec, x) for ec, x in zip(ecs, xs)]
    for _ in range(3):  # overwrite mode: the gate zeroes every member's y each launch
        ys = g.spmv(xd)
        for y, r in zip(ys, refs):
            assert rel_err(y.cpu().numpy(), r) <= TOL
    ys = g.spmv(xd, ys=ys, accumulate=True)
    for y, r in zip(ys, refs):
        assert rel_err(y.cpu().numpy(), 2 * r) <= TOL
    ys = g.spmv(xd, ordered=True)
    for y, r in zip(ys, refs):
        assert np.array_equal(y.cpu().numpy(), r)


def test_group_graph_replay_and_stream_reuse():
    ecs, xs, Ws = _members(NAMES[:3], seed=1)
    g = SpmvGroup(Ws)
    xd = [_x16(x) for x in xs]
    ys = [torch.full((W.num_rows,), 7.0, device="cuda") for W in Ws]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g.spmv(xd, ys, stream=s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for _ in range(4):
            g.spmv(xd, ys, stream=s)
    refs = [_ref16(ec, x) for ec, x in zip(ecs, xs)]
    for _ in range(5):
        for y in ys:
            y.fill_(3.0)
        graph.replay()
        torch.cuda.synchronize()
        for y, r in zip(ys, refs):
            assert rel_err(y.cpu().numpy(), r) <= TOL


def test_group_of_bench_shapes():
    # one launch for matrices of different K (x of 8 KB and 22 KB side by side)
    mats = [(1024, 4096, 0.5), (2048, 4096, 0.5), (1024, 11008, 0.5)]
    ecs = [convert_csr(make_matrix("magnitude", m, k, s, 60 + i, dtype=np.float32))
           for i, (m, k, s) in enumerate(mats)]
    Ws = [to_device(ec) for ec in ecs]
    g = SpmvGroup(Ws)
    rng = np.random.default_rng(4)
    xs = [rng.uniform(-1, 1, ec.num_cols) for ec in ecs]
    ys = g.spmv([_x16(x) for x in xs])
    for ec, x, y in zip(ecs, xs, ys):
        assert rel_err(y.cpu().numpy(), _ref16(ec, x)) <= TOL


def test_group_mixes_one_and_two_ctas_per_sm():
    # x of 40 KB packs for one CTA per SM, the others for two: the group issues one
    # launch per class
    ecs, xs, Ws = _members(NAMES[:2], seed=6)
    ec = convert_csr(make_matrix("magnitude", 256, 20000, 0.98, 5, dtype=np.float32))
    ecs.append(ec)
    xs.append(np.random.default_rng(7).uniform(-1, 1, 20000))
    Ws.append(to_device(ec))
    g = SpmvGroup(Ws)
    info = g.info()
    assert info["launches"] == 2 and sum(info["ctas"]) == info["grid"]
    for _ in range(3):
        ys = g.spmv([_x16(x) for x in xs])
        for e, x, y in zip(ecs, xs, ys):
            assert rel_err(y.cpu().numpy(), _ref16(e, x)) <= TOL


def test_group_single_member_equals_handle():
    ecs, xs, Ws = _members(NAMES[:1], seed=2)
    g = SpmvGroup(Ws)
    assert g.info()["grid"] == Ws[0].bytes()["grid"]
    y = g.spmv([_x16(xs[0])])[0].cpu().numpy()
    assert rel_err(y, _ref16(ecs[0], xs[0])) <= TOL


def test_group_rejects_bad_members():
    ecs, xs, Ws = _members(NAMES[:2])
    with pytest.raises(ValueError):
        SpmvGroup([Ws[0], to_device(ecs[1], force_generic=True)])  # generic layout
    with pytest.raises(ValueError):
        SpmvGroup(Ws * 5)  # 10 > 8 members
    g = SpmvGroup(Ws)
    with pytest.raises(ValueError):
        g.spmv([_x16(xs[0])])


@pytest.mark.parametrize("grouped", [False, True])
def test_memset_path_equals_gated_path(grouped):
    # the overwrite mode's two implementations -- the in-kernel zero-y gate and the
    # memset + ungated launch (taken when the grid cannot be co-resident) -- give the
    # same y, launch after launch
    ecs, xs, Ws = _members(NAMES, seed=3)
    xd = [_x16(x) for x in xs]
    refs = [_ref16(ec, x) for ec, x in zip(ecs, xs)]
    g = SpmvGroup(Ws) if grouped else None
    for i in range(10):
        ys = g.spmv(xd, memset_y=bool(i % 2)) if grouped else \
            [spmv(W, x, memset_y=bool(i % 2)) for W, x in zip(Ws, xd)]
        for y, r in zip(ys, refs):
            assert rel_err(y.cpu().numpy(), r) <= TOL


def test_gate_survives_sm_contention():
    # a long launch on another stream holds SMs while ours starts: not every CTA of our
    # grid can be resident at first, so resident CTAs either wait or claim the missing
    # slices; the result must be exact either way
    big = to_device(vstack([load_golden(NAMES[0])["ec"]] * 64))
    ecs, xs, Ws = _members(NAMES[:2], seed=5)
    xd = [_x16(x) for x in xs]
    refs = [_ref16(ec, x) for ec, x in zip(ecs, xs)]
    xb = _x16(np.ones(big.num_cols))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for _ in range(5):
        with torch.cuda.stream(s1):
            for _ in range(4):
                spmv(big, xb, stream=s1)
        with torch.cuda.stream(s2):
            outs.append([spmv(W, x, stream=s2) for W, x in zip(Ws, xd)])
    torch.cuda.synchronize()
    for ys in outs:
        for y, r in zip(ys, refs):
            assert rel_err(y.cpu().numpy(), r) <= TOL
