"""GPU parity: the CUDA path (through the C-ABI) vs the reference's outputs and the oracle.

Bars (north_star):
  * encodings: unpack(pack(ec)) reproduces every reference array bit-exactly
    (values: their fp16 rounding) -- tolerance 0;
  * y, ordered mode: bitwise equal to the reference's f32 arithmetic on fp16-rounded
    values and x (`y16`), and the generic f32/f64 handles bitwise equal to the
    reference's compiled backend (`y32`, `y64`) -- tolerance 0;
  * y, fast (atomic) mode: rel-inf <= 1e-5 vs y16 (only the y-accumulation order
    differs) and rel-L2 <= 1e-3 vs the reference's FP32 result y32.
"""

import numpy as np
import pytest

import oracle
from conftest import golden_names, load_golden, rel_err, rel_l2
from paper_2507_12205_b200 import container as C

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2507_12205_b200 import backend  # noqa: E402
from paper_2507_12205_b200.device import spmv, to_device, unpack, vstack  # noqa: E402

TIGHT_ATOMIC = 1e-5
NORTH_STAR_L2 = 1e-3


def _x16(x):
    return torch.from_numpy(x.astype(np.float16)).cuda()


@pytest.mark.parametrize("name", golden_names())
def test_f16_ordered_bitwise_and_atomic_tolerance(name):
    g = load_golden(name)
    ec, x = g["ec"], g["x"]
    W = to_device(ec)
    expect_tiled = (ec.warp_size == 32 and ec.delta_bits <= 8 and len(ec.sets) > 0
                    and all(s.vector_size in (1, 4) for s in ec.sets))
    assert (W.layout == "tiled") == expect_tiled
    y_ord = spmv(W, _x16(x), ordered=True).cpu().numpy()
    assert y_ord.dtype == np.float32
    assert np.array_equal(y_ord, g["y16"]), rel_err(y_ord, g["y16"])
    y_fast = spmv(W, _x16(x)).cpu().numpy()
    assert rel_err(y_fast, g["y16"]) <= TIGHT_ATOMIC
    assert rel_l2(y_fast, g["y32"]) <= NORTH_STAR_L2


@pytest.mark.parametrize("name", golden_names())
def test_generic_handles_bitwise_vs_reference_backend(name):
    g = load_golden(name)
    ec, x = g["ec"], g["x"]
    W64 = to_device(ec, device_dtype="f64")
    y64 = spmv(W64, torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(y64, g["y64"])
    W32 = to_device(ec.astype(np.float32), device_dtype="f32")
    y32 = spmv(W32, torch.from_numpy(x.astype(np.float32)).cuda()).cpu().numpy()
    assert np.array_equal(y32, g["y32"])
    W16g = to_device(ec, force_generic=True)
    assert W16g.layout == "generic"
    y16 = spmv(W16g, _x16(x)).cpu().numpy()
    assert np.array_equal(y16, g["y16"])


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("force_generic", [False, True])
def test_unpack_reproduces_encoding_bit_exactly(name, force_generic):
    g = load_golden(name)
    ec = g["ec"]
    W = to_device(ec, force_generic=force_generic)
    back = unpack(W, np.float64)
    assert (back.num_rows, back.num_cols, back.warp_size, back.delta_bits) == (
        ec.num_rows, ec.num_cols, ec.warp_size, ec.delta_bits)
    assert len(back.sets) == len(ec.sets)
    for a, b in zip(ec.sets, back.sets):
        assert (a.granularity, a.vector_size, a.num_blocks, a.stored_cols, a.real_nnz) == (
            b.granularity, b.vector_size, b.num_blocks, b.stored_cols, b.real_nnz)
        for f in ("row_indices", "block_indptr", "base_indices", "delta_indices", "pad_mask"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
        assert np.array_equal(a.block_values.astype(np.float16).astype(np.float64), b.block_values)
    ec16 = ec.astype(np.float16).astype(np.float64)
    assert C.serialize(back) == C.serialize(ec16)
    assert C.storage_components(back, 16) == g["report"]
    byt = W.bytes()
    assert byt["model_kernel_bytes"] == C.kernel_model_bytes(ec)


@pytest.mark.parametrize("name", ["uniform_256x256_s0.5_b8_seed11", "corpus_049",
                                  "planted_512x384_s0.5_b8_seed15"])
def test_accumulate_mode(name):
    g = load_golden(name)
    ec, x = g["ec"], g["x"]
    W = to_device(ec)
    y0 = np.random.default_rng(1).uniform(-1, 1, ec.num_rows).astype(np.float32)
    y = torch.from_numpy(y0.copy()).cuda()
    spmv(W, _x16(x), y=y, accumulate=True, ordered=True)
    ec16 = ec.astype(np.float16).astype(np.float32)
    ref = y0.copy()
    for s in ec16.sets:
        oracle.spmv_set(s.granularity, ec.warp_size, s.vector_size, s.row_indices,
                        s.block_indptr, s.base_indices, s.delta_indices, s.block_values,
                        x.astype(np.float16).astype(np.float32), ref)
    assert np.array_equal(y.cpu().numpy(), ref)
    y = torch.from_numpy(y0.copy()).cuda()
    spmv(W, _x16(x), y=y, accumulate=True)
    assert rel_err(y.cpu().numpy(), ref) <= TIGHT_ATOMIC


@pytest.mark.parametrize("name", ["corpus_000", "corpus_049", "uniform_200x300_s0.7_b8_seed12",
                                  "kat_two_row_block"])
def test_backend_spmv_set_bitwise_vs_oracle(name):
    g = load_golden(name)
    ec, x = g["ec"], g["x"]
    for dt in (np.float64, np.float32):
        y_gpu = np.random.default_rng(2).uniform(-1, 1, ec.num_rows).astype(dt)
        y_cpu = y_gpu.copy()
        for s in ec.sets:
            args = (s.granularity, ec.warp_size, s.vector_size, s.row_indices, s.block_indptr,
                    s.base_indices, s.delta_indices, s.block_values.astype(dt), x.astype(dt))
            backend.spmv_set(*args, y_gpu)
            oracle.spmv_set(*args, y_cpu)
        assert np.array_equal(y_gpu, y_cpu)


def test_vstack_is_concatenation():
    a = load_golden("uniform_256x256_s0.5_b8_seed11")
    b = load_golden("uniform_256x256_s0.5_b4_seed17")
    ec = vstack([a["ec"], b["ec"]]) if a["ec"].delta_bits == b["ec"].delta_bits else None
    if ec is None:
        ec = vstack([a["ec"], a["ec"]])
        parts = [a, a]
    else:
        parts = [a, b]
    x = a["x"]
    W = to_device(ec)
    y = spmv(W, _x16(x), ordered=True).cpu().numpy()
    ec16 = ec.astype(np.float16).astype(np.float32)
    ref = oracle.spmv_ec_oracle(ec16, x.astype(np.float16).astype(np.float32), np.float32)
    assert np.array_equal(y, ref)
    assert y.shape == (sum(p["ec"].num_rows for p in parts),)


def test_empty_container_gives_zero():
    ec = C.EcCsrMatrix(5, 7, 16, 8, 32, [])
    W = to_device(ec)
    y = spmv(W, torch.ones(7, dtype=torch.float16, device="cuda"))
    assert torch.count_nonzero(y).item() == 0
    y = spmv(W, torch.ones(7, dtype=torch.float16, device="cuda"), ordered=True)
    assert torch.count_nonzero(y).item() == 0


def test_zero_width_block_is_skipped():
    # a hand-built set with a zero-width block between two real ones (_speedups.pyx:105-106)
    g = load_golden("uniform_256x256_s0.5_b8_seed11")
    ec = g["ec"]
    s = ec.sets[0]
    nb = s.num_blocks
    indptr = np.concatenate([s.block_indptr[:2], s.block_indptr[1:]])
    rows = np.concatenate([s.row_indices[:s.granularity], s.row_indices[:s.granularity],
                           s.row_indices[s.granularity:]])
    bases = np.concatenate([s.base_indices[:32], s.base_indices[:32], s.base_indices[32:]])
    s2 = C.EcCsrSet(s.granularity, s.vector_size, nb + 1, s.stored_cols, s.real_nnz, rows,
                    indptr, bases, s.delta_indices, s.pad_mask, s.block_values)
    ec2 = C.EcCsrMatrix(ec.num_rows, ec.num_cols, ec.value_bits, ec.delta_bits, 32,
                        [s2] + ec.sets[1:])
    W = to_device(ec2)
    y = spmv(W, _x16(g["x"]), ordered=True).cpu().numpy()
    assert np.array_equal(y, g["y16"])
    back = unpack(W, np.float64)
    assert np.array_equal(back.sets[0].block_indptr, indptr)


def test_cuda_graph_replay_and_determinism():
    g = load_golden("planted_512x384_s0.5_b8_seed15")
    W = to_device(g["ec"])
    x = _x16(g["x"])
    y = torch.empty(W.num_rows, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        spmv(W, x, y=y, ordered=True)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        spmv(W, x, y=y, ordered=True)
    for _ in range(3):
        y.fill_(7.0)
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), g["y16"])


def test_x_dtype_and_shape_errors():
    g = load_golden("uniform_256x256_s0.5_b8_seed11")
    W = to_device(g["ec"])
    with pytest.raises(ValueError):
        spmv(W, torch.ones(255, dtype=torch.float16, device="cuda"))
    with pytest.raises(ValueError):
        spmv(W, torch.ones(256, dtype=torch.float32, device="cuda"))


@pytest.mark.parametrize("name", ["planted_512x384_s0.5_b8_seed15", "magnitude_256x512_s0.7_b8_seed14"])
def test_overwrite_mode_zeroes_y_in_kernel_across_graph_replays(name):
    # fast overwrite: the kernel zeroes y itself behind a generation-counted grid gate;
    # back-to-back launches of one handle (same stream, PDL) must never see stale y.
    g = load_golden(name)
    W = to_device(g["ec"])
    x = _x16(g["x"])
    ys = [torch.full((W.num_rows,), 1e6, dtype=torch.float32, device="cuda") for _ in range(3)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        spmv(W, x, y=ys[0])
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for y in ys:
            spmv(W, x, y=y)
    for rep in range(4):
        for y in ys:
            y.fill_(-3e5 * (rep + 1))
        graph.replay()
        torch.cuda.synchronize()
        for y in ys:
            assert rel_err(y.cpu().numpy(), g["y16"]) <= TIGHT_ATOMIC


@pytest.mark.parametrize("tile_kb", [4, 8])
def test_ring_wraps_many_times_small_tiles(tile_kb):
    # records handed out several ring cycles ahead of the producer (regression: parity
    # aliasing of the full barriers): small tiles (pack flag ECSR_PACK_TILE_KB)
    g = load_golden("planted_512x384_s0.5_b8_seed15")
    ec = vstack([g["ec"]] * 6)
    W = to_device(ec, tile_kb=tile_kb)
    assert W.bytes()["tiles"] > 8 * W.bytes()["stages"]
    x = g["x"]
    y = spmv(W, _x16(x), ordered=True).cpu().numpy()
    ref = oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32),
                                x.astype(np.float16).astype(np.float32), np.float32)
    assert np.array_equal(y, ref)
    ys = [spmv(W, _x16(x)) for _ in range(20)]
    torch.cuda.synchronize()
    assert all(rel_err(v.cpu().numpy(), ref) <= TIGHT_ATOMIC for v in ys)


@pytest.mark.parametrize("rows,sparsity,per_cta", [(4096, 0.5, 32), (114688, 0.95, 256)])
def test_many_tiles_per_cta_wrap_stage_map(rows, sparsity, per_cta):
    # > 32 tiles per CTA: the producer's 32-tile record-count window slides and the
    # 32-entry tile -> stage map wraps many times (1 KB tiles, one record each); > 256:
    # the consumers' shared prefix-count cache overflows to global loads
    from paper_2507_12205_b200.encoder import convert_csr
    from paper_2507_12205_b200.generators import make_matrix

    ec = convert_csr(make_matrix("magnitude", rows, 4096, sparsity, 7, dtype=np.float32))
    W = to_device(ec, tile_kb=1)
    b = W.bytes()
    assert b["tiles"] > per_cta * b["grid"], (b["tiles"], b["grid"])
    x = np.random.default_rng(2).uniform(-1, 1, 4096)
    xd = _x16(x)
    ref = oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32),
                                x.astype(np.float16).astype(np.float32), np.float32)
    y = spmv(W, xd, ordered=True).cpu().numpy()
    assert np.array_equal(y, ref)
    for _ in range(5):
        assert rel_err(spmv(W, xd).cpu().numpy(), ref) <= TIGHT_ATOMIC


def test_concurrent_streams_share_one_handle():
    # one handle, two streams, launches interleaved without host syncs: each stream has
    # its own workspace (gate counter, partials), so overwrite mode (grid gate) and
    # ordered mode (partials) stay exact while the launches overlap
    g = load_golden("planted_512x384_s0.5_b8_seed15")
    ec = vstack([g["ec"]] * 8)
    W = to_device(ec)
    rng = np.random.default_rng(11)
    xs = [rng.uniform(-1, 1, ec.num_cols) for _ in range(2)]
    refs = [oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32),
                                  x.astype(np.float16).astype(np.float32), np.float32) for x in xs]
    streams = [torch.cuda.Stream() for _ in range(2)]
    xd = [_x16(x) for x in xs]
    ys = [[torch.empty(ec.num_rows, device="cuda") for _ in range(16)] for _ in range(2)]
    torch.cuda.synchronize()
    for i in range(16):
        for s in range(2):
            spmv(W, xd[s], y=ys[s][i], ordered=(i % 4 == 3), stream=streams[s])
    torch.cuda.synchronize()
    for s in range(2):
        for i, y in enumerate(ys[s]):
            got = y.cpu().numpy()
            if i % 4 == 3:
                assert np.array_equal(got, refs[s])
            else:
                assert rel_err(got, refs[s]) <= TIGHT_ATOMIC


def test_fifth_stream_is_rejected_and_device_checked():
    g = load_golden("planted_512x384_s0.5_b8_seed15")
    W = to_device(g["ec"])
    x = _x16(g["x"])
    streams = [torch.cuda.Stream() for _ in range(5)]
    for s in streams[:4]:
        spmv(W, x, stream=s)
    with pytest.raises(ValueError, match="other streams"):
        spmv(W, x, stream=streams[4])
    torch.cuda.synchronize()
    with pytest.raises(ValueError):
        spmv(W, x, y=torch.empty(W.num_rows))  # host y
