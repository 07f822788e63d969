"""BASELINE.json configs 1-5 at full matrix sizes on the B200 (native encoder inputs).

The reference encoder takes minutes to hours at these shapes, so the
inputs come from the native encoder (byte-identical to the reference:
tests/test_encoder.py). Checks are size-independent: the device layout unpacks to the
encoding bit for bit, ordered-mode y equals the C oracle of the reference kernel on
fp16-rounded inputs bit for bit, fast mode is within rel-inf 1e-5 of it, and the
whole-matrix product matches the f64 CSR oracle within the north-star rel-L2 1e-3.
Also the padding/NaN edge case of SURVEY.md §8(a) a15(3).
"""

import numpy as np
import pytest

import oracle
from conftest import rel_err, rel_l2
from paper_2507_12205_b200 import container as C

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2507_12205_b200.device import spmv, to_device, unpack  # noqa: E402
from paper_2507_12205_b200.encoder import convert_csr  # noqa: E402
from paper_2507_12205_b200.generators import make_matrix  # noqa: E402
from paper_2507_12205_b200.sharded import row_slice, shard_bounds  # noqa: E402

CASES = [
    # (label, generator, rows, cols, sparsity, seed, row-shard (i, n) or None)
    ("13B-q planted 5120x5120 @50%", "planted", 5120, 5120, 0.5, 31, None),
    ("13B-up planted 13824x5120 @60%, shard 3/8", "planted", 13824, 5120, 0.6, 32, (3, 8)),
    ("OPT-30B-q 7168x7168 @70%", "magnitude", 7168, 7168, 0.7, 33, None),
    ("OPT-30B-fc2 7168x28672 @70%, shard 0/8", "magnitude", 7168, 28672, 0.7, 34, (0, 8)),
    ("70B-up 28672x8192 @50%, shard 5/8", "magnitude", 28672, 8192, 0.5, 35, (5, 8)),
    # configs[0] and configs[1] at the sparsities the bench does not time
    ("config-1 4096x4096 @50% seed 1", "magnitude", 4096, 4096, 0.5, 1, None),
    ("7B-q 4096x4096 @60%", "magnitude", 4096, 4096, 0.6, 36, None),
    ("7B-q 4096x4096 @70%", "magnitude", 4096, 4096, 0.7, 37, None),
    ("7B-up 11008x4096 @60%", "magnitude", 11008, 4096, 0.6, 38, None),
    ("7B-up 11008x4096 @70%", "magnitude", 11008, 4096, 0.7, 39, None),
    ("7B-down 4096x11008 @60%", "magnitude", 4096, 11008, 0.6, 40, None),
    ("7B-down 4096x11008 @70%", "magnitude", 4096, 11008, 0.7, 41, None),
    ("OPT-30B-fc1 28672x7168 @70% unsharded", "magnitude", 28672, 7168, 0.7, 42, None),
    # K > 65535: the u32-base record variant (ecsr_kernels.cuh, p.wide)
    ("wide K 1024x70000 @90%", "magnitude", 1024, 70000, 0.9, 43, None),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_config_scale_parity(case):
    _, kind, m, k, s, seed, shard = case
    a = make_matrix(kind, m, k, s, seed, dtype=np.float32)
    if shard is not None:
        b = shard_bounds(a.row_ptr, shard[1])
        a = row_slice(a, b[shard[0]], b[shard[0] + 1])
    ec = convert_csr(a)
    W = to_device(ec)
    assert W.layout == "tiled"
    back = unpack(W, np.float64)
    assert C.serialize(back) == C.serialize(ec.astype(np.float16).astype(np.float64))
    x = np.random.default_rng(seed).uniform(-1, 1, k)
    x16 = x.astype(np.float16)
    xd = torch.from_numpy(x16).cuda()
    ec16 = ec.astype(np.float16).astype(np.float32)
    ref16 = oracle.spmv_ec_oracle(ec16, x16.astype(np.float32), np.float32)
    y_ord = spmv(W, xd, ordered=True).cpu().numpy()
    assert np.array_equal(y_ord, ref16)
    y = spmv(W, xd).cpu().numpy()
    assert rel_err(y, ref16) <= 1e-5
    y64 = oracle.spmv_oracle_f64(a, x)
    assert rel_l2(y, y64) <= 1e-3


def test_padding_is_multiplied_so_nonfinite_x_propagates():
    # storage.py:197-201: padding repeats a real column (or column 0) with value 0, and
    # the kernel multiplies it (no pad_mask branch): x = inf there gives NaN in the
    # reference too. Ordered mode must match bit for bit.
    a = make_matrix("uniform", 96, 200, 0.9, 5, dtype=np.float32)
    ec = convert_csr(a)
    x = np.random.default_rng(0).uniform(-1, 1, 200).astype(np.float16)
    x[0] = np.inf
    W = to_device(ec)
    y = spmv(W, torch.from_numpy(x).cuda(), ordered=True).cpu().numpy()
    ref = oracle.spmv_ec_oracle(ec.astype(np.float16).astype(np.float32), x.astype(np.float32),
                                np.float32)
    assert np.array_equal(np.isnan(y), np.isnan(ref)) and np.isnan(ref).any()
    fin = np.isfinite(ref)
    assert np.array_equal(y[fin], ref[fin])


@pytest.mark.parametrize("shapes", [[(4096, 4096)] * 3, [(11008, 4096)] * 2],
                         ids=["stacked q|k|v 3x4096x4096 @50%", "stacked gate|up 2x11008x4096 @50%"])
def test_stacked_launch_parity(shapes):
    # the bench's row-stacked launches (matrices sharing x packed as one handle)
    from paper_2507_12205_b200.device import vstack

    ecs = [convert_csr(make_matrix("magnitude", m, k, 0.5, 50 + i, dtype=np.float32))
           for i, (m, k) in enumerate(shapes)]
    ec = vstack(ecs)
    W = to_device(ec)
    assert W.layout == "tiled"
    k = shapes[0][1]
    x16 = np.random.default_rng(9).uniform(-1, 1, k).astype(np.float16)
    ref16 = np.concatenate([oracle.spmv_ec_oracle(e.astype(np.float16).astype(np.float32),
                                                  x16.astype(np.float32), np.float32) for e in ecs])
    xd = torch.from_numpy(x16).cuda()
    assert np.array_equal(spmv(W, xd, ordered=True).cpu().numpy(), ref16)
    assert rel_err(spmv(W, xd).cpu().numpy(), ref16) <= 1e-5
