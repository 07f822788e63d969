"""Pin the CPU oracle (oracle/liboracle.so) to the reference: golden vectors + live reference."""

import numpy as np
import pytest

import oracle
from conftest import golden_names, load_golden, needs_reference, rel_err


@pytest.mark.parametrize("name", golden_names())
def test_oracle_bitwise_vs_golden(name):
    g = load_golden(name)
    ec = g["ec"]
    x = g["x"]
    assert np.array_equal(oracle.spmv_ec_oracle(ec, x, np.float64), g["y64"])
    assert np.array_equal(oracle.spmv_ec_oracle(ec, x.astype(np.float32), np.float32), g["y32"])
    ec16 = ec.astype(np.float16).astype(np.float32)
    x16 = x.astype(np.float16).astype(np.float32)
    assert np.array_equal(oracle.spmv_ec_oracle(ec16, x16, np.float32), g["y16"])
    assert rel_err(g["y64"], g["yoracle"]) <= 1e-12


@needs_reference
@pytest.mark.parametrize("seed", range(4))
def test_oracle_bitwise_vs_live_reference(seed):
    from ecsr import _speedups, core, storage
    from ecsr.extraction import ExtractionConfig

    m = core.generate_uniform(96, 160, 0.6, seed=seed)
    ec = storage.convert_csr(m, ExtractionConfig(32, 4, 8))
    x = np.random.default_rng(seed).uniform(-1, 1, 160)
    for dt in (np.float64, np.float32):
        a = oracle.spmv_ec_oracle(ec, x, dt)
        b = oracle.spmv_ec_oracle(ec, x, dt, set_fn=_speedups.spmv_set)
        assert np.array_equal(a, b)


def test_reference_speedups_build_matches_oracle():
    ref = oracle.load_reference_speedups()
    if ref is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    g = load_golden("planted_512x384_s0.5_b8_seed15")
    for dt in (np.float64, np.float32):
        a = oracle.spmv_ec_oracle(g["ec"], g["x"], dt)
        b = oracle.spmv_ec_oracle(g["ec"], g["x"], dt, set_fn=ref.spmv_set)
        assert np.array_equal(a, b)
