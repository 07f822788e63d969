"""Coalescing audit of the device layout.

The kernel's reads, replayed by ecsr_b200_trace over the device arena, are audited with
the reference's rules (executor.py:171-221: one aligned span of W*v deltas / W*v*g values
per warp step, tiling each block exactly) -- by the reference's own check_coalescing when
the reference package is importable -- and with the tiled layout's device rules (every
span one 16-B-aligned reference chunk). Like pkg/tests/test_executor.py:134-150, a
corrupted trace must be flagged.
"""

import numpy as np
import pytest

from conftest import golden_names, have_reference, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2507_12205_b200.device import to_device  # noqa: E402
from paper_2507_12205_b200.trace import (as_reference_trace, check_device_coalescing,  # noqa: E402
                                         device_trace)


def _stored_chunks(ec):
    return sum(int(s.stored_cols) // (ec.warp_size * int(s.vector_size)) for s in ec.sets)


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("force_generic", [False, True])
def test_device_trace_is_coalesced(name, force_generic):
    ec = load_golden(name)["ec"]
    W = to_device(ec, force_generic=force_generic)
    tr = device_trace(W)
    assert len(tr) == 2 * _stored_chunks(ec)
    assert check_device_coalescing(ec, tr, tiled=W.layout == "tiled") == []
    if have_reference():
        from ecsr import executor

        assert executor.check_coalescing(ec, as_reference_trace(tr, executor)) == []


def test_trace_at_config_scale_and_wide_k():
    from paper_2507_12205_b200.encoder import convert_csr
    from paper_2507_12205_b200.generators import make_matrix

    for m, k, s in [(4096, 4096, 0.5), (256, 70000, 0.99)]:
        ec = convert_csr(make_matrix("magnitude", m, k, s, 3, dtype=np.float32))
        W = to_device(ec)
        assert W.layout == "tiled"
        tr = device_trace(W)
        assert len(tr) == 2 * _stored_chunks(ec)
        assert check_device_coalescing(ec, tr) == []


def test_corrupted_trace_is_flagged():
    ec = load_golden("planted_512x384_s0.5_b8_seed15")["ec"]
    tr = device_trace(to_device(ec))
    i = next(i for i, r in enumerate(tr) if r.array == "deltas")
    bad = list(tr)
    bad[i] = tr[i]._replace(start=tr[i].start + 1)
    assert any("aligned" in v for v in check_device_coalescing(ec, bad))
    bad = list(tr)
    bad[i] = tr[i]._replace(dev_offset=tr[i].dev_offset + 8)
    assert any("16-B" in v for v in check_device_coalescing(ec, bad))
    assert any("never read" in v or "tile" in v for v in check_device_coalescing(ec, tr[2:]))
