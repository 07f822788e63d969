"""Native encoder (libecsr_b200 ecsr_b200_encode) vs the reference's convert_csr.

Gate: serialize(native) == serialize(reference), byte for byte,
on every golden case (reference encodings committed under tests/golden/) and, where
the reference is importable, on fresh seeded matrices including the clip_limit and
max_levels knobs (storage.py:700-708, extraction.py:341-356, balance.py:20-44).
"""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, golden_manifest, load_golden, needs_reference
from paper_2507_12205_b200 import container as C
from paper_2507_12205_b200.encoder import convert_csr
from paper_2507_12205_b200.errors import ContainerError
from paper_2507_12205_b200.generators import CsrMatrix, generate_uniform, make_matrix

sys.path.insert(0, GOLDEN)
from cases import golden_matrix  # noqa: E402


@pytest.mark.parametrize("name", list(golden_manifest()))
def test_native_encoder_matches_reference_golden(name):
    case = golden_manifest()[name]
    g = load_golden(name)
    ec = convert_csr(golden_matrix(case), case["warp"], case["vector"], case["delta_bits"],
                     dtype=np.float64)
    assert C.serialize(ec) == g["blob"]


@needs_reference
@pytest.mark.parametrize("kind,m,k,s,seed,w,v,b,clip,levels", [
    ("uniform", 300, 400, 0.6, 7, 32, 4, 8, None, None),
    ("magnitude", 512, 384, 0.5, 8, 32, 4, 8, None, None),
    ("planted", 640, 512, 0.6, 9, 32, 4, 8, None, None),
    ("planted", 256, 300, 0.5, 10, 8, 2, 4, None, None),
    ("uniform", 200, 700, 0.8, 11, 4, 1, 16, None, None),
    ("planted", 384, 384, 0.5, 12, 32, 4, 8, 200, None),
    ("planted", 384, 384, 0.5, 13, 32, 4, 8, None, 1),
    ("uniform", 64, 1024, 0.97, 14, 32, 4, 4, None, None),
    # K >= 65536: overlaps exceed the uint16 cache, the matching computes them on the fly
    ("planted", 128, 66000, 0.9, 15, 32, 4, 8, None, None),
])
def test_native_encoder_matches_live_reference(kind, m, k, s, seed, w, v, b, clip, levels):
    from ecsr import core, storage
    from ecsr.extraction import ExtractionConfig

    a = make_matrix(kind, m, k, s, seed, dtype=np.float32)
    ref = storage.convert_csr(core.CsrMatrix(a.num_rows, a.num_cols, a.row_ptr, a.col_idx, a.values),
                              ExtractionConfig(w, v, b, max_levels=levels), clip_limit=clip)
    ours = convert_csr(a, w, v, b, max_levels=levels, clip_limit=clip)
    assert C.serialize(ours) == storage.serialize(ref)


def test_encoder_round_trip_partitions_matrix():
    # every nonzero lands in exactly one block exactly once (extraction.py:341-356)
    a = make_matrix("planted", 256, 256, 0.6, 3, dtype=np.float64)
    ec = convert_csr(a)
    dense = np.zeros((256, 256))
    for s in ec.sets:
        for bi in range(s.num_blocks):
            st, en = s.block_indptr[bi], s.block_indptr[bi + 1]
            n = en - st
            d = s.delta_indices[st:en].reshape(n // (32 * s.vector_size), 32, s.vector_size)
            d = d.transpose(1, 0, 2).reshape(32, -1).astype(np.int64)
            cols = s.base_indices[bi * 32:(bi + 1) * 32, None].astype(np.int64) + np.cumsum(d, axis=1)
            vals = s.block_values[st * s.granularity:en * s.granularity].reshape(
                n // (32 * s.vector_size), 32, s.vector_size, s.granularity).transpose(1, 0, 2, 3)
            mask = s.pad_mask[st:en].reshape(n // (32 * s.vector_size), 32, s.vector_size)
            mask = mask.transpose(1, 0, 2).reshape(32, -1)
            vals = vals.reshape(32, -1, s.granularity)
            for k in range(s.granularity):
                r = s.row_indices[bi * s.granularity + k]
                np.add.at(dense[r], cols[~mask], vals[..., k][~mask])
    assert np.array_equal(dense, a.to_dense())


def test_encoder_empty_and_degenerate_inputs():
    empty = CsrMatrix(5, 7, np.zeros(6, np.int64), np.zeros(0, np.int64), np.zeros(0))
    ec = convert_csr(empty)
    assert ec.sets == [] and (ec.num_rows, ec.num_cols) == (5, 7)
    one = generate_uniform(1, 64, 0.0, seed=0)
    ec = convert_csr(one)
    assert sum(s.real_nnz for s in ec.sets) == 64


def test_encoder_rejects_bad_input():
    a = generate_uniform(8, 8, 0.5, seed=0)
    with pytest.raises(ValueError):
        convert_csr(a, delta_bits=5)
    bad = CsrMatrix(1, 4, np.array([0, 2]), np.array([2, 1]), np.array([1.0, 2.0]))
    with pytest.raises(ValueError):
        convert_csr(bad)
    oob = CsrMatrix(1, 4, np.array([0, 1]), np.array([9]), np.array([1.0]))
    with pytest.raises(ValueError):
        convert_csr(oob)
