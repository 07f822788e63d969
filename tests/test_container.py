"""Host container mirror vs the reference: wire format, byte model, validation, generators."""

import numpy as np
import pytest

from conftest import golden_manifest, golden_names, load_golden, needs_reference
from paper_2507_12205_b200 import container as C
from paper_2507_12205_b200.errors import ContainerError
from paper_2507_12205_b200.generators import generate_uniform, magnitude_pruned, planted_blocks


@pytest.mark.parametrize("name", golden_names())
def test_serialize_roundtrip_byte_identical(name):
    g = load_golden(name)
    assert C.serialize(g["ec"]) == g["blob"]


@pytest.mark.parametrize("name", golden_names())
def test_storage_components_match_reference_report(name):
    g = load_golden(name)
    assert C.storage_components(g["ec"], 16) == g["report"]


@pytest.mark.parametrize("name", golden_names())
def test_validate_accepts_reference_output(name):
    C.validate_container(load_golden(name)["ec"])


def test_manifest_hashes_match_blobs():
    import hashlib

    for name, case in golden_manifest().items():
        assert hashlib.sha256(load_golden(name)["blob"]).hexdigest() == case["sha256"]


@pytest.mark.parametrize("mutate,pattern", [
    (lambda b: b"WXYZ" + b[4:], "magic"),
    (lambda b: b[:4] + bytes([42]) + b[5:], "version"),
    (lambda b: b[: len(b) - 8], "truncated"),
    (lambda b: b + b"junk", "trailing"),
])
def test_deserialize_rejects_corruption(mutate, pattern):
    # acceptance criterion C10 (pkg/tests/test_acceptance.py:250-265)
    blob = load_golden("uniform_256x256_s0.5_b8_seed11")["blob"]
    with pytest.raises(ContainerError, match=pattern):
        C.deserialize(mutate(blob))


def test_validate_rejects_malformed():
    # pkg/tests/test_executor.py:72-85
    ec = load_golden("uniform_256x256_s0.5_b8_seed11")["ec"]
    ec.sets[0].block_indptr = ec.sets[0].block_indptr.copy()
    ec.sets[0].block_indptr[-1] += 128
    with pytest.raises(ContainerError):
        C.validate_container(ec)


def test_validate_rejects_out_of_range_decode():
    ec = load_golden("uniform_256x256_s0.5_b8_seed11")["ec"]
    s = ec.sets[0]
    s.base_indices = s.base_indices.copy()
    s.delta_indices = s.delta_indices.copy()
    s.base_indices[0] = 250
    s.delta_indices[:] = 200
    with pytest.raises(ContainerError):
        C.validate_container(ec)


def test_kernel_model_bytes_formula():
    g = load_golden("magnitude_384x256_s0.5_b8_seed13")
    ec, rep = g["ec"], g["report"]
    expect = sum(v for k, v in rep.items() if k not in ("pad_mask", "desc"))
    assert C.kernel_model_bytes(ec) == expect + 2 * ec.num_cols + 4 * ec.num_rows


def test_empty_container_roundtrip():
    ec = C.EcCsrMatrix(4, 4, 64, 8, 2, [])
    assert C.deserialize(C.serialize(ec)).sets == []


@needs_reference
@pytest.mark.parametrize("m,k,s,seed", [(64, 96, 0.5, 0), (300, 17, 0.9, 3), (1, 64, 0.0, 0)])
def test_generate_uniform_matches_reference(m, k, s, seed):
    from ecsr import core

    a = generate_uniform(m, k, s, seed)
    b = core.generate_uniform(m, k, s, seed)
    assert np.array_equal(a.row_ptr, b.row_ptr)
    assert np.array_equal(a.col_idx, b.col_idx)
    assert a.values.tobytes() == b.values.tobytes()


def test_magnitude_pruned_properties():
    a = magnitude_pruned(64, 128, 0.5, seed=3)
    assert a.nnz == 64 * 64
    dense = np.random.default_rng(3).standard_normal((64, 128), dtype=np.float32)
    dense *= np.float32(1.0 / np.sqrt(128))
    for r in range(64):
        cols = a.col_idx[a.row_ptr[r]:a.row_ptr[r + 1]]
        assert np.all(np.diff(cols) > 0)
        kept = np.abs(dense[r, cols]).min()
        dropped = np.delete(np.abs(dense[r]), cols).max()
        assert kept >= dropped
        assert np.array_equal(a.values[a.row_ptr[r]:a.row_ptr[r + 1]], dense[r, cols])


def test_planted_blocks_has_shared_patterns():
    a = planted_blocks(128, 256, 0.5, seed=1)
    pats = {}
    for r in range(128):
        key = a.col_idx[a.row_ptr[r]:a.row_ptr[r + 1]].tobytes()
        pats[key] = pats.get(key, 0) + 1
    sizes = sorted(pats.values(), reverse=True)
    assert sizes[0] == 8 and 4 in sizes and 2 in sizes


@pytest.mark.parametrize("name", golden_names())
def test_decode_round_trip_and_matches_reference_decode(name):
    # storage.decode_ec_csr (storage.py:260-309): decode(convert(A)) == A exactly
    import sys

    from conftest import GOLDEN

    sys.path.insert(0, GOLDEN)
    from cases import golden_matrix

    g = load_golden(name)
    case = golden_manifest()[name]
    a = golden_matrix(case)
    d = C.decode_ec_csr(g["ec"])
    assert np.array_equal(d.row_ptr, a.row_ptr)
    assert np.array_equal(d.col_idx, a.col_idx)
    assert np.array_equal(d.values, np.asarray(a.values, dtype=d.values.dtype))


@needs_reference
@pytest.mark.parametrize("name", golden_names())
def test_native_deserialize_equals_reference(name):
    # the native parser (ecsr_b200_blob_*) against the reference's storage.deserialize
    from ecsr import storage

    blob = load_golden(name)["blob"]
    ref, got = storage.deserialize(blob), C.deserialize(blob)
    assert (ref.num_rows, ref.num_cols, ref.value_bits, ref.delta_bits, ref.warp_size) == \
        (got.num_rows, got.num_cols, got.value_bits, got.delta_bits, got.warp_size)
    assert len(ref.sets) == len(got.sets)
    for a, b in zip(ref.sets, got.sets):
        assert (a.granularity, a.vector_size, a.num_blocks, a.stored_cols, a.real_nnz) == \
            (b.granularity, b.vector_size, b.num_blocks, b.stored_cols, b.real_nnz)
        for f in ("row_indices", "block_indptr", "base_indices", "delta_indices", "pad_mask", "block_values"):
            x, y = np.asarray(getattr(a, f)), np.asarray(getattr(b, f))
            assert x.shape == y.shape and np.array_equal(x.astype(y.dtype), y), f
        assert np.asarray(b.block_values).dtype == np.asarray(a.block_values).dtype
    assert storage.serialize(ref) == C.serialize(got) == blob
