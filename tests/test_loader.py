"""Native `.ecsr` loader (csrc/ecsr_loader.cpp) against the
reference's own `deserialize` (storage.py:431-483): same acceptance, same ContainerError
messages. The device half (load -> unpack bit-exact, SpMV parity) is
marked gpu."""

import struct

import numpy as np
import pytest

from conftest import golden_names, have_reference, load_golden
from paper_2507_12205_b200 import container as C
from paper_2507_12205_b200.device import parse_blob
from paper_2507_12205_b200.errors import ContainerError

NAME = "uniform_256x256_s0.5_b8_seed11"


@pytest.mark.parametrize("name", golden_names())
def test_parse_accepts_golden_and_matches_header(name):
    g = load_golden(name)
    ec = C.deserialize(g["blob"])
    info = parse_blob(g["blob"])
    assert info["num_rows"] == ec.num_rows and info["num_cols"] == ec.num_cols
    assert info["nsets"] == len(ec.sets) and info["warp_size"] == ec.warp_size
    assert info["delta_bits"] == ec.delta_bits and info["value_bits"] == ec.value_bits
    assert info["stored_cols"] == sum(s.stored_cols for s in ec.sets)
    assert info["num_blocks"] == sum(s.num_blocks for s in ec.sets)
    assert info["real_nnz"] == sum(s.real_nnz for s in ec.sets)


def _mutations(blob):
    hdr = 4
    yield "magic", b"WXYZ" + blob[4:]
    yield "version", blob[:hdr] + bytes([42]) + blob[hdr + 1:]
    yield "vsize", blob[:hdr + 1] + bytes([3]) + blob[hdr + 2:]
    yield "vbits", blob[:hdr + 2] + bytes([24]) + blob[hdr + 3:]
    yield "dbits", blob[:hdr + 3] + bytes([7]) + blob[hdr + 4:]
    yield "warp", blob[:hdr + 4] + struct.pack("<H", 0) + blob[hdr + 6:]
    yield "trailing", blob + b"junk"
    desc = 4 + 26
    yield "g0", blob[:desc] + struct.pack("<L", 0) + blob[desc + 4:]
    # a row_indices length one entry longer than the blob can hold / than the set needs
    yield "rows+1", blob[:desc + 32] + struct.pack("<Q", struct.unpack_from("<Q", blob, desc + 32)[0] + 1) + \
        blob[desc + 40:]
    for cut in (0, 3, 4, 10, 29, 30, 45, 61, 100, len(blob) // 2, len(blob) - 1):
        yield f"cut{cut}", blob[:cut]


def _reference_error(blob):
    """The reference's own deserialize (storage.py:431-483) on the same bytes."""
    if not have_reference():
        pytest.skip("reference package (baseline/_ref) not importable")
    from ecsr import storage
    from ecsr.errors import ContainerError as RefContainerError

    try:
        storage.deserialize(blob)
    except (RefContainerError, ContainerError) as e:
        return str(e)
    return None


@pytest.mark.parametrize("which", [m for m, _ in _mutations(load_golden(NAME)["blob"])])
def test_parse_rejects_corruption_like_reference(which):
    blob = dict(_mutations(load_golden(NAME)["blob"]))[which]
    want = _reference_error(blob)
    assert want is not None
    with pytest.raises(ContainerError) as ei:
        parse_blob(blob)
    assert str(ei.value).endswith(want) or want in str(ei.value)


def test_parse_rejects_bad_shapes_like_reference():
    ec = load_golden(NAME)["ec"]
    s = ec.sets[0]
    bad = [
        ("indptr", dict(block_indptr=np.concatenate([s.block_indptr[:-1], s.block_indptr[-1:] + 128]))),
        ("width", dict(block_indptr=np.concatenate([[0], s.block_indptr[1:] + 1]).astype(np.int64))),
        ("bases", dict(base_indices=s.base_indices[:-1])),
        ("rows", dict(row_indices=s.row_indices[:-1])),
        ("values", dict(block_values=s.block_values[:-1])),
    ]
    for what, repl in bad:
        fields = {f: getattr(s, f) for f in ("granularity", "vector_size", "num_blocks", "stored_cols",
                                               "real_nnz", "row_indices", "block_indptr", "base_indices",
                                               "delta_indices", "pad_mask", "block_values")}
        fields.update(repl)
        s2 = C.EcCsrSet(**fields)
        ec2 = C.EcCsrMatrix(ec.num_rows, ec.num_cols, ec.value_bits, ec.delta_bits, ec.warp_size,
                            [s2] + ec.sets[1:])
        blob = _serialize_unchecked(ec2)
        want = _reference_error(blob)
        assert want is not None, what
        with pytest.raises(ContainerError, match=None) as ei:
            parse_blob(blob)
        assert want in str(ei.value), (what, want, str(ei.value))


def _pack_deltas(d, bits):
    d = np.asarray(d).astype(np.uint32)
    if bits == 4:
        lo, hi = d[0::2], np.append(d[1::2], np.zeros(len(d) % 2, np.uint32))
        return (lo | (hi << 4)).astype(np.uint8).tobytes()
    return d.astype(np.uint8 if bits == 8 else "<u2").tobytes()


def _serialize_unchecked(ec):
    """serialize without the shape checks, to build malformed blobs."""
    out = [C.MAGIC, struct.pack("<BBBBHQQL", C.VERSION, ec.sets[0].block_values.dtype.itemsize,
                                ec.value_bits, ec.delta_bits, ec.warp_size, ec.num_rows, ec.num_cols,
                                len(ec.sets))]
    for s in ec.sets:
        out.append(struct.pack("<LLQQQ", s.granularity, s.vector_size, s.num_blocks, s.stored_cols,
                               s.real_nnz))
        for arr, dt in ((s.row_indices, "<u4"), (s.block_indptr, "<u8"), (s.base_indices, "<u4")):
            a = np.asarray(arr).astype(dt)
            out.append(struct.pack("<Q", a.size) + a.tobytes())
        d = np.asarray(s.delta_indices)
        out.append(struct.pack("<Q", d.size) + _pack_deltas(d, ec.delta_bits))
        m = np.asarray(s.pad_mask, dtype=bool)
        out.append(struct.pack("<Q", m.size) + np.packbits(m, bitorder="little").tobytes())
        v = np.asarray(s.block_values)
        out.append(struct.pack("<Q", v.size) + v.astype(v.dtype.newbyteorder("<")).tobytes())
    return b"".join(out)


def test_unchecked_serializer_matches_on_valid_input():
    g = load_golden(NAME)
    assert _serialize_unchecked(g["ec"]) == g["blob"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", golden_names()[::4])
def test_load_device_matches_to_device(name):
    import torch

    from paper_2507_12205_b200.device import load_device, spmv, to_device

    g = load_golden(name)
    ec = C.deserialize(g["blob"])
    for dt in ("f16", "f32"):
        a, b = load_device(g["blob"], device_dtype=dt), to_device(ec, device_dtype=dt)
        assert a.bytes() == b.bytes()
        ua, ub = a.unpack(), b.unpack()
        assert C.serialize(ua) == C.serialize(ub)
        x = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, ec.num_cols)).to(a.x_dtype).cuda()
        ya = spmv(a, x, ordered=True)
        yb = spmv(b, x, ordered=True)
        assert torch.equal(ya, yb)

