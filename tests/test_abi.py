"""The C-ABI library: loads, exports every declared symbol, host-only entry points."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2507_12205_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "ecsr_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ecsr_b200_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name


def test_version_and_device_count_without_gpu():
    assert b"sm_100a" in _lib.lib().ecsr_b200_version()
    assert _lib.lib().ecsr_b200_device_count() >= 0


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_to_f16_matches_numpy_rne():
    rng = np.random.default_rng(0)
    vals = np.concatenate([
        rng.standard_normal(20000) * 10.0 ** rng.integers(-9, 6, 20000),
        np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 1e9, -1e9, np.inf, -np.inf,
                  2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26, 2.0 ** -14, 2.0 ** -14 * (1 - 2 ** -12),
                  1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11, 5.960464477539063e-08]),
    ])
    for dt in (np.float64, np.float32):
        v = vals.astype(dt)
        got = np.empty(v.size, np.uint16)
        rc = _lib.lib().ecsr_b200_to_f16(v.ctypes.data, _lib.dtype_code(dt), got.ctypes.data, v.size)
        assert rc == 0
        assert np.array_equal(got, v.astype(np.float16).view(np.uint16))
    nan = np.array([np.nan], np.float64)
    got = np.empty(1, np.uint16)
    _lib.lib().ecsr_b200_to_f16(nan.ctypes.data, _lib.F64, got.ctypes.data, 1)
    assert np.isnan(got.view(np.float16)[0])


def _host_set(ec, check_shapes=True):
    from paper_2507_12205_b200.device import _host_sets

    arr, keep, dt = _host_sets(ec, check_shapes)
    return arr, keep, dt


def test_short_arrays_rejected_before_the_c_abi():
    """Arrays shorter than the declared sizes never reach the native validator (which
    would read past them): ContainerError like the reference's _check_set_shapes."""
    from conftest import load_golden

    from paper_2507_12205_b200.errors import ContainerError

    ec = load_golden("uniform_256x256_s0.5_b8_seed11")["ec"]
    ec.sets[0].delta_indices = ec.sets[0].delta_indices[:-128]
    with pytest.raises(ContainerError, match="length mismatch"):
        _host_set(ec)


@pytest.mark.parametrize("corrupt,code", [
    ("indptr", _lib.ERR_CONTAINER), ("delta", _lib.ERR_CONTAINER), ("base", _lib.ERR_CONTAINER),
    ("row", _lib.ERR_CONTAINER), ("warp", _lib.ERR_VALUE),
])
def test_pack_validation_errors_need_no_gpu(corrupt, code):
    from conftest import load_golden

    ec = load_golden("uniform_256x256_s0.5_b8_seed11")["ec"]
    s = ec.sets[0]
    warp = ec.warp_size
    if corrupt == "indptr":  # last block 64 columns wider: not a multiple of W*v = 128
        s.block_indptr = s.block_indptr.copy()
        s.block_indptr[-1] += 64
        s.stored_cols += 64
        s.delta_indices = np.concatenate([s.delta_indices, np.zeros(64, s.delta_indices.dtype)])
        s.pad_mask = np.concatenate([s.pad_mask, np.ones(64, np.bool_)])
        s.block_values = np.concatenate([s.block_values,
                                         np.zeros(64 * s.granularity, s.block_values.dtype)])
    elif corrupt == "delta":
        s.delta_indices = s.delta_indices.copy()
        s.delta_indices[3] = 256
    elif corrupt == "base":
        s.base_indices = s.base_indices.copy()
        s.base_indices[0] = 250
        s.delta_indices = np.full_like(s.delta_indices, 200)
    elif corrupt == "row":
        s.row_indices = s.row_indices.copy()
        s.row_indices[0] = ec.num_rows
    elif corrupt == "warp":
        warp = 33
    # the native validator on its own (array lengths are consistent; contents are not)
    arr, keep, dt = _host_set(ec, check_shapes=False)
    out = ctypes.c_void_p()
    rc = _lib.lib().ecsr_b200_pack(arr, len(ec.sets), ec.num_rows, ec.num_cols, warp,
                                   ec.delta_bits, 16, _lib.dtype_code(dt), _lib.F16, 0,
                                   ctypes.byref(out))
    assert rc == code, _lib.last_error()
    assert not out.value
    assert _lib.last_error()


def test_host_io_rejects_bad_calls_before_any_device_work():
    """ecsr_b200_host_io's argument checks run on the host (no GPU needed)."""
    from paper_2507_12205_b200.device import _IoSpan

    lib = _lib.lib()
    buf = np.zeros(64, np.float32)
    one = (_IoSpan * 1)(_IoSpan(buf.ctypes.data, buf.ctypes.data, 256))
    assert lib.ecsr_b200_host_io(one, 17, 0, None) == _lib.ERR_VALUE
    assert "entries" in _lib.last_error()
    assert lib.ecsr_b200_host_io(one, 1, 2, None) == _lib.ERR_VALUE
    assert "flags" in _lib.last_error()
    odd = (_IoSpan * 1)(_IoSpan(buf.ctypes.data + 4, buf.ctypes.data, 16))
    assert lib.ecsr_b200_host_io(odd, 1, 0, None) == _lib.ERR_VALUE
    assert "16-B aligned" in _lib.last_error()
    # pageable host memory is not reachable by the kernel (no GPU here: also not device memory)
    assert lib.ecsr_b200_host_io(one, 1, 0, None) == _lib.ERR_VALUE
    assert "pinned" in _lib.last_error()
