"""B200-native EC-CSR SpMV (arxiv 2507.12205 hot path), a drop-in for the `ecsr` package.

Public API (names follow the reference `ecsr` package, pkg/src/ecsr/__init__.py):

    to_device(ec) -> DeviceMatrix          validate once + pack (libecsr_b200.so)
    load_device(path | bytes)              .ecsr blob -> DeviceMatrix in one native call
    parse_blob(path | bytes)               native host-only parse + shape check of a blob
    spmv(W, x) -> y                        y = W x on the GPU (fp16 in, fp32 accumulate)
    group([W1, W2, ..]).spmv([x1, x2, ..]) independent products in ONE launch
    spmv_ec(ec, x)                         executor.spmv_ec-compatible convenience
    EcCsrMatrix / EcCsrSet, serialize, deserialize, storage_components,
    kernel_model_bytes, validate_container  host container (storage.py mirror)
    backend.register()                     plug into ecsr._kernels as backend "b200"
    linear.SparseLinear                    torch.nn.Module for decode-time linear layers
"""

from .container import (  # noqa: F401
    EcCsrMatrix,
    EcCsrSet,
    decode_ec_csr,
    deserialize,
    from_reference,
    kernel_model_bytes,
    load_container,
    save_container,
    serialize,
    storage_components,
    validate_container,
)
from .errors import ContainerError, DeltaOverflowError, DeviceError, EcsrError  # noqa: F401

__version__ = "0.1.0"


def to_device(ec, device_dtype: str = "f16", force_generic: bool = False, device=None):
    from .device import to_device as _to_device

    return _to_device(ec, device_dtype=device_dtype, force_generic=force_generic, device=device)


def load_device(blob_or_path, device_dtype: str = "f16", force_generic: bool = False, device=None):
    from .device import load_device as _load_device

    return _load_device(blob_or_path, device_dtype=device_dtype, force_generic=force_generic,
                        device=device)


def parse_blob(blob_or_path) -> dict:
    from .device import parse_blob as _parse_blob

    return _parse_blob(blob_or_path)


def spmv(W, x, y=None, accumulate: bool = False, ordered: bool = False, stream=None):
    from .device import spmv as _spmv

    return _spmv(W, x, y=y, accumulate=accumulate, ordered=ordered, stream=stream)


def group(mats):
    """One launch for several independent products (device.SpmvGroup)."""
    from .device import SpmvGroup

    return SpmvGroup(mats)


def spmv_ec(ec, x, ordered: bool = True):
    """`executor.spmv_ec(ec, x)` (executor.py:80-96) computed on the GPU.

    Packs in the container's precision (generic kernel, bitwise equal to the
    reference's compiled backend) and returns a host array of the container dtype.
    """
    import numpy as np

    from .device import spmv_host, to_device as _to_device

    x = np.asarray(x)
    if x.shape != (ec.num_cols,):
        raise ValueError(f"x has shape {x.shape}, expected ({ec.num_cols},)")
    dt = "f64" if np.dtype(ec.dtype) == np.float64 else "f32"
    W = _to_device(ec, device_dtype=dt)
    return spmv_host(W, x, ordered=ordered)
