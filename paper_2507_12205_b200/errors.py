"""Exception types, mirroring `ecsr.errors` (`pkg/src/ecsr/errors.py:4-16`).

When the reference package is importable (tests, this container) the classes
ARE the reference's, so `pytest.raises(ecsr.errors.ContainerError)` catches
errors raised by this package and vice versa. On the GPU box, where the
reference is absent, same-named local classes stand in.
"""

try:  # pragma: no cover - depends on the environment
    from ecsr.errors import (  # type: ignore
        ContainerError,
        DeltaOverflowError,
        EcsrError,
        MatrixFormatError,
    )
except ImportError:  # the GPU box: no reference installed

    class EcsrError(Exception):
        """Base class for all errors raised by this package."""

    class MatrixFormatError(EcsrError):
        """A matrix file could not be parsed."""

    class ContainerError(EcsrError):
        """An EC-CSR container is malformed, truncated, or inconsistent."""

    class DeltaOverflowError(EcsrError):
        """A column gap exceeds the configured delta range."""


class DeviceError(EcsrError):
    """A CUDA call inside libecsr_b200 failed (C-ABI return code 3)."""


__all__ = ["EcsrError", "MatrixFormatError", "ContainerError", "DeltaOverflowError",
           "DeviceError"]
