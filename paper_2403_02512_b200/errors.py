"""Exception taxonomy of the drop-in boundary.

Mirrors the reference hierarchy class-for-class (errors.py:4-17 of the
reference: ``SvkitError``, ``ValidationError(ValueError)``, ``CapacityError``,
``UnsupportedOperationError``) so callers that catch the reference's classes
keep working. The C-ABI returns an integer status; :func:`raise_for_status`
maps it 1:1 onto these classes ("errors: mapped 1:1").
"""


class SvkitError(Exception):
    """Base class for all errors raised through the B200 state-vector boundary."""


class ValidationError(SvkitError, ValueError):
    """Invalid argument: bad wire index, arity mismatch, malformed structure."""


class CapacityError(SvkitError):
    """Requested register exceeds what the device(s) can allocate or address."""


class UnsupportedOperationError(SvkitError):
    """Operation is well-formed but outside the supported set."""


class DeviceError(SvkitError):
    """CUDA or NCCL runtime failure (no reference counterpart; status 4)."""


# Status codes of include/svb200.h (SV_OK .. SV_ERR_DEVICE).
SV_OK = 0
SV_ERR_VALIDATION = 1
SV_ERR_CAPACITY = 2
SV_ERR_UNSUPPORTED = 3
SV_ERR_DEVICE = 4

_BY_STATUS = {
    SV_ERR_VALIDATION: ValidationError,
    SV_ERR_CAPACITY: CapacityError,
    SV_ERR_UNSUPPORTED: UnsupportedOperationError,
    SV_ERR_DEVICE: DeviceError,
}


def raise_for_status(status, message):
    """Raise the exception class that C-ABI ``status`` maps to (no-op for SV_OK)."""
    if status == SV_OK:
        return
    cls = _BY_STATUS.get(status, SvkitError)
    raise cls(message)
