"""svb200: B200-native complex128 state-vector hot path (gate apply, expval, adjoint Jacobian).

Drop-in for the device API of the reference CPU library ``svkit``.
The numerical work runs in ``libsvb200.so`` (hand-written sm_100a CUDA behind a C-ABI,
include/svb200.h); importing :class:`Device` or :mod:`.state` loads it and fails loudly if
it is missing -- there is no CPU fallback.
"""

from .errors import (CapacityError, DeviceError, SvkitError, UnsupportedOperationError,  # noqa: F401
                     ValidationError)
from .observables import DenseHermitian, Hamiltonian, PauliWord, SparseHermitian  # noqa: F401
from .ops import GATE_KINDS, Op, gate  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    if name in ("Device", "bind_device"):
        from . import device
        return getattr(device, name)
    raise AttributeError(name)
