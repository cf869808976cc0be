"""Reference-shaped host API over the B200 state (mirror of ``svkit.state``, state.py:1-303).

Same names, argument meaning and error classes as the reference module, so code and tests
written against ``svkit.state`` run unchanged on the GPU:

* ``StateVector`` / ``zero_state`` / ``StateVector.from_amplitudes``  (state.py:24-92)
* ``get_masks`` / ``MaskSet``                                          (state.py:100-151)
* ``apply_single_qubit``            -- Alg. 1                          (state.py:154-171)
* ``apply_controlled_single_qubit`` -- Alg. 2                          (state.py:192-226)
* ``apply_matrix``                                                     (state.py:278-303)

Difference by necessity: the reference's coefficient interaction is an arbitrary Python
callable ``f(amps, i0, i1)`` that cannot run on the GPU. Here ``f`` is a
:class:`CoefficientInteraction` (``interaction_of(kind, params)`` or any 2x2 matrix); a bare
callable raises UnsupportedOperationError. Amplitudes live in HBM; ``.amplitudes`` copies
them out (copy-out marshalling).
"""

from dataclasses import dataclass

import numpy as np

from .device import Device
from .errors import CapacityError, UnsupportedOperationError, ValidationError
from .ops import KIND_CODE, Op

BIT_WIDTH = 64
UINT_MAX = (1 << BIT_WIDTH) - 1
MAX_QUBITS = 62
_NORM_TOL = {"f64": 1e-12, "f32": 1e-5}


class StateVector:
    """2**n_qubits amplitudes resident on a B200; fresh instances hold |0...0>.

    ``precision`` selects complex128 ("f64", default) or complex64 ("f32"), as the reference's
    StateVector (state.py:20, 24-31).
    """

    __slots__ = ("n_qubits", "_dev")

    def __init__(self, n_qubits, precision="f64", device=0):
        if precision not in ("f64", "f32"):
            raise ValidationError(f"unknown precision {precision!r}; expected 'f64' or 'f32'")
        if not isinstance(n_qubits, (int, np.integer)) or isinstance(n_qubits, bool) or n_qubits < 1:
            raise ValidationError(f"n_qubits must be a positive integer, got {n_qubits!r}")
        if n_qubits > MAX_QUBITS:
            raise CapacityError(f"n_qubits={n_qubits} exceeds the {MAX_QUBITS}-qubit addressing limit")
        self._dev = Device(int(n_qubits), precision=precision, device=device)
        self.n_qubits = int(n_qubits)

    @classmethod
    def from_amplitudes(cls, amplitudes, copy=True):
        """Upload an amplitude array; its length must be a power of two (state.py:49-66)."""
        amps = np.asarray(amplitudes)
        if amps.ndim != 1 or amps.size < 2 or amps.size & (amps.size - 1):
            raise ValidationError("amplitude array length must be a power of two >= 2")
        n = int(amps.size.bit_length() - 1)
        if n > MAX_QUBITS:
            raise CapacityError(f"{n} qubits exceeds the {MAX_QUBITS}-qubit limit")
        # complex64 input keeps its precision; anything else becomes complex128 (state.py:56-60)
        precision = "f32" if amps.dtype == np.complex64 else "f64"
        sv = cls(n, precision)
        sv._dev.set_state(amps)
        return sv

    @property
    def device(self):
        return self._dev

    @property
    def amplitudes(self):
        return self._dev.get_state()

    @property
    def precision(self):
        return self._dev.precision

    @property
    def dtype(self):
        return np.dtype(self._dev.dtype)

    def norm(self):
        return float(self._dev.norm())

    def copy(self):
        return StateVector.from_amplitudes(self.amplitudes)

    def __repr__(self):
        return f"StateVector(n_qubits={self.n_qubits}, precision={self.precision!r}, device='cuda:{self._dev.device}')"


def zero_state(n_qubits, precision="f64"):
    """|0...0> on ``n_qubits`` qubits (state.py:90-92)."""
    return StateVector(n_qubits, precision)


@dataclass(frozen=True)
class MaskSet:
    """Disjoint bit masks partitioning the non-excluded window bits (state.py:100-124)."""

    masks: tuple
    strides: tuple

    def expand(self, k):
        i0 = k & self.masks[0]
        for i in range(1, len(self.masks)):
            i0 |= (k << i) & self.masks[i]
        return i0

    def expand_array(self, ks):
        out = ks & np.uint64(self.masks[0])
        for i in range(1, len(self.masks)):
            out |= (ks << np.uint64(i)) & np.uint64(self.masks[i])
        return out


def get_masks(excluded_bit_offsets, n_qubits):
    """n_excluded + 1 masks around the excluded bit offsets (state.py:128-151).

    This is host-side index bookkeeping (the same rule the CUDA kernels apply with shifts
    when they insert the fixed bits); it returns the reference's MaskSet.
    """
    bits = sorted(excluded_bit_offsets)
    if len(set(bits)) != len(bits):
        raise ValidationError(f"excluded bit offsets contain duplicates: {excluded_bit_offsets}")
    for b in bits:
        if not 0 <= b < n_qubits:
            raise ValidationError(f"excluded bit offset {b} outside [0, {n_qubits})")
    window = (1 << n_qubits) - 1
    if not bits:
        return MaskSet(masks=(window,), strides=())
    masks = [(1 << bits[0]) - 1]
    for lo, hi in zip(bits[:-1], bits[1:]):
        masks.append(((1 << hi) - 1) ^ ((1 << (lo + 1)) - 1))
    masks.append(window & ~((1 << (bits[-1] + 1)) - 1))
    return MaskSet(masks=tuple(masks), strides=tuple(1 << b for b in bits))


class CoefficientInteraction:
    """A single-qubit gate's pairwise update (Listing 1 role), as a 2x2 matrix
    that the GPU applies to every (i0, i1) pair."""

    __slots__ = ("matrix", "name")

    def __init__(self, matrix, name="Matrix"):
        m = np.asarray(matrix, dtype=np.complex128)
        if m.shape != (2, 2):
            raise ValidationError(f"a coefficient interaction is a 2x2 matrix, got shape {m.shape}")
        self.matrix = m
        self.name = name

    def __call__(self, amps, i0, i1):
        raise UnsupportedOperationError("interactions execute on the GPU; apply them with apply_single_qubit")


def interaction_of(kind, params=()):
    """CoefficientInteraction of a single-qubit GateKind; the matrix is built
    by the native gate library."""
    if kind not in KIND_CODE:
        raise ValidationError(f"unknown gate kind {kind!r}")
    op = Op(kind, (0,), tuple(params))
    if len(op.wires) != 1 or kind in ("Matrix", "ControlledMatrix"):
        raise UnsupportedOperationError(f"{kind} is not a single-qubit kind")
    d = Device(1)
    try:
        d.apply([op], fuse=False)
        col0 = d.get_state()
        d.set_basis_state(1)
        d.apply([op], fuse=False)
        col1 = d.get_state()
    finally:
        d.release()
    return CoefficientInteraction(np.stack([col0, col1], axis=1), kind)


def _as_matrix(f):
    if isinstance(f, CoefficientInteraction):
        return f.matrix
    if callable(f):
        raise UnsupportedOperationError(
            "arbitrary Python interaction callables cannot run on the GPU; pass a CoefficientInteraction "
            "(interaction_of) or a 2x2 matrix")
    return CoefficientInteraction(f).matrix


def _check_qubit(q, n_qubits, label="qubit"):
    if not 0 <= q < n_qubits:
        raise ValidationError(f"{label} {q} out of range for {n_qubits}-qubit register")


def _normalize_ctrl_values(ctrls, ctrl_values):
    """state.py:174-189: default all ones; a binary string or 0/1 sequence aligned with ctrls."""
    if ctrl_values is None or (isinstance(ctrl_values, (tuple, list)) and len(ctrl_values) == 0 and len(ctrls) > 0):
        return (1,) * len(ctrls)
    if isinstance(ctrl_values, str):
        if not all(c in "01" for c in ctrl_values):
            raise ValidationError(f"control value string must be binary, got {ctrl_values!r}")
        values = tuple(int(c) for c in ctrl_values)
    else:
        values = tuple(int(v) for v in ctrl_values)
        if not all(v in (0, 1) for v in values):
            raise ValidationError(f"control values must be bits, got {ctrl_values!r}")
    if len(values) != len(ctrls):
        raise ValidationError(f"{len(ctrls)} controls but {len(values)} control values")
    return values


def apply_single_qubit(sv, q, f):
    """Alg. 1 on the GPU: ``f`` updates each of the 2**(n-1) disjoint pairs of qubit ``q``."""
    _check_qubit(q, sv.n_qubits)
    m = _as_matrix(f)
    sv.device.apply([Op("Matrix", (q,), matrix=m)], fuse=False)


def apply_controlled_single_qubit(sv, ctrls, q, f, ctrl_values=None):
    """Alg. 2 on the GPU: ``f`` on qubit ``q`` where the control bits match ``ctrl_values``."""
    n = sv.n_qubits
    _check_qubit(q, n)
    ctrls = tuple(ctrls)
    if len(set(ctrls)) != len(ctrls):
        raise ValidationError(f"duplicate control qubits: {ctrls}")
    if q in ctrls:
        raise ValidationError(f"target qubit {q} overlaps controls {ctrls}")
    for c in ctrls:
        _check_qubit(c, n, "control")
    values = _normalize_ctrl_values(ctrls, ctrl_values)
    m = _as_matrix(f)
    sv.device.apply([Op("ControlledMatrix", (q,), ctrls=ctrls, ctrl_values=values, matrix=m)], fuse=False)


def apply_matrix(sv, wires, matrix, validate_unitary=False):
    """Dense 2**w x 2**w contraction on ordered wires, in place (wires[0] = MSB; state.py:278-303)."""
    wires = tuple(wires)
    if len(set(wires)) != len(wires):
        raise ValidationError(f"duplicate wires: {wires}")
    for w in wires:
        _check_qubit(w, sv.n_qubits, "wire")
    matrix = np.asarray(matrix)
    if matrix.shape != (1 << len(wires), 1 << len(wires)):
        raise ValidationError(f"matrix shape {matrix.shape} does not match {len(wires)} wires")
    if validate_unitary:
        err = np.abs(matrix.conj().T @ matrix - np.eye(1 << len(wires))).max()
        if err > 1e-10:
            raise ValidationError(f"matrix is not unitary (max deviation {err:.2e})")
    sv.device.apply_matrix(wires, matrix)
