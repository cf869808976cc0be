"""Operation record and gate vocabulary of the drop-in boundary.

The reference's circuit op is ``{kind, wires, params, ctrls, ctrl_values,
trainable flags}`` over the GateKind vocabulary of SPEC.md:129.
Gate *arithmetic* (matrices, generators) lives in the native library
(csrc/gates.cu); this module only names kinds, checks arities and packs
records for the C-ABI -- no binding-layer arithmetic.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError

# Order and spelling follow SPEC.md:129; the integer codes are the
# ``sv_gate_kind`` enum of include/svb200.h.
GATE_KINDS = (
    "I", "X", "Y", "Z", "H", "S", "T", "Phase", "RX", "RY", "RZ", "Rot",
    "CNOT", "CZ", "SWAP", "IsingXX", "IsingXY", "IsingYY", "IsingZZ",
    "SingleExcitation", "DoubleExcitation", "ControlledMatrix", "Matrix",
)
KIND_CODE = {name: i for i, name in enumerate(GATE_KINDS)}

# (number of target wires, number of parameters); None = any (Matrix kinds).
ARITY = {
    "I": (1, 0), "X": (1, 0), "Y": (1, 0), "Z": (1, 0), "H": (1, 0),
    "S": (1, 0), "T": (1, 0), "Phase": (1, 1), "RX": (1, 1), "RY": (1, 1),
    "RZ": (1, 1), "Rot": (1, 3), "CNOT": (2, 0), "CZ": (2, 0), "SWAP": (2, 0),
    "IsingXX": (2, 1), "IsingXY": (2, 1), "IsingYY": (2, 1), "IsingZZ": (2, 1),
    "SingleExcitation": (2, 1), "DoubleExcitation": (4, 1),
    "ControlledMatrix": (None, 0), "Matrix": (None, 0),
}

# Kinds with a single-parameter generator; Rot is
# differentiable through its RZ.RY.RZ decomposition.
DIFFERENTIABLE = frozenset({
    "Phase", "RX", "RY", "RZ", "Rot", "IsingXX", "IsingXY", "IsingYY",
    "IsingZZ", "SingleExcitation", "DoubleExcitation",
})


@dataclass
class Op:
    """One gate application.

    ``wires`` are the target wires (for CNOT: ``(control, target)`` as in the
    reference's Bell example); ``ctrls``/``ctrl_values`` add extra
    controls to any kind (Alg. 2 generalised); ``ctrl_values``
    align with ``ctrls`` as given (state.py:214-215). ``trainable`` is a tuple
    of per-parameter flags; ``inverse`` applies the adjoint.
    """

    name: str
    wires: tuple
    params: tuple = ()
    ctrls: tuple = ()
    ctrl_values: tuple = ()
    trainable: tuple = ()
    inverse: bool = False
    matrix: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        if self.name not in KIND_CODE:
            raise ValidationError(f"unknown gate kind {self.name!r}")
        self.wires = tuple(int(w) for w in np.atleast_1d(self.wires))
        self.params = tuple(float(p) for p in np.atleast_1d(self.params)) if len(np.atleast_1d(self.params)) else ()
        self.ctrls = tuple(int(c) for c in self.ctrls)
        if isinstance(self.ctrl_values, str):
            if not all(c in "01" for c in self.ctrl_values):
                raise ValidationError(f"control value string must be binary, got {self.ctrl_values!r}")
            self.ctrl_values = tuple(int(c) for c in self.ctrl_values)
        else:
            self.ctrl_values = tuple(int(v) for v in self.ctrl_values)
        if self.ctrls and not self.ctrl_values:
            self.ctrl_values = (1,) * len(self.ctrls)  # default all ones, state.py:175-176
        if any(v not in (0, 1) for v in self.ctrl_values):
            raise ValidationError(f"control values must be bits, got {self.ctrl_values!r}")
        if len(self.ctrl_values) != len(self.ctrls):
            raise ValidationError(f"{len(self.ctrls)} controls but {len(self.ctrl_values)} control values")
        nw, npar = ARITY[self.name]
        if self.matrix is not None:
            self.matrix = np.ascontiguousarray(self.matrix, dtype=np.complex128)
        if nw is None:
            if self.matrix is None:
                raise ValidationError(f"{self.name} needs a matrix")
            dim = 1 << len(self.wires)
            if self.matrix.shape != (dim, dim):
                raise ValidationError(
                    f"matrix shape {self.matrix.shape} does not match {len(self.wires)} wires")
        elif len(self.wires) != nw:
            raise ValidationError(f"{self.name} acts on {nw} wires, got {len(self.wires)}")
        if npar is not None and len(self.params) != npar:
            raise ValidationError(f"{self.name} takes {npar} parameters, got {len(self.params)}")
        if self.trainable in (True, False):
            self.trainable = (bool(self.trainable),) * len(self.params)
        self.trainable = tuple(bool(t) for t in self.trainable)
        if self.trainable and len(self.trainable) != len(self.params):
            raise ValidationError(
                f"{self.name}: {len(self.trainable)} trainable flags for {len(self.params)} parameters")

    @property
    def n_trainable(self):
        return sum(self.trainable)

    @property
    def all_wires(self):
        return self.ctrls + self.wires


def gate(name, wires, *params, ctrls=(), ctrl_values=(), trainable=(), inverse=False, matrix=None):
    """Convenience constructor: ``gate("RX", 3, 0.2, trainable=True)``."""
    return Op(name, wires, tuple(params), tuple(ctrls), ctrl_values, trainable, inverse, matrix)


def trainable_columns(ops):
    """(op index, param index) for every Jacobian column, in circuit order."""
    cols = []
    for i, op in enumerate(ops):
        for p, t in enumerate(op.trainable):
            if t:
                cols.append((i, p))
    return cols
