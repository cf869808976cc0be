"""Observable records of the drop-in boundary.

Variants: ``PauliWord`` (list of (wire, P) with P in I/X/Y/Z), ``Hamiltonian``
(coefficients + Pauli words, H = sum_t c_t P_t) and
``DenseHermitian`` (wires + 2^w x 2^w matrix). Sparse CSR observables are the
"next" row of SURVEY.md §8(f) and raise UnsupportedOperationError.
These classes only validate and pack; every number is computed on the GPU.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError

PAULIS = "IXYZ"


@dataclass
class PauliWord:
    """Tensor product of single-qubit Paulis, e.g. ``PauliWord([(0, "Z"), (3, "X")])``."""

    factors: tuple

    def __post_init__(self):
        facs = []
        for w, p in self.factors:
            p = str(p).upper()
            if p not in PAULIS:
                raise ValidationError(f"unknown Pauli {p!r}")
            facs.append((int(w), p))
        wires = [w for w, _ in facs]
        if len(set(wires)) != len(wires):
            raise ValidationError(f"duplicate wire within Pauli word: {wires}")
        self.factors = tuple(facs)

    @classmethod
    def from_string(cls, s, wires=None):
        """``"XZ"`` on wires (0,1) by default, or explicit ``wires``."""
        wires = range(len(s)) if wires is None else wires
        return cls(tuple(zip(wires, s)))

    @property
    def wires(self):
        return tuple(w for w, _ in self.factors)

    def max_wire(self):
        return max(self.wires, default=-1)


@dataclass
class Hamiltonian:
    """Weighted sum of Pauli words."""

    coeffs: tuple
    terms: tuple

    def __post_init__(self):
        self.coeffs = tuple(float(c) for c in self.coeffs)
        self.terms = tuple(t if isinstance(t, PauliWord) else PauliWord(t) for t in self.terms)
        if len(self.coeffs) != len(self.terms):
            raise ValidationError(
                f"Hamiltonian has {len(self.coeffs)} coefficients but {len(self.terms)} terms")

    def max_wire(self):
        return max((t.max_wire() for t in self.terms), default=-1)


@dataclass
class DenseHermitian:
    """Dense observable on ``wires`` (wires[0] = MSB of the matrix index, state.py:281)."""

    wires: tuple
    matrix: np.ndarray = field(repr=False)

    def __post_init__(self):
        self.wires = tuple(int(w) for w in self.wires)
        self.matrix = np.ascontiguousarray(self.matrix, dtype=np.complex128)
        dim = 1 << len(self.wires)
        if self.matrix.shape != (dim, dim):
            raise ValidationError(
                f"matrix shape {self.matrix.shape} does not match {len(self.wires)} wires")
        if len(set(self.wires)) != len(self.wires):
            raise ValidationError(f"duplicate wires: {self.wires}")

    def max_wire(self):
        return max(self.wires, default=-1)


@dataclass
class SparseHermitian:
    """CSR observable over the whole register: row pointers, column indices and
    complex values over LOGICAL basis indices (qubit 0 = MSB). The structure is validated here
    (monotone row pointers, in-range columns) and again behind the C-ABI."""

    indptr: np.ndarray = field(repr=False)
    indices: np.ndarray = field(repr=False)
    data: np.ndarray = field(repr=False)

    def __post_init__(self):
        self.indptr = np.ascontiguousarray(self.indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(self.indices, dtype=np.int64)
        self.data = np.ascontiguousarray(self.data, dtype=np.complex128)
        dim = len(self.indptr) - 1
        if dim < 1 or self.indptr[0] != 0 or np.any(np.diff(self.indptr) < 0):
            raise ValidationError("malformed CSR: row pointers must start at 0 and be monotone")
        if self.indptr[-1] != len(self.indices) or len(self.indices) != len(self.data):
            raise ValidationError("malformed CSR: nnz mismatch between row pointers, columns and values")
        if len(self.indices) and (self.indices.min() < 0 or self.indices.max() >= dim):
            raise ValidationError("malformed CSR: column index out of range")

    @property
    def dim(self):
        return len(self.indptr) - 1

    @classmethod
    def from_dense(cls, matrix):
        m = np.asarray(matrix, dtype=np.complex128)
        rows, cols = np.nonzero(m)
        indptr = np.zeros(m.shape[0] + 1, dtype=np.int64)
        np.add.at(indptr, rows + 1, 1)
        return cls(np.cumsum(indptr), cols, m[rows, cols])

    @classmethod
    def from_scipy(cls, a):
        a = a.tocsr()
        return cls(a.indptr, a.indices, a.data)

    def to_dense(self):
        m = np.zeros((self.dim, self.dim), dtype=np.complex128)
        for r in range(self.dim):
            for k in range(self.indptr[r], self.indptr[r + 1]):
                m[r, self.indices[k]] += self.data[k]
        return m

    def max_wire(self):
        return self.dim.bit_length() - 2


def as_observable(obs):
    """Accept a PauliWord/Hamiltonian/DenseHermitian/SparseHermitian or a ``[(wire, P), ...]`` list."""
    if isinstance(obs, (PauliWord, Hamiltonian, DenseHermitian, SparseHermitian)):
        return obs
    return PauliWord(tuple(obs))
