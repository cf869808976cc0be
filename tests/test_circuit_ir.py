"""CPU: circuit-ir module -- grammar examples, errors with line/caret, round
trips, templates, and the H2 fixture against the dense-diagonalisation oracle."""

import os

import numpy as np
import pytest

from oracle import svoracle as O
from paper_2403_02512_b200 import circuit_ir as C
from paper_2403_02512_b200.ops import Op

FIX = os.path.join(os.path.dirname(__file__), "fixtures", "h2.ham")


def dense(h, n):
    return np.stack([O.apply_observable(np.eye(1 << n, dtype=np.complex128)[:, k], n, h) for k in range(1 << n)],
                    axis=1)


def test_grammar_examples():
    c = C.parse_circuit("qubits 1\nX 0")
    assert c.n_qubits == 1 and [o.name for o in c.ops] == ["X"]
    bell = C.parse_circuit("qubits 2\nH 0\nCTRL[0] X 1")
    psi = O.run_circuit(2, bell.ops)
    assert np.allclose(psi, np.array([1, 0, 0, 1]) / np.sqrt(2))
    c = C.parse_circuit("# format: 1\nqubits 4\nCTRL[0,3=10] RZ(0.1) 2 train\ninv RX(0.3) 1  # comment")
    op = c.ops[0]
    assert op.ctrls == (0, 3) and op.ctrl_values == (1, 0) and op.trainable == (True,)
    assert c.ops[1].inverse and c.n_trainable == 1


@pytest.mark.parametrize("text,line,col", [
    ("qubits 2\nRX(0.5 0", 2, 3),            # SPEC example: caret at the open parenthesis
    ("qubits 2\nFOO 0", 2, 1),               # unknown gate
    ("qubits 2\nCNOT 0", 2, 1),              # arity mismatch
    ("qubits 2\nX 5", 2, 3),                 # wire out of range (caret at the wire)
    ("qubits 3\nCTRL[0=11] X 1", 3 - 1, 8),  # malformed control spec (2 bits for 1 control)
    ("X 0", 1, 1),                           # missing header
])
def test_parse_errors_carry_position(text, line, col):
    with pytest.raises(C.ParseError) as e:
        C.parse_circuit(text)
    assert e.value.line_no == line and e.value.col == col
    assert "^" in str(e.value)


def test_round_trip_random_circuits():
    rng = np.random.default_rng(0)
    kinds = [k for k in C._TEXT_KINDS]
    for _ in range(30):
        n = int(rng.integers(4, 9))
        ops = []
        for _ in range(40):
            k = kinds[int(rng.integers(len(kinds)))]
            nw, npar = C.ARITY[k]
            nc = int(rng.integers(0, 3)) if n - nw >= 2 else 0
            qs = rng.choice(n, size=nw + nc, replace=False)
            ops.append(Op(k, tuple(int(q) for q in qs[:nw]), tuple(rng.normal(size=npar)),
                          ctrls=tuple(int(q) for q in qs[nw:]),
                          ctrl_values=tuple(int(v) for v in rng.integers(0, 2, size=nc)),
                          trainable=(bool(rng.random() < 0.5),) * npar, inverse=bool(rng.random() < 0.2)))
        c = C.Circuit(n, ops)
        assert C.parse_circuit(C.serialize_circuit(c)) == c


def test_hamiltonian_format_and_h2_fixture():
    h = C.parse_hamiltonian("0.5 [Z0]\n-0.25 [X0 X1]")
    assert len(h.terms) == 2
    ident = C.parse_hamiltonian("1.0 []")
    psi = np.array([0.6, 0.8j], dtype=np.complex128)
    assert abs(O.expval(psi, 1, ident) - 1.0) < 1e-15
    with pytest.raises(C.ParseError):
        C.parse_hamiltonian("1.0 [Q0]")                  # malformed Pauli token
    with pytest.raises(C.ParseError):
        C.parse_hamiltonian("1.0 [X0 Z0]")               # duplicate wire within a term
    h2 = C.parse_hamiltonian(open(FIX).read())
    assert len(h2.terms) == 15
    assert C.parse_hamiltonian(C.serialize_hamiltonian(h2)) == h2
    e0 = np.linalg.eigvalsh(dense(h2, 4))[0]
    assert abs(e0 - (-1.1361894540)) < 1e-8           # H2 / STO-3G ground energy


def test_templates():
    c = C.strongly_entangling_layers(2, 1, np.zeros((1, 2, 3)))
    assert [o.name for o in c.ops] == ["Rot", "Rot", "CNOT", "CNOT"]
    c = C.strongly_entangling_layers(4, 3, np.zeros((3, 4, 3)))
    assert sum(o.name == "Rot" for o in c.ops) == 12 and sum(o.name == "CNOT" for o in c.ops) == 12
    assert c.n_trainable == 36
    c = C.strongly_entangling_layers(3, 1, np.zeros((1, 3, 3)))
    assert [o.wires for o in c.ops if o.name == "CNOT"] == [(0, 1), (1, 2), (2, 0)]
    with pytest.raises(C.ValidationError):
        C.strongly_entangling_layers(3, 1, np.zeros((1, 2, 3)))
    singles, doubles = C.excitations(4, 2)
    assert len(singles) == 2 and len(doubles) == 1
    h2 = C.parse_hamiltonian(open(FIX).read())
    c = C.singles_doubles_ansatz(4, 2, np.zeros(3))
    psi = O.run_circuit(4, c.ops)
    hf = np.zeros(16)
    hf[0b1100] = 1
    assert np.allclose(psi, hf)                          # zero params -> Hartree-Fock state
    assert abs(O.expval(psi, 4, h2) - dense(h2, 4)[12, 12].real) < 1e-14
    with pytest.raises(C.ValidationError):
        C.singles_doubles_ansatz(4, 2, np.zeros(2))
