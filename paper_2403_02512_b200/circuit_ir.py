"""Circuit / Hamiltonian text formats and workload templates (circuit-ir).

The SPEC's bespoke line grammar (no OpenQASM), versioned by a ``# format: 1`` header line;
files use the extensions ``.qc`` (circuit) and ``.ham`` (Hamiltonian).

Circuit grammar (EBNF; whitespace separates tokens, ``#`` starts a comment)::

    circuit   = [ "# format: 1" NL ] "qubits" INT NL { op NL } ;
    op        = [ "inv" ] [ ctrl ] KIND [ "(" REAL { "," REAL } ")" ] WIRE { WIRE } [ "train" ] ;
    ctrl      = "CTRL[" WIRE { "," WIRE } [ "=" BITS ] "]" ;      (* BITS aligned with the wires *)
    KIND      = "I" | "X" | "Y" | "Z" | "H" | "S" | "T" | "Phase" | "RX" | "RY" | "RZ" | "Rot"
              | "CNOT" | "CZ" | "SWAP" | "IsingXX" | "IsingXY" | "IsingYY" | "IsingZZ"
              | "SingleExcitation" | "DoubleExcitation" ;

``train`` marks every parameter of the op trainable; ``inv`` applies the adjoint. Examples:
``RX(0.3) 2``, ``CTRL[0,3=10] RZ(0.1) 2`` (controls 0 and 3 with values 1, 0), ``H 0``.

Hamiltonian grammar::

    hamiltonian = [ "# format: 1" NL ] { term NL } ;
    term        = REAL "[" [ PAULI WIRE { PAULI WIRE } ] "]" ;    (* e.g. -0.25 [X0 X1]; [] = identity *)

Errors are ``ParseError`` (a ``ValidationError``) carrying line, column and a caret line.
Everything here is host-side data plumbing in front of the device API; no amplitude math.
"""

import re
from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError
from .observables import Hamiltonian, PauliWord
from .ops import ARITY, Op

FORMAT_HEADER = "# format: 1"
_TEXT_KINDS = tuple(k for k in ARITY if k not in ("Matrix", "ControlledMatrix"))


class ParseError(ValidationError):
    def __init__(self, msg, line_no, col, line):
        self.line_no, self.col, self.line = line_no, col, line
        super().__init__(f"line {line_no}, column {col}: {msg}\n  {line}\n  {' ' * (col - 1)}^")


@dataclass
class Circuit:
    """``n_qubits`` + ordered ops."""

    n_qubits: int
    ops: list = field(default_factory=list)

    def __post_init__(self):
        for op in self.ops:
            for w in op.all_wires:
                if not 0 <= w < self.n_qubits:
                    raise ValidationError(f"wire {w} out of range for {self.n_qubits} qubits")

    @property
    def n_trainable(self):
        return sum(op.n_trainable for op in self.ops)

    def __eq__(self, other):
        if not isinstance(other, Circuit) or self.n_qubits != other.n_qubits or len(self.ops) != len(other.ops):
            return False
        return all((a.name, a.wires, a.params, a.ctrls, a.ctrl_values, a.trainable, a.inverse) ==
                   (b.name, b.wires, b.params, b.ctrls, b.ctrl_values, b.trainable, b.inverse)
                   for a, b in zip(self.ops, other.ops))


_OP_RE = re.compile(
    r"^(?P<inv>inv\s+)?(?:CTRL\[(?P<ctrl>[^\]]*)\]\s*)?(?P<kind>[A-Za-z]+)(?:\((?P<params>[^)]*)\))?"
    r"(?P<wires>(?:\s+\d+)+)(?P<train>\s+train)?\s*$")


def _strip(line):
    i = line.find("#")
    return line if i < 0 else line[:i]


def parse_circuit(text):
    """Parse the circuit format into a ``Circuit``."""
    lines = text.splitlines()
    n_qubits, ops = None, []
    for no, raw in enumerate(lines, start=1):
        line = _strip(raw).rstrip()
        if not line.strip():
            continue
        body = line.lstrip()
        col0 = len(line) - len(body) + 1
        if n_qubits is None:
            m = re.match(r"^qubits\s+(\d+)\s*$", body)
            if not m:
                raise ParseError("expected header 'qubits N'", no, col0, raw)
            n_qubits = int(m.group(1))
            if n_qubits < 1:
                raise ParseError("qubit count must be >= 1", no, col0 + body.index(m.group(1)), raw)
            continue
        if body.count("(") != body.count(")"):
            raise ParseError("unbalanced parenthesis", no, col0 + max(body.find("("), 0), raw)
        m = _OP_RE.match(body)
        if not m:
            raise ParseError("malformed operation", no, col0, raw)
        kind = m.group("kind")
        kcol = col0 + m.start("kind")
        if kind not in _TEXT_KINDS:
            raise ParseError(f"unknown gate {kind!r}", no, kcol, raw)
        params = ()
        if m.group("params") is not None:
            try:
                params = tuple(float(p) for p in m.group("params").split(",") if p.strip() != "")
            except ValueError:
                raise ParseError("malformed parameter list", no, col0 + m.start("params"), raw) from None
        wires = tuple(int(w) for w in m.group("wires").split())
        nw, npar = ARITY[kind]
        if len(wires) != nw or len(params) != npar:
            raise ParseError(f"{kind} takes {nw} wire(s) and {npar} parameter(s), got {len(wires)} and "
                             f"{len(params)}", no, kcol, raw)
        ctrls, cvals = (), ()
        if m.group("ctrl") is not None:
            spec = m.group("ctrl")
            ccol = col0 + m.start("ctrl")
            wpart, _, vpart = spec.partition("=")
            try:
                ctrls = tuple(int(c) for c in wpart.split(","))
            except ValueError:
                raise ParseError("malformed control spec", no, ccol, raw) from None
            if vpart:
                if len(vpart) != len(ctrls) or any(c not in "01" for c in vpart):
                    raise ParseError("control values must be one bit per control", no, ccol + len(wpart) + 1, raw)
                cvals = tuple(int(c) for c in vpart)
        for w in ctrls + wires:
            if not 0 <= w < n_qubits:
                raise ParseError(f"wire {w} out of range for {n_qubits} qubits", no, col0 + m.start("wires") + 1,
                                 raw)
        if len(set(ctrls + wires)) != len(ctrls + wires):
            raise ParseError("repeated wire", no, col0 + m.start("wires") + 1, raw)
        train = m.group("train") is not None
        if train and not params:
            raise ParseError(f"{kind} has no parameters to train", no, col0 + m.start("train") + 1, raw)
        ops.append(Op(kind, wires, params, ctrls=ctrls, ctrl_values=cvals, trainable=(train,) * len(params),
                      inverse=m.group("inv") is not None))
    if n_qubits is None:
        raise ParseError("missing header 'qubits N'", max(1, len(lines)), 1, lines[-1] if lines else "")
    return Circuit(n_qubits, ops)


def serialize_circuit(c):
    """Canonical text (parse_circuit(serialize_circuit(c)) == c; floats written with repr)."""
    out = [FORMAT_HEADER, f"qubits {c.n_qubits}"]
    for op in c.ops:
        if op.name not in _TEXT_KINDS:
            raise ValidationError(f"{op.name} has no text form")
        if op.trainable and len(set(op.trainable)) > 1:
            raise ValidationError("the text format marks all parameters of an op trainable or none")
        s = "inv " if op.inverse else ""
        if op.ctrls:
            s += "CTRL[" + ",".join(map(str, op.ctrls))
            if any(v != 1 for v in op.ctrl_values):
                s += "=" + "".join(map(str, op.ctrl_values))
            s += "] "
        s += op.name
        if op.params:
            s += "(" + ",".join(repr(float(p)) for p in op.params) + ")"
        s += " " + " ".join(map(str, op.wires))
        if op.trainable and op.trainable[0]:
            s += " train"
        out.append(s)
    return "\n".join(out) + "\n"


_TERM_RE = re.compile(r"^(?P<coeff>\S+)\s*\[(?P<body>[^\]]*)\]\s*$")
_FACTOR_RE = re.compile(r"^([XYZI])(\d+)$")


def parse_hamiltonian(text, n_qubits=None):
    """``<coeff> [P<w> P<w> ...]`` per line into a Hamiltonian."""
    coeffs, terms = [], []
    lines = text.splitlines()
    for no, raw in enumerate(lines, start=1):
        line = _strip(raw).rstrip()
        if not line.strip():
            continue
        body = line.lstrip()
        col0 = len(line) - len(body) + 1
        m = _TERM_RE.match(body)
        if not m:
            raise ParseError("expected '<coeff> [P<w> ...]'", no, col0, raw)
        try:
            c = float(m.group("coeff"))
        except ValueError:
            raise ParseError("malformed coefficient", no, col0, raw) from None
        factors, seen = [], set()
        pos = col0 + m.start("body")
        for tok in m.group("body").split():
            tcol = pos + m.group("body").index(tok)
            fm = _FACTOR_RE.match(tok)
            if not fm:
                raise ParseError(f"malformed Pauli token {tok!r}", no, tcol, raw)
            p, w = fm.group(1), int(fm.group(2))
            if w in seen:
                raise ParseError(f"duplicate wire {w} within a term", no, tcol, raw)
            if n_qubits is not None and w >= n_qubits:
                raise ParseError(f"wire {w} out of range for {n_qubits} qubits", no, tcol, raw)
            seen.add(w)
            if p != "I":
                factors.append((w, p))
        coeffs.append(c)
        terms.append(PauliWord(tuple(factors)))
    return Hamiltonian(tuple(coeffs), tuple(terms))


def serialize_hamiltonian(h):
    out = [FORMAT_HEADER]
    for c, t in zip(h.coeffs, h.terms):
        out.append(f"{c!r} [" + " ".join(f"{p}{w}" for w, p in t.factors) + "]")
    return "\n".join(out) + "\n"


def strongly_entangling_layers(n_qubits, layers, params, r=1, trainable=True):
    """SEL template: per layer Rot(3 params) on every qubit, then CNOT(i, (i+r) % q)."""
    p = np.asarray(params, dtype=np.float64)
    if p.shape != (layers, n_qubits, 3):
        raise ValidationError(f"SEL params must have shape {(layers, n_qubits, 3)}, got {p.shape}")
    ops = []
    for layer in range(layers):
        for q in range(n_qubits):
            ops.append(Op("Rot", (q,), tuple(p[layer, q]), trainable=(trainable,) * 3))
        if n_qubits > 1:
            for q in range(n_qubits):
                ops.append(Op("CNOT", (q, (q + r) % n_qubits)))
    return Circuit(n_qubits, ops)


def excitations(n_qubits, electrons):
    """Spin-conserving excitations from the Hartree-Fock occupation (wires 0..electrons-1 occupied;
    spin orbital i has spin i % 2): singles (r, p) ascending, then doubles (r, s, p, q)."""
    if not 0 <= electrons <= n_qubits:
        raise ValidationError("electrons must be between 0 and n_qubits")
    occ, virt = range(electrons), range(electrons, n_qubits)
    singles = [(r, p) for r in occ for p in virt if r % 2 == p % 2]
    doubles = [(r, s, p, q) for r in occ for s in occ if r < s for p in virt for q in virt if p < q
               and (r % 2) + (s % 2) == (p % 2) + (q % 2)]
    return singles, doubles


def singles_doubles_ansatz(n_qubits, electrons, params, trainable=True):
    """Hartree-Fock preparation + SingleExcitation / DoubleExcitation on every valid excitation
    (SPEC.md:533-541)."""
    singles, doubles = excitations(n_qubits, electrons)
    p = np.atleast_1d(np.asarray(params, dtype=np.float64))
    if len(p) != len(singles) + len(doubles):
        raise ValidationError(f"expected {len(singles) + len(doubles)} parameters "
                              f"({len(singles)} singles + {len(doubles)} doubles), got {len(p)}")
    ops = [Op("X", (w,)) for w in range(electrons)]
    k = 0
    for ex in singles:
        ops.append(Op("SingleExcitation", ex, (p[k],), trainable=(trainable,)))
        k += 1
    for ex in doubles:
        ops.append(Op("DoubleExcitation", ex, (p[k],), trainable=(trainable,)))
        k += 1
    return Circuit(n_qubits, ops)
