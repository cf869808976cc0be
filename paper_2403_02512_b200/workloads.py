"""Seeded synthetic workloads for the BASELINE.json configs.

Pure host-side op-list builders (no arithmetic on amplitudes):

* ``strongly_entangling_layers`` -- SEL template: per layer a
  Rot on every qubit, then CNOT(i, (i + r) mod q). Config 1 (20q, L=4).
* ``random_circuit`` -- config 2/4: per layer each qubit gets RX/RY/RZ(theta),
  theta ~ U(0, 2pi), then a brickwork CNOT(q, q+1) for q = d (mod 2).
* ``qaoa_maxcut`` -- config 3: |+>^n, p layers of IsingZZ(2 gamma) per edge of a
  seeded random 4-regular graph and RX(2 beta) per qubit; C = sum 1/2 (1 - Z_i Z_j).
* ``hardware_efficient_ansatz`` + ``random_pauli_hamiltonian`` -- config 5.
"""

import numpy as np

from .observables import Hamiltonian, PauliWord
from .ops import Op


def strongly_entangling_layers(n_qubits, weights, r=1):
    """SEL circuit; ``weights`` has shape (L, n_qubits, 3)."""
    weights = np.asarray(weights, dtype=np.float64)
    if weights.ndim != 3 or weights.shape[1:] != (n_qubits, 3):
        raise ValueError(f"weights must have shape (L, {n_qubits}, 3), got {weights.shape}")
    ops = []
    for layer in weights:
        for q in range(n_qubits):
            ops.append(Op("Rot", (q,), tuple(layer[q]), trainable=(True, True, True)))
        if n_qubits > 1:
            for q in range(n_qubits):
                ops.append(Op("CNOT", (q, (q + r) % n_qubits)))
    return ops


def sel_config(n_qubits=20, layers=4, seed=0):
    """Config 1: SEL weights ~ U(0, 2pi) from default_rng(seed); observables Z_0..Z_{n-1}."""
    rng = np.random.default_rng(seed)
    w = rng.uniform(0, 2 * np.pi, size=(layers, n_qubits, 3))
    ops = strongly_entangling_layers(n_qubits, w)
    obs = [PauliWord(((q, "Z"),)) for q in range(n_qubits)]
    return ops, obs


def random_circuit(n_qubits, depth, seed=0, trainable=False):
    """Config 2 generator: 1q rotations on every qubit, then brickwork CNOTs, per layer."""
    rng = np.random.default_rng(seed)
    ops = []
    for d in range(depth):
        kinds = rng.integers(0, 3, size=n_qubits)
        thetas = rng.uniform(0, 2 * np.pi, size=n_qubits)
        for q in range(n_qubits):
            ops.append(Op(("RX", "RY", "RZ")[kinds[q]], (q,), (thetas[q],), trainable=(trainable,)))
        for q in range(d % 2, n_qubits - 1, 2):
            ops.append(Op("CNOT", (q, q + 1)))
    return ops


def random_regular_graph(degree, n, seed=0):
    """Seeded random d-regular simple graph (pairing model with restarts)."""
    if (degree * n) % 2:
        raise ValueError("degree * n must be even")
    rng = np.random.default_rng(seed)
    for _ in range(10000):
        stubs = np.repeat(np.arange(n), degree)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        edges = set()
        ok = True
        for a, b in pairs:
            a, b = int(min(a, b)), int(max(a, b))
            if a == b or (a, b) in edges:
                ok = False
                break
            edges.add((a, b))
        if ok:
            return sorted(edges)
    raise RuntimeError("could not build a simple regular graph")


def qaoa_maxcut(n_qubits, p=2, seed=0, degree=4):
    """Config 3: QAOA MaxCut ops (H layer + p x [IsingZZ per edge, RX per qubit]) and cost H."""
    edges = random_regular_graph(degree, n_qubits, seed)
    rng = np.random.default_rng(seed + 1)
    gammas = rng.uniform(0, np.pi, size=p)
    betas = rng.uniform(0, np.pi, size=p)
    ops = [Op("H", (q,)) for q in range(n_qubits)]
    for layer in range(p):
        for a, b in edges:
            ops.append(Op("IsingZZ", (a, b), (2 * gammas[layer],), trainable=(True,)))
        for q in range(n_qubits):
            ops.append(Op("RX", (q,), (2 * betas[layer],), trainable=(True,)))
    coeffs = [0.5 * len(edges)] + [-0.5] * len(edges)
    terms = [PauliWord(())] + [PauliWord(((a, "Z"), (b, "Z"))) for a, b in edges]
    return ops, Hamiltonian(coeffs, terms), edges


def hardware_efficient_ansatz(n_qubits, layers=18, n_trainable=1000, seed=0):
    """Config 5: layers x [RY, RZ on each qubit + CNOT ladder (q, q+1)]; first n_trainable params trainable."""
    rng = np.random.default_rng(seed)
    ops = []
    k = 0
    for _ in range(layers):
        for kind in ("RY", "RZ"):
            for q in range(n_qubits):
                ops.append(Op(kind, (q,), (rng.uniform(0, 2 * np.pi),), trainable=(k < n_trainable,)))
                k += 1
        for q in range(n_qubits - 1):
            ops.append(Op("CNOT", (q, q + 1)))
    return ops


def random_pauli_hamiltonian(n_qubits, n_terms, seed=0, max_weight=4):
    """Seeded random Pauli sum: weight 1..max_weight, coefficients N(0,1)/sqrt(T)."""
    rng = np.random.default_rng(seed)
    coeffs, terms = [], []
    for _ in range(n_terms):
        w = int(rng.integers(1, max_weight + 1))
        wires = rng.choice(n_qubits, size=min(w, n_qubits), replace=False)
        paulis = rng.choice(list("XYZ"), size=len(wires))
        terms.append(PauliWord(tuple((int(a), str(b)) for a, b in zip(wires, paulis))))
        coeffs.append(rng.normal() / np.sqrt(n_terms))
    return Hamiltonian(coeffs, terms)


def algorithmic_bytes(ops, n_qubits):
    """Unfused algorithmic HBM bytes of an op list.

    32 B x amplitudes read-and-written when unfused: dense 1q/2q/kq 2^(n+5);
    each control halves it; diagonal single-phase gates (Phase/S/T/Z) touch half,
    CZ a quarter; SWAP half.
    """
    full = 32 * (1 << n_qubits)
    total = 0
    for op in ops:
        b = full
        if op.name in ("Phase", "S", "T", "Z"):
            b //= 2
        elif op.name == "CZ":
            b //= 4
        elif op.name in ("CNOT", "SWAP"):
            b //= 2
        elif op.name == "I":
            b = 0
        total += b >> len(op.ctrls)
    return total
