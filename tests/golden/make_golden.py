"""Generate golden vectors from the REAL reference (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--sel20]

Imports ``svkit.state`` from /root/reference (read-only) and records, for seeded
inputs, the outputs of the reference's own ``get_masks`` (state.py:128),
``apply_single_qubit`` (Alg. 1, state.py:154), ``apply_controlled_single_qubit``
(Alg. 2, state.py:192) and ``apply_matrix`` (state.py:278, both the <=4-wire
gather path and the general transpose path).

Circuit-level goldens (named gates, expvals, adjoint Jacobians) are produced by
the oracle's restated algorithm with its gate primitives REPLACED by the
reference's ``apply_matrix`` / Alg. 1 / Alg. 2, so every amplitude update in
those vectors is the reference's own arithmetic.
``--sel20`` additionally runs config 1 (20-qubit SEL, L=4, 20 x 240 Jacobian)
which takes several minutes.

The vectors are committed as tests/golden/*.npz; /root/reference is never read
at test time.
"""

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import svkit.state as ref  # noqa: E402  (the reference, read-only)

from oracle import svoracle  # noqa: E402
from paper_2403_02512_b200 import workloads  # noqa: E402
from paper_2403_02512_b200.observables import DenseHermitian, Hamiltonian, PauliWord  # noqa: E402
from paper_2403_02512_b200.ops import Op  # noqa: E402


def rand_state(rng, n):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def rand_unitary(rng, d):
    z = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def interaction(m):
    """A CoefficientInteraction f(amps, i0, i1) for a 2x2 matrix."""
    def f(amps, i0, i1):
        a0, a1 = amps[i0], amps[i1]
        amps[i0] = m[0, 0] * a0 + m[0, 1] * a1
        amps[i1] = m[1, 0] * a0 + m[1, 1] * a1
    return f


def ref_sv(amps):
    return ref.StateVector.from_amplitudes(np.array(amps, dtype=np.complex128))


# --- reference-backed primitives patched into the oracle -------------------

def _ref_apply_matrix(amps, n, wires, matrix):
    sv = ref.StateVector.from_amplitudes(amps, copy=False)
    ref.apply_matrix(sv, wires, matrix)


def _ref_apply_single_qubit(amps, n, q, m):
    _ref_apply_matrix(amps, n, (q,), m)        # vectorised reference path (Alg. 1 loop is ~2 us/pair)


def _ref_apply_controlled(amps, n, ctrls, q, m, ctrl_values=None):
    vals = tuple(ctrl_values) if ctrl_values else (1,) * len(ctrls)
    full = svoracle._controlled(m, len(ctrls), vals)
    _ref_apply_matrix(amps, n, tuple(ctrls) + (q,), full)


def patch_oracle_with_reference():
    svoracle.apply_matrix = _ref_apply_matrix
    svoracle.apply_single_qubit = _ref_apply_single_qubit
    svoracle.apply_controlled_single_qubit = _ref_apply_controlled


# ---------------------------------------------------------------------------

def kernel_goldens(rng):
    out = {}
    # get_masks (state.py:128-151)
    masks = []
    for n in range(1, 9):
        for k in range(0, min(n, 4) + 1):
            excl = sorted(rng.choice(n, size=k, replace=False).tolist())
            ms = ref.get_masks(excl, n)
            masks.append((n, excl, list(ms.masks), list(ms.strides)))
    out["masks_repr"] = np.array(repr(masks))

    # Alg. 1 on the real per-pair loop, every q, n <= 7
    cases = []
    for n in range(1, 8):
        for q in range(n):
            psi = rand_state(rng, n)
            m = rand_unitary(rng, 2)
            sv = ref_sv(psi)
            ref.apply_single_qubit(sv, q, interaction(m))
            cases.append((n, q, psi, m, sv.amplitudes.copy()))
    out["alg1_n"] = np.array([c[0] for c in cases])
    out["alg1_q"] = np.array([c[1] for c in cases])
    out["alg1_in"] = np.array([np.pad(c[2], (0, 128 - len(c[2]))) for c in cases])
    out["alg1_m"] = np.array([c[3] for c in cases])
    out["alg1_out"] = np.array([np.pad(c[4], (0, 128 - len(c[4]))) for c in cases])

    # Alg. 2 with random controls and control values, n <= 7
    cases = []
    for _ in range(60):
        n = int(rng.integers(2, 8))
        nc = int(rng.integers(1, min(3, n - 1) + 1))
        qs = rng.choice(n, size=nc + 1, replace=False).tolist()
        q, ctrls = qs[0], qs[1:]
        vals = rng.integers(0, 2, size=nc).tolist()
        psi = rand_state(rng, n)
        m = rand_unitary(rng, 2)
        sv = ref_sv(psi)
        ref.apply_controlled_single_qubit(sv, ctrls, q, interaction(m), ctrl_values=vals)
        cases.append((n, q, ctrls + [-1] * (3 - nc), vals + [-1] * (3 - nc), psi, m, sv.amplitudes.copy()))
    out["alg2_n"] = np.array([c[0] for c in cases])
    out["alg2_q"] = np.array([c[1] for c in cases])
    out["alg2_ctrls"] = np.array([c[2] for c in cases])
    out["alg2_vals"] = np.array([c[3] for c in cases])
    out["alg2_in"] = np.array([np.pad(c[4], (0, 128 - len(c[4]))) for c in cases])
    out["alg2_m"] = np.array([c[5] for c in cases])
    out["alg2_out"] = np.array([np.pad(c[6], (0, 128 - len(c[6]))) for c in cases])

    # apply_matrix, w = 1..6 (gather path w<=4, general path w>=5), n <= 9, incl. non-unitary
    cases = []
    for _ in range(60):
        n = int(rng.integers(1, 10))
        w = int(rng.integers(1, min(n, 6) + 1))
        wires = rng.choice(n, size=w, replace=False).tolist()
        psi = rand_state(rng, n)
        if rng.random() < 0.25:
            m = rng.normal(size=(1 << w, 1 << w)) + 1j * rng.normal(size=(1 << w, 1 << w))
        else:
            m = rand_unitary(rng, 1 << w)
        sv = ref_sv(psi)
        ref.apply_matrix(sv, wires, m)
        cases.append((n, wires + [-1] * (6 - w), psi, m.reshape(-1), sv.amplitudes.copy()))
    out["mat_n"] = np.array([c[0] for c in cases])
    out["mat_wires"] = np.array([c[1] for c in cases])
    out["mat_in"] = np.array([np.pad(c[2], (0, 512 - len(c[2]))) for c in cases])
    out["mat_m_flat"] = np.concatenate([c[3] for c in cases])
    out["mat_m_off"] = np.cumsum([0] + [len(c[3]) for c in cases])
    out["mat_out"] = np.array([np.pad(c[4], (0, 512 - len(c[4]))) for c in cases])
    return out


def named_gate_ops(rng, n, count):
    """Random ops over every named kind, with random extra controls and inverses."""
    kinds = ["I", "X", "Y", "Z", "H", "S", "T", "Phase", "RX", "RY", "RZ", "Rot", "CNOT", "CZ",
             "SWAP", "IsingXX", "IsingXY", "IsingYY", "IsingZZ", "SingleExcitation",
             "DoubleExcitation", "Matrix", "ControlledMatrix"]
    from paper_2403_02512_b200.ops import ARITY
    ops = []
    while len(ops) < count:
        k = kinds[int(rng.integers(len(kinds)))]
        nw, npar = ARITY[k]
        if nw is None:
            nw = int(rng.integers(1, 4))
        ncmax = n - nw
        if ncmax < 0:
            continue
        nc = int(rng.integers(0, min(2, ncmax) + 1)) if (k == "ControlledMatrix" or rng.random() < 0.3) else 0
        qs = rng.choice(n, size=nw + nc, replace=False).tolist()
        params = tuple(rng.uniform(-np.pi, np.pi, size=npar or 0))
        m = rand_unitary(rng, 1 << nw) if k in ("Matrix", "ControlledMatrix") else None
        ops.append(Op(k, tuple(qs[:nw]), params, ctrls=tuple(qs[nw:]),
                      ctrl_values=tuple(int(v) for v in rng.integers(0, 2, size=nc)),
                      inverse=bool(rng.random() < 0.2), matrix=m))
    return ops


def pack_ops(ops):
    """Serialise an op list into plain arrays for the npz."""
    recs = []
    mats = []
    for op in ops:
        recs.append(repr((op.name, op.wires, op.params, op.ctrls, op.ctrl_values, op.trainable, op.inverse,
                          len(mats) if op.matrix is not None else -1)))
        if op.matrix is not None:
            mats.append(op.matrix)
    return np.array(recs), mats


def pack_obs(obs):
    recs, mats = [], []
    for o in obs:
        if isinstance(o, PauliWord):
            recs.append(repr(("pauli", o.factors)))
        elif isinstance(o, Hamiltonian):
            recs.append(repr(("ham", o.coeffs, tuple(t.factors for t in o.terms))))
        else:
            recs.append(repr(("dense", o.wires, len(mats))))
            mats.append(o.matrix)
    return np.array(recs), mats


def circuit_goldens(rng):
    out = {}
    # random named-gate circuits (state after each circuit)
    for i, n in enumerate([4, 5, 6, 7]):
        ops = named_gate_ops(rng, n, 40)
        psi0 = rand_state(rng, n)
        psi = svoracle.run_circuit(n, ops, psi0)
        recs, mats = pack_ops(ops)
        out[f"circ{i}_n"] = np.array(n)
        out[f"circ{i}_ops"] = recs
        for j, m in enumerate(mats):
            out[f"circ{i}_mat{j}"] = m
        out[f"circ{i}_in"] = psi0
        out[f"circ{i}_out"] = psi

    # adjoint Jacobians: SEL n=6 L=2 (SPEC.md:461-463 shape), random param circuits, QAOA n=8
    jobs = []
    w = rng.uniform(0, 2 * np.pi, size=(2, 6, 3))
    ops = workloads.strongly_entangling_layers(6, w)
    obs = [PauliWord(((q, "Z"),)) for q in range(6)] + [
        Hamiltonian([0.3, -1.2, 0.7], [PauliWord(((0, "X"), (2, "Y"))), PauliWord(((1, "Z"),)),
                                       PauliWord(((3, "Y"), (4, "X"), (5, "Z")))])]
    jobs.append(("sel6", 6, ops, obs))
    par_kinds = ["RX", "RY", "RZ", "Phase", "IsingXX", "IsingXY", "IsingYY", "IsingZZ",
                 "SingleExcitation", "DoubleExcitation", "Rot", "CNOT", "H", "CZ"]
    from paper_2403_02512_b200.ops import ARITY
    for t in range(3):
        n = 5
        ops = []
        for _ in range(25):
            k = par_kinds[int(rng.integers(len(par_kinds)))]
            nw, npar = ARITY[k]
            nc = 1 if (nw == 1 and rng.random() < 0.25) else 0
            qs = rng.choice(n, size=nw + nc, replace=False).tolist()
            ops.append(Op(k, tuple(qs[:nw]), tuple(rng.uniform(-np.pi, np.pi, size=npar)), ctrls=tuple(qs[nw:]),
                          trainable=(True,) * npar, inverse=bool(rng.random() < 0.2)))
        herm = rand_unitary(rng, 4)
        herm = herm + herm.conj().T
        obs = [PauliWord(((0, "Z"), (1, "Z"))), PauliWord(((2, "X"),)),
               DenseHermitian((3, 1), herm)]
        jobs.append((f"rand{t}", n, ops, obs))
    qops, ham, _ = workloads.qaoa_maxcut(8, p=2, seed=0)
    jobs.append(("qaoa8", 8, qops, [ham]))
    for name, n, ops, obs in jobs:
        print(f"  adjoint {name} n={n} ops={len(ops)} obs={len(obs)}", flush=True)
        jac, ev = svoracle.adjoint_jacobian(n, ops, obs)
        recs, mats = pack_ops(ops)
        out[f"adj_{name}_n"] = np.array(n)
        out[f"adj_{name}_ops"] = recs
        for j, m in enumerate(mats):
            out[f"adj_{name}_mat{j}"] = m
        orecs, omats = pack_obs(obs)
        out[f"adj_{name}_obs"] = orecs
        for j, m in enumerate(omats):
            out[f"adj_{name}_omat{j}"] = m
        out[f"adj_{name}_jac"] = jac
        out[f"adj_{name}_expvals"] = ev
        if n <= 8:
            psi = svoracle.run_circuit(n, ops)
            out[f"adj_{name}_probs_all"] = svoracle.probabilities(psi, n)
            out[f"adj_{name}_probs_w"] = svoracle.probabilities(psi, n, [n - 1, 0])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sel20", action="store_true")
    args = ap.parse_args()
    rng = np.random.default_rng(20240302)
    kg = kernel_goldens(rng)
    np.savez_compressed(os.path.join(HERE, "state_golden.npz"), **kg)
    print("wrote state_golden.npz")
    patch_oracle_with_reference()
    cg = circuit_goldens(rng)
    np.savez_compressed(os.path.join(HERE, "circuit_golden.npz"), **cg)
    print("wrote circuit_golden.npz")
    if args.sel20:
        ops, obs = workloads.sel_config(20, 4, seed=0)
        jac, ev = svoracle.adjoint_jacobian(20, ops, obs)
        np.savez_compressed(os.path.join(HERE, "sel20_golden.npz"), jac=jac, expvals=ev)
        print("wrote sel20_golden.npz")


if __name__ == "__main__":
    main()
