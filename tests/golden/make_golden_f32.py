"""complex64 ("f32") golden vectors from the REAL reference (run in the build container only).

    python tests/golden/make_golden_f32.py

The reference's StateVector has a complex64 instantiation (state.py:20); its apply_matrix
casts the gate matrix to the state dtype before the contraction (state.py:264, 273), so every
update is complex64 arithmetic.  This script records, for seeded inputs:

* ``am_*``: apply_matrix on a complex64 state, w = 1..6 (the <=4-wire gather path and the
  general transpose path), random unitaries;
* ``circ_*``: a random RX/RY/RZ/CNOT circuit (the BASELINE config-2 generator at n = 10,
  depth 8) with every gate executed by the reference's apply_matrix on a complex64 state.

Writes tests/golden/f32_golden.npz; /root/reference is never read at test time.
"""

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


def rand_state64(rng, n):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return (v / np.linalg.norm(v)).astype(np.complex64)


def rand_unitary(rng, d):
    z = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def main():
    rng = np.random.default_rng(32)
    out = {}
    n = 7
    am_wires, am_in, am_m, am_out = [], [], [], []
    for w in range(1, 7):
        for _ in range(3):
            wires = [int(x) for x in rng.choice(n, size=w, replace=False)]
            psi = rand_state64(rng, n)
            m = rand_unitary(rng, 1 << w)
            sv = ref.StateVector.from_amplitudes(psi)
            assert sv.precision == "f32"
            ref.apply_matrix(sv, wires, m)
            am_wires.append(wires + [-1] * (6 - w))
            am_in.append(psi)
            am_m.append(np.pad(m, ((0, 64 - (1 << w)), (0, 64 - (1 << w)))))
            am_out.append(sv.amplitudes.copy())
    out["am_n"] = np.array(n)
    out["am_wires"] = np.array(am_wires, dtype=np.int32)
    out["am_in"] = np.array(am_in)
    out["am_m"] = np.array(am_m)
    out["am_out"] = np.array(am_out)

    nc, depth = 10, 8
    ops = workloads.random_circuit(nc, depth, seed=5)
    sv = ref.zero_state(nc, "f32")
    for op in ops:
        m = svoracle.base_matrix(op)
        ctrls = tuple(op.ctrls)
        vals = tuple(op.ctrl_values) if op.ctrl_values else (1,) * len(ctrls)
        ref.apply_matrix(sv, list(ctrls) + list(op.wires), svoracle._controlled(m, len(ctrls), vals))
    assert sv.amplitudes.dtype == np.complex64
    out["circ_n"] = np.array(nc)
    out["circ_depth"] = np.array(depth)
    out["circ_seed"] = np.array(5)
    out["circ_out"] = sv.amplitudes.copy()
    np.savez_compressed(os.path.join(HERE, "f32_golden.npz"), **out)
    print("wrote f32_golden.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
