"""CPU: the C port of Alg. 1 / Alg. 2 (oracle/c/svport.c, the bench's CPU baseline) agrees with
the numpy oracle, which is itself pinned to the reference's golden vectors."""

import numpy as np

from oracle import cport
from oracle import svoracle as O
from paper_2403_02512_b200 import workloads
from paper_2403_02512_b200.ops import Op


def test_cport_matches_oracle_random_circuit():
    n = 12
    ops = workloads.random_circuit(n, 6, seed=2)
    rng = np.random.default_rng(0)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    ref = O.run_circuit(n, ops, psi)
    got = psi.copy()
    for op in ops:
        cport.apply_op(got, n, op)
    assert np.abs(got - ref).max() < 1e-13


def test_cport_controlled_values():
    n = 7
    rng = np.random.default_rng(1)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    for ctrls, vals, q in [((0,), (0,), 6), ((6, 2), (1, 0), 3), ((1, 5, 3), (0, 1, 1), 0)]:
        m = np.linalg.qr(rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2)))[0]
        ref = psi.copy()
        O.apply_controlled_single_qubit(ref, n, ctrls, q, m, vals)
        got = psi.copy()
        cport.apply_ctrl_1q(got, n, ctrls, vals, q, m)
        assert np.abs(got - ref).max() < 1e-13
