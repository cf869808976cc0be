"""TEST INFRASTRUCTURE (checker only): closed-form p = 1 QAOA MaxCut expectation.

Wang, Hadfield, Jiang, Rieffel, "Quantum approximate optimization algorithm for MaxCut: a
fermionic view", Phys. Rev. A 97, 022304 (2018), Thm. 1: for U_C = exp(-i gamma C),
C = sum_(u,v) (1 - Z_u Z_v) / 2, U_B = exp(-i beta sum X) on |+>^n,

  <C_uv> = 1/2 + 1/4 sin(4 beta) sin(gamma) (cos^d_u gamma + cos^d_v gamma)
               - 1/4 sin^2(2 beta) cos^(d_u + d_v - 2 l_uv) gamma (1 - cos^l_uv (2 gamma))

with d_u = deg(u) - 1, d_v = deg(v) - 1 and l_uv the number of triangles on edge (u, v).  Not in the
reference (SURVEY §8(d) config 3 names it as a size-independent parity check for 33 qubits, where
no CPU state vector fits).  The circuit of workloads.qaoa_maxcut applies IsingZZ(2 g) =
exp(-i g Z Z) per edge, i.e. exp(-i gamma C) up to a global phase with gamma = -2 g, and
RX(2 b) = exp(-i b X), i.e. beta = b; tests/test_oracle.py pins this mapping against the oracle.
"""

import numpy as np


def maxcut_p1_expectation(n_qubits, edges, g, b):
    """<C> after H^n, IsingZZ(2 g) on every edge, RX(2 b) on every qubit (workloads.qaoa_maxcut, p=1)."""
    gamma, beta = -2.0 * g, b
    nbr = [set() for _ in range(n_qubits)]
    for u, v in edges:
        nbr[u].add(v)
        nbr[v].add(u)
    total = 0.0
    for u, v in edges:
        du, dv = len(nbr[u]) - 1, len(nbr[v]) - 1
        lam = len(nbr[u] & nbr[v])
        c = np.cos(gamma)
        total += (0.5 + 0.25 * np.sin(4 * beta) * np.sin(gamma) * (c ** du + c ** dv)
                  - 0.25 * np.sin(2 * beta) ** 2 * c ** (du + dv - 2 * lam) * (1 - np.cos(2 * gamma) ** lam))
    return float(total)
