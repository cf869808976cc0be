"""Small fused workloads for compute-sanitizer (racecheck / synccheck / memcheck): a random circuit
and a fused adjoint sweep at 13-14 qubits through the generated pass kernels (svb200_pass) or, with
SVB200_JIT=0, the op-interpreting k_fused; checked against the oracle so a silent race shows too.

    compute-sanitizer --tool racecheck python benchmarks/sanitize_fused.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import svoracle as O  # noqa: E402
from paper_2403_02512_b200 import workloads  # noqa: E402
from paper_2403_02512_b200.device import Device  # noqa: E402

n = int(os.environ.get("SAN_N", "14"))
ops = workloads.random_circuit(n, 4, seed=3)
with Device(n) as d:
    d.apply(ops)
    err = float(np.abs(d.get_state() - O.run_circuit(n, ops)).max())
    qops, ham, _ = workloads.qaoa_maxcut(n, p=1, seed=2)
    d.reset()
    jac = d.adjoint_jacobian(qops, [ham])
    jref, _ = O.adjoint_jacobian(n, qops, [ham])
    jerr = float(np.abs(jac - jref).max())
print(f"sanitize_fused n={n} jit={os.environ.get('SVB200_JIT', '1')} pp={os.environ.get('SVB200_JIT_PP', '0')} "
      f"state_err={err:.2e} jac_err={jerr:.2e}")
assert err < 1e-12 and jerr < 1e-10
