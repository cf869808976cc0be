"""Time expval of the config-5 Hamiltonian (28 qubits, 1000 random Pauli terms) on the HEA state."""
import sys
import time
sys.path.insert(0, ".")
from paper_2403_02512_b200 import workloads  # noqa: E402
from paper_2403_02512_b200.device import Device  # noqa: E402
n = 28
ops = workloads.hardware_efficient_ansatz(n, layers=18, n_trainable=1000, seed=0)
ham = workloads.random_pauli_hamiltonian(n, 1000, seed=0)
with Device(n) as d:
    d.apply(ops)
    e = d.expval(ham)
    ts = []
    for _ in range(3):
        d.synchronize()
        t0 = time.perf_counter()
        e = d.expval(ham)
        ts.append(time.perf_counter() - t0)
    print({"s_expval": min(ts), "expval": e})
