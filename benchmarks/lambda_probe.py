import sys; sys.path.insert(0, ".")
from paper_2403_02512_b200 import workloads
from paper_2403_02512_b200.device import Device
n = 28
ops = workloads.hardware_efficient_ansatz(n, layers=18, n_trainable=1000, seed=0)
ham = workloads.random_pauli_hamiltonian(n, 1000, seed=0)
with Device(n) as d:
    d.apply(ops)
    for _ in range(2):
        d.expval(ham)
    d.synchronize()
