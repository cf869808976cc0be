"""Observable batching: the chunk plan on CPU; pooled GPU workers vs the
unbatched adjoint (GPU)."""

import numpy as np
import pytest

from paper_2403_02512_b200 import errors, workloads
from paper_2403_02512_b200.batching import batched_expval_and_grad, plan_chunks


def test_plan_partition_rules():
    sizes = [len(idx) for _, idx in plan_chunks(9, 4)]
    assert sizes == [3, 2, 2, 2]
    assert sum(1 for _, idx in plan_chunks(1, 5) if idx) == 1
    plan = plan_chunks(10, 3, batch_size=4)
    assert [idx for _, idx in plan] == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9]]
    assert [w for w, _ in plan] == [0, 1, 2]
    covered = sorted(i for _, idx in plan_chunks(1000, 7) for i in idx)
    assert covered == list(range(1000))
    with pytest.raises(errors.ValidationError):
        plan_chunks(3, 0)                                          # g == 0 -> validation error


def test_canonical_chunks_depend_on_the_hamiltonian_only():
    from paper_2403_02512_b200.batching import canonical_chunks
    assert [len(c) for c in canonical_chunks(9)] == [2, 1, 1, 1, 1, 1, 1, 1]
    assert [len(c) for c in canonical_chunks(40)] == [5] * 8
    assert canonical_chunks(3) == [[0], [1], [2]]
    assert sorted(i for c in canonical_chunks(1000) for i in c) == list(range(1000))


@pytest.mark.gpu
def test_batching_bit_identical_across_workers_and_batch_sizes():
    """energy/gradient bit-identical for g in {1,2,4,8} and b in {1,3,n}."""
    n = 12
    ops = workloads.hardware_efficient_ansatz(n, layers=3, n_trainable=60, seed=11)
    ham = workloads.random_pauli_hamiltonian(n, 40, seed=11)
    ref = None
    for g in (1, 2, 4, 8):
        for b in (None, 1, 3, 40):
            e, grad = batched_expval_and_grad(ops, ham, n_workers=g, batch_size=b, n_qubits=n)
            if ref is None:
                ref = (e, grad)
            assert e == ref[0] and (grad == ref[1]).all(), (g, b)


@pytest.mark.gpu
def test_batched_matches_unbatched():
    from paper_2403_02512_b200.device import Device
    n = 12
    ops = workloads.hardware_efficient_ansatz(n, layers=3, n_trainable=60, seed=7)
    ham = workloads.random_pauli_hamiltonian(n, 40, seed=7)
    with Device(n) as d:
        jac, ev = d.adjoint_jacobian(ops, [ham], return_expvals=True)
    ref_e, ref_g = float(ev[0]), jac[0]
    results = [batched_expval_and_grad(ops, ham, n_workers=g, batch_size=b, n_qubits=n)
               for g, b in ((1, None), (4, None), (3, 5), (2, 1))]
    for e, g in results:
        assert abs(e - ref_e) < 1e-12
        assert np.abs(g - ref_g).max() < 1e-12
    e1, g1 = batched_expval_and_grad(ops, ham, n_workers=4, n_qubits=n)
    assert e1 == results[1][0] and (g1 == results[1][1]).all()     # bit-identical for fixed (g, b)
