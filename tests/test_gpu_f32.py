"""GPU parity of the complex64 ("f32") instantiation (reference StateVector precision, state.py:20).

A complex64 handle runs the one-kernel-per-op gate kernels in FP32 (the reference casts the gate
matrix to the state dtype, state.py:264, 273) and accumulates every reduction in FP64.

Tolerances (float32 eps = 6e-8; the reference's own f32 norm tolerance is 1e-5, state.py:21):
* vs the reference's complex64 goldens (tests/golden/f32_golden.npz): |d| < 2e-6 per amplitude;
* vs the complex128 oracle after k gates: |d| < 1e-6 * sqrt(k) + 2e-6;
* expvals / variances / probabilities: |d| <= 1e-5 * max(1, ||O||_1);
* adjoint Jacobian entries: |d| <= 1e-4 * max(1, ||O||_1)  (two FP32 sweeps, ~100 gates);
* state I/O round trip: bit-exact complex64.
"""

import numpy as np
import pytest

from oracle import svoracle as O
from paper_2403_02512_b200 import errors, workloads
from paper_2403_02512_b200 import state as S
from paper_2403_02512_b200.device import Device
from paper_2403_02512_b200.observables import DenseHermitian, PauliWord
from paper_2403_02512_b200.ops import ARITY
from tests.golden_io import load
from tests.test_gpu_parity import KINDS, obs_norm1, rand_state, random_op

pytestmark = pytest.mark.gpu


def c64(v):
    return np.asarray(v).astype(np.complex64)


def test_f32_state_io_roundtrip_bit_exact():
    rng = np.random.default_rng(1)
    psi = c64(rand_state(rng, 12))
    with Device(12, precision="f32") as d:
        assert d.precision == "f32"
        d.set_state(psi)
        out = d.get_state()
        assert out.dtype == np.complex64
        assert np.array_equal(out.view(np.uint32), psi.view(np.uint32))
        assert abs(d.norm() - float(np.linalg.norm(psi.astype(np.complex128)))) < 1e-12


def test_f32_statevector_mirror():
    psi = c64(rand_state(np.random.default_rng(2), 5))
    sv = S.StateVector.from_amplitudes(psi)                 # complex64 input keeps f32 (state.py:56-60)
    assert sv.precision == "f32" and sv.dtype == np.complex64
    assert sv.amplitudes.dtype == np.complex64
    sv2 = S.StateVector.from_amplitudes(psi.astype(np.complex128))
    assert sv2.precision == "f64"
    z = S.zero_state(4, "f32")
    a = z.amplitudes
    assert a.dtype == np.complex64 and a[0] == 1 and not a[1:].any()
    assert z.copy().precision == "f32"


def test_f32_reference_golden_apply_matrix():
    d = load("f32_golden.npz")
    n = int(d["am_n"])
    for wires, psi, m, out in zip(d["am_wires"], d["am_in"], d["am_m"], d["am_out"]):
        w = [int(x) for x in wires if x >= 0]
        with Device(n, precision="f32") as dev:
            dev.set_state(psi)
            dev.apply_matrix(w, m[: 1 << len(w), : 1 << len(w)])
            got = dev.get_state()
        assert np.abs(got - out).max() < 2e-6, w


def test_f32_reference_golden_circuit():
    d = load("f32_golden.npz")
    n = int(d["circ_n"])
    ops = workloads.random_circuit(n, int(d["circ_depth"]), seed=int(d["circ_seed"]))
    with Device(n, precision="f32") as dev:
        dev.apply(ops)
        got = dev.get_state()
        assert dev.launch_count > 0
    assert np.abs(got - d["circ_out"]).max() < 1e-5


@pytest.mark.parametrize("kind", KINDS + ["Matrix", "ControlledMatrix"])
def test_f32_every_kind(kind):
    rng = np.random.default_rng(7 + sum(map(ord, kind)))
    n = 8
    psi = c64(rand_state(rng, n))
    for _ in range(4):
        op = random_op(rng, n, kind)
        ref = psi.astype(np.complex128)
        O.apply_op(ref, n, op)
        with Device(n, precision="f32") as d:
            d.set_state(psi)
            d.apply([op])          # fuse ignored: complex64 runs one kernel per op
            got = d.get_state()
        assert got.dtype == np.complex64
        assert np.abs(got - ref).max() < 3e-6, op


@pytest.mark.parametrize("n", [6, 14, 22])
def test_f32_random_circuits_vs_oracle(n):
    rng = np.random.default_rng(300 + n)
    ops = [random_op(rng, n) for _ in range(100)]
    psi = c64(rand_state(rng, n))
    ref = O.run_circuit(n, ops, psi.astype(np.complex128))
    with Device(n, precision="f32") as d:
        d.set_state(psi)
        d.apply(ops)
        got = d.get_state()
    assert np.abs(got - ref).max() < 1e-6 * np.sqrt(len(ops)) + 2e-6


def test_f32_measurements_vs_oracle():
    rng = np.random.default_rng(11)
    n = 10
    psi = c64(rand_state(rng, n))
    ref_psi = psi.astype(np.complex128)
    obs = [PauliWord(((0, "Z"), (3, "X"), (7, "Y"))), workloads.random_pauli_hamiltonian(n, 40, seed=3),
           DenseHermitian((4, 1), np.diag([1.0, -2.0, 0.5, 3.0]).astype(complex)),
           DenseHermitian((9, 0, 5, 2, 6), (lambda a: (a + a.conj().T) / 16)(
               rng.normal(size=(32, 32)) + 1j * rng.normal(size=(32, 32))))]   # 5 wires: scratch-buffer path
    with Device(n, precision="f32") as d:
        d.set_state(psi)
        for o in obs:
            tol = 1e-5 * max(1.0, obs_norm1(o))
            assert abs(d.expval(o) - O.expval(ref_psi, n, o)) <= tol
            assert abs(d.var(o) - O.variance(ref_psi, n, o)) <= 10 * tol
        for wires in ([0], [9, 2], [3, 1, 8], list(range(n))):
            assert np.abs(d.probs(wires) - O.probabilities(ref_psi, n, wires)).max() < 1e-6
        shots = d.sample_indices(2000, seed=5)
        assert shots.shape[0] == 2000 and shots.min() >= 0 and shots.max() < (1 << n)


@pytest.mark.parametrize("seed", range(2))
def test_f32_adjoint_vs_oracle(seed):
    rng = np.random.default_rng(500 + seed)
    n = 6
    kinds = ["RX", "RY", "RZ", "Phase", "Rot", "IsingXX", "IsingZZ", "SingleExcitation", "CNOT", "H", "CZ"]
    ops = []
    for _ in range(30):
        op = random_op(rng, n, kinds[int(rng.integers(len(kinds)))])
        op.inverse = False
        if ARITY[op.name][1]:
            op.trainable = tuple(bool(x) for x in rng.integers(0, 2, size=ARITY[op.name][1]))
        ops.append(op)
    obs = [PauliWord(((0, "Z"), (3, "X"))), workloads.random_pauli_hamiltonian(n, 12, seed=seed)]
    ref, ref_ev = O.adjoint_jacobian(n, ops, obs)
    with Device(n, precision="f32") as d:
        jac, ev = d.adjoint_jacobian(ops, obs, return_expvals=True)
    for k, o in enumerate(obs):
        tol = 1e-4 * max(1.0, obs_norm1(o))
        assert np.abs(jac[k] - ref[k]).max() <= tol, (k, np.abs(jac[k] - ref[k]).max())
        assert abs(ev[k] - ref_ev[k]) <= tol


def test_f32_sqrt2_kat_and_errors():
    with Device(1, precision="f32") as d:
        d.apply([("H", (0,))])
        st = d.get_state()
        assert abs(st[0] - np.float32(1 / np.sqrt(2))) < 1e-7
        with pytest.raises(errors.ValidationError):
            d.set_state(np.zeros(4, dtype=np.complex64))
    with pytest.raises(errors.UnsupportedOperationError):
        Device(4, precision="f32", _sharded=(0, 1, b"\0" * 128))
