"""GPU parity: libsvb200 (through the C-ABI) vs the reference's golden vectors and the oracle.

Tolerances (SURVEY.md §8(d) / SPEC.md:681-686): states |d| < 1e-12 elementwise; expvals and
Jacobian entries |d| <= 1e-10 * max(|ref|, ||O||_1) with ||O||_1 = sum |c_t|.
"""

import ast

import numpy as np
import pytest

from oracle import svoracle as O
from paper_2403_02512_b200 import errors, workloads
from paper_2403_02512_b200.device import Device
from paper_2403_02512_b200.observables import DenseHermitian, Hamiltonian, PauliWord
from paper_2403_02512_b200.ops import ARITY, Op
from tests.golden_io import ADJ_JOBS, load, unpack_obs, unpack_ops

pytestmark = pytest.mark.gpu

STATE_TOL = 1e-12


def obs_norm1(o):
    if isinstance(o, Hamiltonian):
        return sum(abs(c) for c in o.coeffs)
    if isinstance(o, DenseHermitian):
        return float(np.abs(np.linalg.eigvalsh(o.matrix)).max())
    return 1.0


def assert_grad_close(got, ref, obs):
    for k, o in enumerate(obs):
        scale = max(obs_norm1(o), float(np.abs(ref[k]).max()) if ref[k].size else 1.0)
        assert np.abs(got[k] - ref[k]).max() <= 1e-10 * scale, (k, np.abs(got[k] - ref[k]).max())


def rand_state(rng, n):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


@pytest.fixture(scope="module")
def sg():
    return load("state_golden.npz")


@pytest.fixture(scope="module")
def cg():
    return load("circuit_golden.npz")


# ---- reference golden vectors through the reference-shaped API (state.py mirror) -----------

def test_alg1_golden_via_state_api(sg):
    from paper_2403_02512_b200 import state as S
    for n, q, psi, m, out in zip(sg["alg1_n"], sg["alg1_q"], sg["alg1_in"], sg["alg1_m"], sg["alg1_out"]):
        sv = S.StateVector.from_amplitudes(psi[: 1 << n])
        S.apply_single_qubit(sv, int(q), S.CoefficientInteraction(m))
        assert np.abs(sv.amplitudes - out[: 1 << n]).max() < STATE_TOL


def test_alg2_golden_via_state_api(sg):
    from paper_2403_02512_b200 import state as S
    for i in range(len(sg["alg2_n"])):
        n, q = int(sg["alg2_n"][i]), int(sg["alg2_q"][i])
        ctrls = [int(c) for c in sg["alg2_ctrls"][i] if c >= 0]
        vals = [int(v) for v in sg["alg2_vals"][i] if v >= 0]
        sv = S.StateVector.from_amplitudes(sg["alg2_in"][i][: 1 << n])
        S.apply_controlled_single_qubit(sv, ctrls, q, S.CoefficientInteraction(sg["alg2_m"][i]), vals)
        assert np.abs(sv.amplitudes - sg["alg2_out"][i][: 1 << n]).max() < STATE_TOL


def test_apply_matrix_golden_via_state_api(sg):
    from paper_2403_02512_b200 import state as S
    off = sg["mat_m_off"]
    for i in range(len(sg["mat_n"])):
        n = int(sg["mat_n"][i])
        wires = [int(w) for w in sg["mat_wires"][i] if w >= 0]
        d = 1 << len(wires)
        m = sg["mat_m_flat"][off[i]:off[i + 1]].reshape(d, d)
        sv = S.StateVector.from_amplitudes(sg["mat_in"][i][: 1 << n])
        S.apply_matrix(sv, wires, m)
        ref = sg["mat_out"][i][: 1 << n]
        assert np.abs(sv.amplitudes - ref).max() < 1e-12 * max(1.0, np.abs(ref).max())


def test_state_api_errors():
    from paper_2403_02512_b200 import state as S
    sv = S.zero_state(3)
    with pytest.raises(errors.ValidationError):
        S.apply_single_qubit(sv, 3, S.CoefficientInteraction(np.eye(2)))
    with pytest.raises(errors.ValidationError):
        S.apply_controlled_single_qubit(sv, [1, 1], 0, S.CoefficientInteraction(np.eye(2)))
    with pytest.raises(errors.ValidationError):
        S.apply_controlled_single_qubit(sv, [1], 1, S.CoefficientInteraction(np.eye(2)))
    with pytest.raises(errors.ValidationError):
        S.apply_matrix(sv, [0, 1], np.eye(2))
    with pytest.raises(errors.UnsupportedOperationError):
        S.apply_single_qubit(sv, 0, lambda a, i, j: None)
    with pytest.raises(errors.ValidationError):
        S.StateVector(0)
    with pytest.raises(errors.CapacityError):
        S.StateVector(63)
    with pytest.raises(errors.CapacityError):
        Device(45)


@pytest.mark.parametrize("fuse", [False, True])
@pytest.mark.parametrize("i", range(4))
def test_named_gate_circuits_golden(cg, i, fuse):
    n = int(cg[f"circ{i}_n"])
    ops = unpack_ops(cg, f"circ{i}")
    with Device(n) as d:
        d.set_state(cg[f"circ{i}_in"])
        d.apply(ops, fuse=fuse)
        assert np.abs(d.get_state() - cg[f"circ{i}_out"]).max() < STATE_TOL


@pytest.mark.parametrize("fuse", [False, True])
@pytest.mark.parametrize("job", ADJ_JOBS)
def test_adjoint_golden(cg, job, fuse):
    n = int(cg[f"adj_{job}_n"])
    ops = unpack_ops(cg, f"adj_{job}")
    obs = unpack_obs(cg, f"adj_{job}")
    with Device(n) as d:
        jac, ev = d.adjoint_jacobian(ops, obs, return_expvals=True, fuse=fuse)
    ref = cg[f"adj_{job}_jac"]
    assert jac.shape == ref.shape
    assert_grad_close(jac, ref, obs)
    ref_ev = cg[f"adj_{job}_expvals"]
    for k, o in enumerate(obs):
        assert abs(ev[k] - ref_ev[k]) <= 1e-10 * max(obs_norm1(o), abs(ref_ev[k]))


@pytest.mark.parametrize("job", ADJ_JOBS)
def test_probs_golden(cg, job):
    n = int(cg[f"adj_{job}_n"])
    if f"adj_{job}_probs_all" not in cg.files:
        pytest.skip("no probs recorded")
    ops = unpack_ops(cg, f"adj_{job}")
    with Device(n) as d:
        d.apply(ops)
        assert np.abs(d.probs() - cg[f"adj_{job}_probs_all"]).max() < 1e-13
        assert np.abs(d.probs([n - 1, 0]) - cg[f"adj_{job}_probs_w"]).max() < 1e-13


def test_sel20_config1_golden():
    try:
        g = load("sel20_golden.npz")
    except FileNotFoundError:
        pytest.skip("sel20 golden not generated")
    ops, obs = workloads.sel_config(20, 4, seed=0)
    with Device(20) as d:
        jac, ev = d.adjoint_jacobian(ops, obs, return_expvals=True)
    assert_grad_close(jac, g["jac"], obs)
    assert np.abs(ev - g["expvals"]).max() < 1e-10


# ---- SPEC known-answer tests through the device ------------------------------------------

def test_kats_device():
    with Device(1) as d:
        assert np.allclose(d.get_state(), [1, 0])
        d.apply([Op("X", (0,))])
        assert np.allclose(d.get_state(), [0, 1])
    with Device(2) as d:
        d.apply([Op("H", (1,))])
        assert np.allclose(d.get_state(), [2 ** -0.5, 2 ** -0.5, 0, 0])
    with Device(2) as d:
        d.set_basis_state(2)
        d.apply([Op("CNOT", (0, 1))])
        assert np.allclose(d.get_state(), [0, 0, 0, 1])
    with Device(2) as d:
        d.apply([Op("IsingXX", (0, 1), (np.pi,))])
        assert np.allclose(d.get_state(), [0, 0, 0, -1j])
    with Device(1) as d:
        d.apply([Op("H", (0,))])
        assert abs(d.expval(PauliWord(((0, "X"),))) - 1) < 1e-12
        assert np.allclose(d.probs(), [0.5, 0.5])
    with Device(2) as d:
        d.set_basis_state(1)
        h = Hamiltonian([0.5, 0.5], [PauliWord(((0, "Z"),)), PauliWord(((1, "Z"),))])
        assert abs(d.expval(h)) < 1e-12
    with Device(1) as d:
        jac = d.adjoint_jacobian([Op("RX", (0,), (np.pi / 2,), trainable=(True,))], [PauliWord(((0, "Z"),))])
        assert abs(jac[0, 0] + 1) < 1e-12


# ---- oracle sweeps: every kind, every target, random controls -------------------------------

KINDS = [k for k in ARITY if k not in ("Matrix", "ControlledMatrix")]


def random_op(rng, n, kind=None):
    kind = kind or KINDS[int(rng.integers(len(KINDS)))]
    nw, npar = ARITY[kind]
    if kind in ("Matrix", "ControlledMatrix"):
        nw = int(rng.integers(1, 4))
    nc = int(rng.integers(0, min(2, n - nw) + 1)) if rng.random() < 0.3 else 0
    qs = rng.choice(n, size=nw + nc, replace=False)
    m = None
    if kind in ("Matrix", "ControlledMatrix"):
        z = rng.normal(size=(1 << nw, 1 << nw)) + 1j * rng.normal(size=(1 << nw, 1 << nw))
        m = np.linalg.qr(z)[0]
    return Op(kind, tuple(int(q) for q in qs[:nw]), tuple(rng.uniform(-np.pi, np.pi, size=npar)),
              ctrls=tuple(int(q) for q in qs[nw:]), ctrl_values=tuple(int(v) for v in rng.integers(0, 2, size=nc)),
              inverse=bool(rng.random() < 0.2), matrix=m)


@pytest.mark.parametrize("kind", KINDS + ["Matrix", "ControlledMatrix"])
def test_every_kind_every_target(kind):
    rng = np.random.default_rng(sum(map(ord, kind)))
    n = 9
    psi = rand_state(rng, n)
    nw = ARITY[kind][0] or 2
    for t in range(n - nw + 1 if nw > 1 else n):
        op = random_op(rng, n, kind)
        if nw == 1:
            op.wires = (t,)
            op.ctrls = tuple(c for c in op.ctrls if c != t)
            op.ctrl_values = op.ctrl_values[: len(op.ctrls)]
        ref = psi.copy()
        O.apply_op(ref, n, op)
        for fuse in (False, True):
            with Device(n) as d:
                d.set_state(psi)
                d.apply([op], fuse=fuse)
                assert np.abs(d.get_state() - ref).max() < STATE_TOL, (op, fuse)


@pytest.mark.parametrize("n", [6, 11, 16, 20])
def test_random_circuits_vs_oracle(n):
    rng = np.random.default_rng(n)
    ops = [random_op(rng, n) for _ in range(120)]
    psi = rand_state(rng, n)
    ref = O.run_circuit(n, ops, psi)
    for fuse in (False, True):
        with Device(n) as d:
            d.set_state(psi)
            d.apply(ops, fuse=fuse)
            assert np.abs(d.get_state() - ref).max() < 1e-11


def test_every_ordered_pair_cnot():
    n = 7
    rng = np.random.default_rng(5)
    psi = rand_state(rng, n)
    for c in range(n):
        for t in range(n):
            if c == t:
                continue
            ref = psi.copy()
            O.apply_op(ref, n, Op("CNOT", (c, t)))
            with Device(n) as d:
                d.set_state(psi)
                d.apply([Op("CNOT", (c, t))])
                assert np.abs(d.get_state() - ref).max() < STATE_TOL


def test_measurements_vs_oracle():
    rng = np.random.default_rng(11)
    n = 10
    psi = rand_state(rng, n)
    ham = workloads.random_pauli_hamiltonian(n, 40, seed=3)
    dense = rng.normal(size=(8, 8)) + 1j * rng.normal(size=(8, 8))
    dense = DenseHermitian((7, 2, 4), dense + dense.conj().T)
    with Device(n) as d:
        d.set_state(psi)
        assert abs(d.expval(ham) - O.expval(psi, n, ham)) < 1e-12 * max(1, obs_norm1(ham))
        assert abs(d.expval(dense) - O.expval(psi, n, dense)) < 1e-11
        for t in ham.terms[:10]:
            assert abs(d.expval(t) - O.expval(psi, n, t)) < 1e-12
        assert abs(d.norm() - 1) < 1e-13
        for wires in ([0], [9], [3, 1], [9, 0, 4], list(range(n)), [5, 6, 7, 8, 9, 0, 1]):
            assert np.abs(d.probs(wires) - O.probabilities(psi, n, wires)).max() < 1e-14


@pytest.mark.parametrize("seed", range(3))
def test_adjoint_vs_oracle_random(seed):
    rng = np.random.default_rng(100 + seed)
    n = 6
    kinds = ["RX", "RY", "RZ", "Phase", "Rot", "IsingXX", "IsingXY", "IsingYY", "IsingZZ",
             "SingleExcitation", "DoubleExcitation", "CNOT", "H", "CZ", "SWAP", "T"]
    ops = []
    for _ in range(30):
        op = random_op(rng, n, kinds[int(rng.integers(len(kinds)))])
        if ARITY[op.name][1]:
            op.trainable = tuple(bool(x) for x in rng.integers(0, 2, size=ARITY[op.name][1]))
        ops.append(op)
    obs = [PauliWord(((0, "Z"), (3, "X"))), workloads.random_pauli_hamiltonian(n, 12, seed=seed),
           DenseHermitian((4, 1), np.diag([1.0, -2.0, 0.5, 3.0]).astype(complex))]
    ref, ref_ev = O.adjoint_jacobian(n, ops, obs)
    for fuse in (False, True):
        with Device(n) as d:
            jac, ev = d.adjoint_jacobian(ops, obs, return_expvals=True, fuse=fuse)
        assert_grad_close(jac, ref, obs)


# ---- large-n size-independent properties --------------------------------------------------

def test_large_n_inverse_roundtrip_and_norm():
    n = 26
    ops = workloads.random_circuit(n, 4, seed=1)
    inv = [Op(o.name, o.wires, o.params, o.ctrls, o.ctrl_values, (), not o.inverse) for o in reversed(ops)]
    with Device(n) as d:
        d.apply(ops)
        assert abs(d.norm() - 1) < 1e-12
        d.apply(inv)
        st = d.get_state()
    assert abs(st[0] - 1) < 1e-12
    assert np.abs(st[1:]).max() < 1e-12


def test_fused_equals_unfused_mid_size():
    n = 22
    ops = workloads.random_circuit(n, 8, seed=4)
    with Device(n) as a, Device(n) as b:
        a.apply(ops, fuse=False)
        b.apply(ops, fuse=True)
        assert np.abs(a.get_state() - b.get_state()).max() < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_fused_adjoint_single_observable(seed):
    """One observable -> the fused sweep (psi/lambda in one array, GEN bra-kets in the tile)."""
    rng = np.random.default_rng(300 + seed)
    n = [8, 9, 12, 15][seed]
    kinds = ["RX", "RY", "RZ", "Phase", "Rot", "IsingXX", "IsingXY", "IsingYY", "IsingZZ",
             "SingleExcitation", "CNOT", "H", "CZ", "SWAP", "T", "X", "Y"]
    ops = []
    for _ in range(60):
        op = random_op(rng, n, kinds[int(rng.integers(len(kinds)))])
        if ARITY[op.name][1]:
            op.trainable = tuple(bool(x) for x in rng.integers(0, 2, size=ARITY[op.name][1]))
        ops.append(op)
    for obs in (workloads.random_pauli_hamiltonian(n, 10, seed=seed), PauliWord(((0, "Y"), (n - 1, "X"))),
                DenseHermitian((2, n - 2), np.diag([0.5, -1.0, 2.0, 0.25]).astype(complex))):
        ref, ref_ev = O.adjoint_jacobian(n, ops, [obs])
        with Device(n) as d:
            jac, ev = d.adjoint_jacobian(ops, [obs], return_expvals=True, fuse=True)
            st = d.get_state()
        assert_grad_close(jac, ref, [obs])
        assert abs(ev[0] - ref_ev[0]) < 1e-10 * max(1.0, obs_norm1(obs))
        assert np.abs(st - O.run_circuit(n, [])).max() < 1e-10   # the state is swept back to the input


def test_fused_adjoint_qaoa_and_hea_vs_unfused():
    n = 16
    ops, ham, _ = workloads.qaoa_maxcut(n, p=2, seed=1)
    with Device(n) as a, Device(n) as b:
        ja = a.adjoint_jacobian(ops, [ham], fuse=True)
        jb = b.adjoint_jacobian(ops, [ham], fuse=False)
    assert np.abs(ja - jb).max() < 1e-10 * max(1.0, np.abs(jb).max())
    ops = workloads.hardware_efficient_ansatz(n, layers=6, n_trainable=150, seed=2)
    h = workloads.random_pauli_hamiltonian(n, 40, seed=3)
    with Device(n) as a, Device(n) as b:
        ja = a.adjoint_jacobian(ops, [h], fuse=True)
        jb = b.adjoint_jacobian(ops, [h], fuse=False)
    assert np.abs(ja - jb).max() < 1e-10 * max(1.0, sum(abs(c) for c in h.coeffs))


def test_variance_vs_oracle():
    """SPEC.md:313-320 on the device: Pauli words, a Hamiltonian and a dense observable."""
    rng = np.random.default_rng(21)
    n = 11
    psi = rand_state(rng, n)
    obs = [PauliWord(((3, "Z"),)), PauliWord(((0, "X"), (10, "Y"), (5, "Z"))),
           workloads.random_pauli_hamiltonian(n, 25, seed=3),
           DenseHermitian((7, 2), (lambda a: a + a.conj().T)(rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))))]
    with Device(n) as d:
        d.set_state(psi)
        for o in obs:
            got, ref = d.var(o), O.variance(psi, n, o)
            assert abs(got - ref) <= 1e-10 * max(1.0, obs_norm1(o) ** 2), (o, got, ref)
        d.reset()
        assert abs(d.var(PauliWord(((0, "Z"),)))) < 1e-15          # Var(Z) on |0> = 0
        d.apply([Op("H", (0,))])
        assert abs(d.var(PauliWord(((0, "Z"),))) - 1.0) < 1e-12    # Var(Z) on H|0> = 1


def test_sample_vs_oracle_procedure():
    """the device draws the same rows as the oracle's restatement of the
    documented procedure (probabilities agree to ~1e-16, so outcomes coincide), KATs and errors."""
    rng = np.random.default_rng(8)
    n = 12
    ops = workloads.random_circuit(n, 8, seed=2)
    psi = O.run_circuit(n, ops)
    with Device(n) as d:
        d.apply(ops)
        for wires in (None, [3], [11, 0, 5], list(range(n))[::-1]):
            got = d.sample_indices(20_000, seed=1234, wires=wires)
            ref = O.sample(psi, n, 20_000, seed=1234, wires=wires)
            assert (got != ref).sum() <= 1, wires      # a draw on a 1e-16 boundary may differ
        rows = d.sample(64, seed=5, wires=[1, 2])
        assert rows.shape == (64, 2) and set(np.unique(rows)) <= {0, 1}
        assert (d.sample_indices(500, seed=77) == d.sample_indices(500, seed=77)).all()
        with pytest.raises(errors.ValidationError):
            d.sample_indices(0)
        d.set_basis_state((1 << n) - 1)
        assert (d.sample(100, seed=3) == 1).all()              # |1...1> -> all rows ones
        d.reset()
        d.apply([Op("H", (0,))])
        f0 = (d.sample(10_000, seed=42, wires=[0])[:, 0] == 0).mean()
        assert abs(f0 - 0.5) < 0.02


def test_sparse_observable_vs_oracle():
    """SPEC.md:303-311 through the C-ABI: expval, variance and the adjoint Jacobian with a CSR
    observable, on a state whose layout was relabeled by fused passes; structure errors."""
    from paper_2403_02512_b200.observables import SparseHermitian
    rng = np.random.default_rng(17)
    n = 10
    dim = 1 << n
    m = np.zeros((dim, dim), dtype=np.complex128)
    mask = rng.random((dim, dim)) < 0.01
    m[mask] = rng.normal(size=mask.sum()) + 1j * rng.normal(size=mask.sum())
    m = m + m.conj().T
    sp = SparseHermitian.from_dense(m)
    ops = workloads.hardware_efficient_ansatz(n, layers=3, n_trainable=40, seed=3)
    psi = O.run_circuit(n, ops)
    scale = float(np.abs(m).sum(axis=1).max())
    with Device(n) as d:
        d.apply(ops)
        assert abs(d.expval(sp) - np.vdot(psi, m @ psi).real) <= 1e-10 * scale
        assert abs(d.var(sp) - O.variance(psi, n, sp)) <= 1e-10 * scale ** 2
        for fuse in (True, False):
            d.reset()
            jac, ev = d.adjoint_jacobian(ops, [sp], return_expvals=True, fuse=fuse)
            jref, evref = O.adjoint_jacobian(n, ops, [sp])
            assert np.abs(jac - jref).max() <= 1e-10 * scale, fuse
            assert abs(ev[0] - evref[0]) <= 1e-10 * scale
        d.reset()
        with pytest.raises(errors.ValidationError):
            d.expval(SparseHermitian.from_dense(np.eye(8)))      # dimension != 2^n


def test_h2_vqe_energy_and_gradient():
    """circuit-ir end to end on the device: the H2 fixture + singles/doubles ansatz (the
    DoubleExcitation generator takes the per-gate adjoint path), batched and unbatched."""
    import os
    from paper_2403_02512_b200 import circuit_ir as C
    from paper_2403_02512_b200.batching import batched_expval_and_grad
    h2 = C.parse_hamiltonian(open(os.path.join(os.path.dirname(__file__), "fixtures", "h2.ham")).read())
    theta = np.array([0.01, -0.02, 0.21])
    c = C.singles_doubles_ansatz(4, 2, theta)
    jref, evref = O.adjoint_jacobian(4, c.ops, [h2])
    with Device(4) as d:
        jac, ev = d.adjoint_jacobian(c, [h2], return_expvals=True)
    assert abs(ev[0] - evref[0]) < 1e-12 and np.abs(jac - jref).max() < 1e-12
    e, g = batched_expval_and_grad(c.ops, h2, n_workers=3, n_qubits=4)
    assert abs(e - evref[0]) < 1e-12 and np.abs(g - jref[0]).max() < 1e-12
    assert abs(e - (-1.1361894540)) < 2e-3


def test_generated_kernels_reused_across_parameters():
    """Pass compiler (csrc/fused_jit.cpp): a circuit re-run with new angles reuses the compiled
    pass kernels (values travel as kernel parameters) and both runs match the oracle."""
    from paper_2403_02512_b200.device import plan_compile
    from paper_2403_02512_b200.ops import Op as _Op
    n = 14
    a = workloads.random_circuit(n, 10, seed=11)
    b = [_Op(op.name, op.wires, tuple(p + 0.37 for p in op.params), op.ctrls, op.ctrl_values) for op in a]
    probe = [_Op("H", (0,))]
    with Device(n) as d:
        d.apply(a)
        got_a = d.get_state()
        before = plan_compile(8, probe)["kernels_compiled_total"]
        d.reset()
        d.apply(b)
        got_b = d.get_state()
        after = plan_compile(8, probe)["kernels_compiled_total"]
    assert np.abs(got_a - O.run_circuit(n, a)).max() < STATE_TOL
    assert np.abs(got_b - O.run_circuit(n, b)).max() < STATE_TOL
    assert after - before <= 1, (before, after)   # at most the probe's own pass


def test_interpreter_kernel_matches_oracle_subprocess():
    """SVB200_JIT=0 keeps the prebuilt op-interpreting tile kernel (k_fused) as the fused engine;
    it must stay at parity too (run in a child process: the switch is read once per process)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np\n"
        "from oracle import svoracle as O\n"
        "from paper_2403_02512_b200 import workloads\n"
        "from paper_2403_02512_b200.device import Device\n"
        "n = 16\n"
        "ops = workloads.random_circuit(n, 12, seed=5)\n"
        "ops2, obs = workloads.sel_config(10, 2, seed=1)\n"
        "with Device(n) as d:\n"
        "    d.apply(ops)\n"
        "    err = float(np.abs(d.get_state() - O.run_circuit(n, ops)).max())\n"
        "with Device(10) as d:\n"
        "    jac = d.adjoint_jacobian(ops2, obs)\n"
        "ref = O.adjoint_jacobian(10, ops2, obs)[0]\n"
        "errj = float(np.abs(jac - ref).max())\n"
        "assert err < 1e-12 and errj < 1e-10, (err, errj)\n"
        "print('ok', err, errj)\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SVB200_JIT="0", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok")


@pytest.mark.parametrize("wires", [(9, 0, 4, 6, 2), (1, 3, 5, 7, 8, 10)])
def test_dense_observable_many_wires(wires):
    """DenseHermitian on 5+ wires: lambda = O psi in a scratch buffer through the
    shared-memory DENSE kernel, then Re<psi|lambda>; expval and variance vs the oracle."""
    rng = np.random.default_rng(len(wires))
    n = 11
    psi = rand_state(rng, n)
    dim = 1 << len(wires)
    m = rng.normal(size=(dim, dim)) + 1j * rng.normal(size=(dim, dim))
    obs = DenseHermitian(wires, m + m.conj().T)
    with Device(n) as d:
        d.set_state(psi)
        assert abs(d.expval(obs) - O.expval(psi, n, obs)) < 1e-10 * max(1.0, np.abs(obs.matrix).sum())
        got, ref = d.var(obs), O.variance(psi, n, obs)
        assert abs(got - ref) <= 1e-10 * max(1.0, np.abs(obs.matrix).sum() ** 2)
        assert np.abs(d.get_state() - psi).max() == 0.0        # expval leaves the state untouched


@pytest.mark.parametrize("fuse", [False, True])
def test_wide_diagonal_matrix(fuse):
    """A diagonal apply_matrix on 7 wires (state.py:278-303) stays a DENSE primitive (DIAG tables
    hold <= 64 entries) and matches the oracle."""
    rng = np.random.default_rng(5)
    n = 10
    psi = rand_state(rng, n)
    wires = (9, 0, 4, 6, 2, 7, 1)
    m = np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, 1 << len(wires))))
    op = Op("Matrix", wires, matrix=m)
    ref = psi.copy()
    O.apply_op(ref, n, op)
    with Device(n) as d:
        d.set_state(psi)
        d.apply([op], fuse=fuse)
        assert np.abs(d.get_state() - ref).max() < STATE_TOL


@pytest.mark.parametrize("fuse", [False, True])
def test_adjoint_dense_observable_many_wires(fuse):
    """adjoint_jacobian with a 5-wire DenseHermitian observable (lambda = O psi through the
    shared-memory DENSE kernel) vs the oracle."""
    rng = np.random.default_rng(77)
    n = 8
    ops = workloads.random_circuit(n, 5, seed=3)
    for op in ops:
        if ARITY[op.name][1]:
            op.trainable = (True,) * ARITY[op.name][1]
    m = rng.normal(size=(32, 32)) + 1j * rng.normal(size=(32, 32))
    obs = [DenseHermitian((6, 1, 3, 0, 7), m + m.conj().T)]
    ref, ref_ev = O.adjoint_jacobian(n, ops, obs)
    with Device(n) as d:
        jac, ev = d.adjoint_jacobian(ops, obs, return_expvals=True, fuse=fuse)
    assert_grad_close(jac, ref, obs)
    assert abs(ev[0] - ref_ev[0]) < 1e-10 * max(1.0, obs_norm1(obs[0]))


@pytest.mark.parametrize("n", [12, 15, 17])
def test_diagonal_hamiltonian_wht_expval(n):
    """Z-only Hamiltonians with >= 8 terms on states of >= 2^12 amplitudes take the per-tile
    Walsh-Hadamard kernel (k_pauli_diag_wht): identity, low-only, high-only and mixed masks,
    repeated masks, and MaxCut's C = sum 1/2 (I - Z_i Z_j), vs the oracle."""
    rng = np.random.default_rng(n)
    psi = rand_state(rng, n)
    words = [PauliWord(())]
    for _ in range(40):
        k = int(rng.integers(1, 5))
        qs = rng.choice(n, size=k, replace=False)
        words.append(PauliWord(tuple((int(q), "Z") for q in qs)))
    words += [words[3], PauliWord(((0, "Z"),)), PauliWord(((n - 1, "Z"),)), PauliWord(((0, "Z"), (n - 1, "Z")))]
    ham = Hamiltonian(list(rng.normal(size=len(words))), words)
    _, cost, _ = workloads.qaoa_maxcut(n, p=1, seed=1)
    with Device(n) as d:
        d.set_state(psi)
        for h in (ham, cost):
            assert abs(d.expval(h) - O.expval(psi, n, h)) < 1e-12 * max(1.0, obs_norm1(h))
    with Device(n, precision="f32") as d:
        d.set_state(psi.astype(np.complex64))
        ref = O.expval(psi.astype(np.complex64).astype(np.complex128), n, ham)
        assert abs(d.expval(ham) - ref) < 1e-9 * max(1.0, obs_norm1(ham))


@pytest.mark.parametrize("fuse", [False, True])
def test_wht_lambda_adjoint_and_variance(fuse):
    """lambda = H psi through the WHT kernel for the diagonal group (plus ordinary x-groups
    accumulated on top): adjoint Jacobian and variance vs the oracle at n = 13."""
    rng = np.random.default_rng(9)
    n = 13
    ops = workloads.random_circuit(n, 3, seed=2)
    for op in ops:
        if ARITY[op.name][1]:
            op.trainable = (True,) * ARITY[op.name][1]
    zw = [PauliWord(tuple((int(q), "Z") for q in rng.choice(n, size=int(rng.integers(1, 4)), replace=False)))
          for _ in range(20)]
    h_diag = Hamiltonian(list(rng.normal(size=20)), zw)
    h_mixed = Hamiltonian(list(rng.normal(size=23)), zw + [PauliWord(((0, "X"), (5, "Z"))), PauliWord(((12, "Y"),)),
                                                          PauliWord(((3, "X"), (4, "X")))])
    obs = [h_diag, h_mixed]
    ref, ref_ev = O.adjoint_jacobian(n, ops, obs)
    with Device(n) as d:
        jac, ev = d.adjoint_jacobian(ops, obs, return_expvals=True, fuse=fuse)
    assert_grad_close(jac, ref, obs)
    for k in range(2):
        assert abs(ev[k] - ref_ev[k]) < 1e-10 * max(1.0, obs_norm1(obs[k]))
    with Device(n) as d:
        d.apply(ops)
        psi = d.get_state()
        for o in obs:
            assert abs(d.var(o) - O.variance(psi, n, o)) <= 1e-10 * max(1.0, obs_norm1(o) ** 2)
    _, jq = None, None
    with Device(n) as d:   # single-observable fused sweep (lambda from the WHT kernel)
        jac1 = d.adjoint_jacobian(ops, [h_diag], fuse=fuse)
    assert_grad_close(jac1, ref[:1], [h_diag])


def test_alg1_alg2_goldens_through_the_c_abi_entry_points(sg):
    """sv_apply_single_qubit / sv_apply_controlled_single_qubit (include/svb200.h; state.py:154-171
    and :192-226) called directly through ctypes on the reference's Alg. 1 / Alg. 2 goldens."""
    import ctypes
    from paper_2403_02512_b200 import _lib
    L = _lib.lib()
    dbl = ctypes.POINTER(ctypes.c_double)
    i32 = ctypes.POINTER(ctypes.c_int32)
    for n, q, psi, m, out in zip(sg["alg1_n"], sg["alg1_q"], sg["alg1_in"], sg["alg1_m"], sg["alg1_out"]):
        with Device(int(n)) as d:
            d.set_state(psi[: 1 << int(n)])
            mm = np.ascontiguousarray(np.asarray(m, dtype=np.complex128).reshape(4))
            _lib.check(L.sv_apply_single_qubit(d.handle, int(q), mm.view(np.float64).ctypes.data_as(dbl)))
            assert np.abs(d.get_state() - out[: 1 << int(n)]).max() < STATE_TOL
    for i in range(len(sg["alg2_n"])):
        n, q = int(sg["alg2_n"][i]), int(sg["alg2_q"][i])
        ctrls = np.array([c for c in sg["alg2_ctrls"][i] if c >= 0], dtype=np.int32)
        vals = np.array([v for v in sg["alg2_vals"][i] if v >= 0], dtype=np.int32)
        mm = np.ascontiguousarray(np.asarray(sg["alg2_m"][i], dtype=np.complex128).reshape(4))
        with Device(n) as d:
            d.set_state(sg["alg2_in"][i][: 1 << n])
            _lib.check(L.sv_apply_controlled_single_qubit(d.handle, ctrls.ctypes.data_as(i32), len(ctrls), q,
                                                           mm.view(np.float64).ctypes.data_as(dbl),
                                                           vals.ctypes.data_as(i32) if len(vals) else None))
            assert np.abs(d.get_state() - sg["alg2_out"][i][: 1 << n]).max() < STATE_TOL


def test_repeated_apply_restores_layout_and_reuses_kernels():
    """apply() on a relabeled state first restores the canonical layout (one fused SWAP program),
    so repeated applies without reset stay correct and plan/compile nothing new after the first."""
    from paper_2403_02512_b200.device import jit_stats
    n = 16
    ops = workloads.random_circuit(n, 12, seed=21)
    ref = O.run_circuit(n, [])
    with Device(n) as d:
        d.apply(ops)
        d.apply(ops)   # first apply from a drifted layout: compiles the canonicalising program
        before = jit_stats()["compiled"]
        for _ in range(2):
            d.apply(ops)
        after = jit_stats()["compiled"]
        st = d.get_state()
    for _ in range(4):
        ref = O.run_circuit(n, ops, ref)
    assert np.abs(st - ref).max() < 1e-12
    assert after == before, (before, after)


@pytest.mark.parametrize("kind", ["qaoa", "mixed_diag"])
def test_k14_uniform_prefix_write_only_init(kind):
    """K14: from |0...0>, H on every qubit followed by diagonal gates (any controls, any phases) is
    one write-only pass (WHT of the Walsh-expanded phases + sincos); the state equals the oracle's
    gate-by-gate result.  The same list from a non-zero state runs gate by gate."""
    n = 15
    rng = np.random.default_rng(7)
    if kind == "qaoa":
        ops, _, _ = workloads.qaoa_maxcut(n, p=2, seed=4)
    else:
        ops = [Op("H", (q,)) for q in rng.permutation(n)]
        for _ in range(40):
            a, b, c = (int(x) for x in rng.choice(n, size=3, replace=False))
            pick = int(rng.integers(7))
            th = float(rng.uniform(-7, 7))
            ops.append([Op("RZ", (a,), (th,)), Op("IsingZZ", (a, b), (th,)), Op("CZ", (a, b)), Op("T", (a,)),
                        Op("Phase", (a,), (th,), ctrls=(b,)), Op("RZ", (a,), (th,), ctrls=(b, c), ctrl_values=(1, 0)),
                        Op("S", (a,), inverse=True)][pick])
        ops += workloads.random_circuit(n, 3, seed=9)
    ref = O.run_circuit(n, ops)
    with Device(n) as d:
        d.apply(ops)
        st = d.get_state()
        d.set_state(ref)                      # not |0...0>: the prefix must run gate by gate
        d.apply(ops)
        st2 = d.get_state()
    assert np.abs(st - ref).max() < 1e-12
    assert np.abs(st2 - O.run_circuit(n, ops, ref)).max() < 1e-12
