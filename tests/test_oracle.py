"""CPU: pin the oracle (oracle/svoracle.py) against the reference's golden vectors and SPEC KATs.

The golden vectors were produced by the real ``svkit.state`` (tests/golden/make_golden.py).
"""

import ast

import numpy as np
import pytest

from oracle import svoracle as O
from paper_2403_02512_b200 import workloads
from paper_2403_02512_b200.observables import DenseHermitian, Hamiltonian, PauliWord
from paper_2403_02512_b200.ops import Op
from tests.golden_io import ADJ_JOBS, load, unpack_obs, unpack_ops

TOL = 1e-13


@pytest.fixture(scope="module")
def sg():
    return load("state_golden.npz")


@pytest.fixture(scope="module")
def cg():
    return load("circuit_golden.npz")


def test_get_masks_matches_reference(sg):
    for n, excl, masks, strides in ast.literal_eval(str(sg["masks_repr"])):
        m, s = O.get_masks(excl, n)
        assert list(m) == masks and list(s) == strides


def test_alg1_matches_reference(sg):
    for n, q, psi, m, out in zip(sg["alg1_n"], sg["alg1_q"], sg["alg1_in"], sg["alg1_m"], sg["alg1_out"]):
        amps = psi[: 1 << n].copy()
        O.apply_single_qubit(amps, n, q, m)
        assert np.abs(amps - out[: 1 << n]).max() < TOL


def test_alg2_matches_reference(sg):
    for i in range(len(sg["alg2_n"])):
        n, q = int(sg["alg2_n"][i]), int(sg["alg2_q"][i])
        ctrls = [c for c in sg["alg2_ctrls"][i] if c >= 0]
        vals = [v for v in sg["alg2_vals"][i] if v >= 0]
        amps = sg["alg2_in"][i][: 1 << n].copy()
        O.apply_controlled_single_qubit(amps, n, ctrls, q, sg["alg2_m"][i], vals)
        assert np.abs(amps - sg["alg2_out"][i][: 1 << n]).max() < TOL


def test_apply_matrix_matches_reference(sg):
    off = sg["mat_m_off"]
    for i in range(len(sg["mat_n"])):
        n = int(sg["mat_n"][i])
        wires = [w for w in sg["mat_wires"][i] if w >= 0]
        d = 1 << len(wires)
        m = sg["mat_m_flat"][off[i]:off[i + 1]].reshape(d, d)
        amps = sg["mat_in"][i][: 1 << n].copy()
        O.apply_matrix(amps, n, wires, m)
        assert np.abs(amps - sg["mat_out"][i][: 1 << n]).max() < 1e-12


@pytest.mark.parametrize("i", range(4))
def test_named_gate_circuits_match_reference(cg, i):
    n = int(cg[f"circ{i}_n"])
    ops = unpack_ops(cg, f"circ{i}")
    out = O.run_circuit(n, ops, cg[f"circ{i}_in"])
    assert np.abs(out - cg[f"circ{i}_out"]).max() < 1e-12


@pytest.mark.parametrize("job", ADJ_JOBS)
def test_adjoint_matches_reference_backed_golden(cg, job):
    n = int(cg[f"adj_{job}_n"])
    ops = unpack_ops(cg, f"adj_{job}")
    obs = unpack_obs(cg, f"adj_{job}")
    jac, ev = O.adjoint_jacobian(n, ops, obs)
    assert np.abs(jac - cg[f"adj_{job}_jac"]).max() < 1e-11
    assert np.abs(ev - cg[f"adj_{job}_expvals"]).max() < 1e-12


# ---- SPEC known-answer tests ---------------------------------------------------------

def test_kat_zero_state():
    assert np.array_equal(O.zero_state(1), [1, 0])
    assert np.array_equal(O.zero_state(3), np.eye(8)[0])


def test_kat_alg1_pairs():
    i0, i1 = O.alg1_pairs(3, 0)
    assert list(zip(i0.tolist(), i1.tolist())) == [(0, 4), (1, 5), (2, 6), (3, 7)]


def test_kat_x_and_h():
    a = O.zero_state(1)
    O.apply_single_qubit(a, 1, 0, O.matrix_of("X"))
    assert np.allclose(a, [0, 1])
    a = O.zero_state(2)
    O.apply_single_qubit(a, 2, 1, O.matrix_of("H"))
    assert np.allclose(a, [2 ** -0.5, 2 ** -0.5, 0, 0])


def test_kat_cnot_truth_table_and_count():
    a = np.array([0, 0, 1, 0], dtype=complex)
    O.apply_controlled_single_qubit(a, 2, [0], 1, O.matrix_of("X"))
    assert np.allclose(a, [0, 0, 0, 1])
    a = np.array([0, 1, 0, 0], dtype=complex)
    O.apply_controlled_single_qubit(a, 2, [0], 1, O.matrix_of("X"))
    assert np.allclose(a, [0, 1, 0, 0])
    i0, _ = O.alg2_pairs(4, [0, 1], 3)
    assert len(i0) == 2


def test_kat_masks():
    m, _ = O.get_masks([2], 3)
    assert m == (0b011, 0)
    m, _ = O.get_masks([], 4)
    assert m == (0b1111,)
    m, _ = O.get_masks([0, 3], 4)
    assert m[0] | m[1] | m[2] == 0b0110 and m[0] & m[1] == 0 and m[1] & m[2] == 0


def test_kat_gates_and_generators():
    xx = O.matrix_of("IsingXX", [np.pi])                                 # SPEC.md:151-152, Eq. 1
    a = O.zero_state(2)
    O.apply_matrix(a, 2, [0, 1], xx)
    assert np.allclose(a, [0, 0, 0, -1j])
    a = O.zero_state(1)
    O.apply_single_qubit(a, 1, 0, O.matrix_of("RX", [np.pi]))            # SPEC.md:150 RX(pi)|0> = -i|1>
    assert np.allclose(a, [0, -1j])
    rot = O.matrix_of("Rot", [0.1, 0.2, 0.3])
    assert np.allclose(rot, O.matrix_of("RZ", [0.1]) @ O.matrix_of("RY", [0.2]) @ O.matrix_of("RZ", [0.3]))
    import scipy.linalg as sl
    for name in ("RX", "RY", "RZ", "Phase", "IsingXX", "IsingXY", "IsingYY", "IsingZZ",
                 "SingleExcitation", "DoubleExcitation"):
        G, c = O.generator_of(name)
        for th in (0.0, 0.3, -0.3, np.pi / 2, -np.pi / 2, np.pi):
            assert np.abs(sl.expm(1j * c * th * G) - O.matrix_of(name, [th])).max() < 1e-12
        U = O.matrix_of(name, [0.77])
        assert np.abs(U.conj().T @ U - np.eye(len(U))).max() < 1e-13


def test_kat_measurements():
    a = O.zero_state(1)
    assert np.allclose(O.probabilities(a, 1), [1, 0])
    O.apply_single_qubit(a, 1, 0, O.matrix_of("H"))
    assert np.allclose(O.probabilities(a, 1), [0.5, 0.5])
    assert abs(O.expval(a, 1, PauliWord(((0, "X"),))) - 1) < 1e-12
    bell = np.array([1, 0, 0, 1], dtype=complex) / np.sqrt(2)
    assert np.allclose(O.probabilities(bell, 2, [0]), [0.5, 0.5])
    assert abs(O.expval(O.zero_state(1), 1, PauliWord(((0, "Z"),))) - 1) < 1e-12
    s01 = np.eye(4)[1].astype(complex)
    h = Hamiltonian([0.5, 0.5], [PauliWord(((0, "Z"),)), PauliWord(((1, "Z"),))])
    assert abs(O.expval(s01, 2, h)) < 1e-12


def test_kat_adjoint_rx():
    ops = [Op("RX", (0,), (np.pi / 2,), trainable=(True,))]
    jac, _ = O.adjoint_jacobian(1, ops, [PauliWord(((0, "Z"),))])
    assert abs(jac[0, 0] + 1) < 1e-12
    jac, _ = O.adjoint_jacobian(1, [Op("RX", (0,), (0.3,))], [PauliWord(((0, "Z"),))])
    assert jac.shape == (1, 0)


def test_probabilities_wire_order():
    rng = np.random.default_rng(1)
    psi = rng.normal(size=16) + 1j * rng.normal(size=16)
    psi /= np.linalg.norm(psi)
    p = O.probabilities(psi, 4, [2, 0])
    t = (np.abs(psi) ** 2).reshape(2, 2, 2, 2)
    ref = np.einsum("abcd->ca", t).reshape(-1)
    assert np.allclose(p, ref)


@pytest.mark.parametrize("seed", range(4))
def test_adjoint_vs_parameter_shift_and_fd(seed):
    """adjoint vs parameter-shift < 1e-10 and vs FD (h=1e-6) < 1e-6."""
    rng = np.random.default_rng(seed)
    n = 4
    kinds = ["RX", "RY", "RZ", "IsingXX", "IsingYY", "IsingZZ", "Phase", "Rot"]
    ops = []
    for _ in range(20):
        k = kinds[int(rng.integers(len(kinds)))]
        nw = 2 if k.startswith("Ising") else 1
        npar = 3 if k == "Rot" else 1
        qs = rng.choice(n, size=nw, replace=False)
        ops.append(Op(k, tuple(qs), tuple(rng.uniform(-3, 3, size=npar)), trainable=(True,) * npar))
        ops.append(Op("CNOT", tuple(rng.choice(n, size=2, replace=False))))
    obs = [PauliWord(((0, "Z"),)), Hamiltonian([0.4, -0.9], [PauliWord(((1, "X"), (2, "Y"))),
                                                            PauliWord(((3, "Z"),))])]
    jac, _ = O.adjoint_jacobian(n, ops, obs)
    ps = O.parameter_shift_jacobian(n, ops, obs)
    fd = O.finite_diff_jacobian(n, ops, obs)
    assert np.abs(jac - ps).max() < 1e-10
    assert np.abs(jac - fd).max() < 1e-6


def test_adjoint_non_pauli_generators_vs_fd():
    rng = np.random.default_rng(7)
    n = 4
    ops = [Op("H", (q,)) for q in range(n)]
    ops += [Op("IsingXY", (0, 1), (0.7,), trainable=(True,)),
            Op("SingleExcitation", (1, 2), (0.4,), trainable=(True,)),
            Op("DoubleExcitation", (0, 1, 2, 3), (1.1,), trainable=(True,)),
            Op("RY", (2,), (0.3,), ctrls=(0,), ctrl_values=(0,), trainable=(True,)),
            Op("RX", (3,), (0.9,), inverse=True, trainable=(True,))]
    herm = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
    obs = [DenseHermitian((1, 3), herm + herm.conj().T), PauliWord(((0, "Y"), (2, "X")))]
    jac, _ = O.adjoint_jacobian(n, ops, obs)
    fd = O.finite_diff_jacobian(n, ops, obs)
    assert np.abs(jac - fd).max() < 1e-6


def test_sel_template_counts():
    w = np.zeros((3, 4, 3))
    ops = workloads.strongly_entangling_layers(4, w)
    assert sum(op.name == "Rot" for op in ops) == 12
    assert sum(op.name == "CNOT" for op in ops) == 12
    assert sum(op.n_trainable for op in ops) == 36
    ops = workloads.strongly_entangling_layers(3, np.zeros((1, 3, 3)))
    assert [op.wires for op in ops if op.name == "CNOT"] == [(0, 1), (1, 2), (2, 0)]


def test_sharded_model_roundtrip():
    psi = np.arange(8, dtype=complex)
    sh = O.shard(psi, 2)
    assert np.array_equal(sh[0], psi[:4]) and np.array_equal(O.gather(sh), psi)


def test_kat_variance():
    """Var(Z) on |0> = 0, on H|0> = 1; Hamiltonian and dense vs explicit O^2."""
    zero = O.zero_state(1)
    assert abs(O.variance(zero, 1, PauliWord(((0, "Z"),)))) < 1e-15
    plus = np.array([1, 1], dtype=np.complex128) / np.sqrt(2)
    assert abs(O.variance(plus, 1, PauliWord(((0, "Z"),))) - 1.0) < 1e-15
    rng = np.random.default_rng(3)
    n = 5
    psi = rng.normal(size=32) + 1j * rng.normal(size=32)
    psi /= np.linalg.norm(psi)
    h = Hamiltonian([0.3, -1.2], [PauliWord(((0, "X"), (2, "Y"))), PauliWord(((4, "Z"),))])
    M = np.stack([O.apply_observable(np.eye(32, dtype=np.complex128)[:, k], n, h) for k in range(32)], axis=1)
    ref = np.vdot(psi, M @ M @ psi).real - np.vdot(psi, M @ psi).real ** 2
    assert abs(O.variance(psi, n, h) - ref) < 1e-12


def test_kat_sample():
    """|1> -> all ones; H|0> frequency 0.5 +- 0.02 at 1e4 shots; same seed ->
    identical rows; shots = 0 rejected; chi-square against |psi|^2."""
    one = np.array([0, 1], dtype=np.complex128)
    assert (O.sample(one, 1, 100, seed=7) == 1).all()
    plus = np.array([1, 1], dtype=np.complex128) / np.sqrt(2)
    s = O.sample(plus, 1, 10_000, seed=11)
    assert abs((s == 0).mean() - 0.5) < 0.02
    assert (O.sample(plus, 1, 500, seed=3) == O.sample(plus, 1, 500, seed=3)).all()
    with pytest.raises(O.OracleError):
        O.sample(plus, 1, 0)
    rng = np.random.default_rng(0)
    n = 4
    psi = rng.normal(size=16) + 1j * rng.normal(size=16)
    psi /= np.linalg.norm(psi)
    shots = 100_000
    counts = np.bincount(O.sample(psi, n, shots, seed=5), minlength=16)
    expected = np.abs(psi) ** 2 * shots
    chi2 = float(((counts - expected) ** 2 / expected).sum())
    assert chi2 < 37.7   # chi-square(15 dof) at p = 0.001
    # marginal over wires (2, 0): same procedure on the marginal vector
    m = O.sample(psi, n, 1000, seed=9, wires=[2, 0])
    assert m.min() >= 0 and m.max() < 4


def rand_sparse_herm(rng, n, density=0.08):
    dim = 1 << n
    m = np.zeros((dim, dim), dtype=np.complex128)
    mask = rng.random((dim, dim)) < density
    m[mask] = rng.normal(size=mask.sum()) + 1j * rng.normal(size=mask.sum())
    return m + m.conj().T


def test_kat_sparse_expval():
    """CSR identity -> 1; CSR of Z on |1> -> -1; random sparse Hermitian (n=6)
    vs the dense contraction; malformed CSR -> validation error."""
    from paper_2403_02512_b200.errors import ValidationError
    from paper_2403_02512_b200.observables import SparseHermitian
    rng = np.random.default_rng(4)
    psi = rng.normal(size=8) + 1j * rng.normal(size=8)
    psi /= np.linalg.norm(psi)
    assert abs(O.expval(psi, 3, SparseHermitian.from_dense(np.eye(8))) - 1.0) < 1e-14
    one = np.array([0, 1], dtype=np.complex128)
    assert abs(O.expval(one, 1, SparseHermitian.from_dense(np.diag([1.0, -1.0]))) + 1.0) < 1e-15
    n = 6
    m = rand_sparse_herm(rng, n)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    sp = SparseHermitian.from_dense(m)
    assert np.allclose(sp.to_dense(), m)
    assert abs(O.expval(psi, n, sp) - np.vdot(psi, m @ psi).real) < 1e-10
    with pytest.raises(ValidationError):
        SparseHermitian([0, 2, 1], [0, 1], [1.0, 1.0])          # non-monotone row pointers
    with pytest.raises(ValidationError):
        SparseHermitian([0, 1, 2], [0, 5], [1.0, 1.0])          # column out of range


# ---- complex64 ("f32", state.py:20) goldens from the reference's own complex64 arithmetic ----

F32_TOL = 2e-6   # a few float32 roundings of O(1) amplitudes (reference _NORM_TOL f32 = 1e-5)


def test_f32_golden_apply_matrix_vs_oracle():
    d = load("f32_golden.npz")
    n = int(d["am_n"])
    for wires, psi, m, out in zip(d["am_wires"], d["am_in"], d["am_m"], d["am_out"]):
        w = [int(x) for x in wires if x >= 0]
        assert psi.dtype == np.complex64 and out.dtype == np.complex64
        amps = psi.astype(np.complex128)
        O.apply_matrix(amps, n, w, m[: 1 << len(w), : 1 << len(w)])
        assert np.abs(amps - out).max() < F32_TOL


def test_f32_golden_circuit_vs_oracle():
    d = load("f32_golden.npz")
    n = int(d["circ_n"])
    ops = workloads.random_circuit(n, int(d["circ_depth"]), seed=int(d["circ_seed"]))
    ref = O.run_circuit(n, ops)
    assert d["circ_out"].dtype == np.complex64
    assert np.abs(ref - d["circ_out"]).max() < 1e-5


def test_qaoa_p1_closed_form_matches_oracle():
    """The closed-form p=1 MaxCut expectation (the 33-qubit parity check, where no CPU state fits)
    equals the oracle's <C> on small graphs, 3- and 4-regular, with triangles."""
    from oracle.qaoa_closed_form import maxcut_p1_expectation
    for n, seed, deg in [(10, 0, 3), (12, 3, 3), (11, 5, 4), (12, 7, 4)]:
        ops, ham, edges = workloads.qaoa_maxcut(n, p=1, seed=seed, degree=deg)
        ev = O.expval(O.run_circuit(n, ops), n, ham)
        g, b = ops[n].params[0] / 2, ops[-1].params[0] / 2
        assert abs(ev - maxcut_p1_expectation(n, edges, g, b)) < 1e-12


def test_product_get_masks_matches_reference(sg):
    """The package's own get_masks (paper_2403_02512_b200/state.py) against the reference's
    recorded get_masks outputs (masks_repr golden, state.py:128-151)."""
    from paper_2403_02512_b200 import state as S
    for n, excl, masks, strides in ast.literal_eval(str(sg["masks_repr"])):
        ms = S.get_masks(excl, n)
        got_m = list(ms.masks) if hasattr(ms, "masks") else list(ms[0])
        got_s = list(ms.strides) if hasattr(ms, "strides") else list(ms[1])
        assert got_m == masks and got_s == strides
