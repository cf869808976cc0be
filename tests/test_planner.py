"""CPU: the fusion planner's program (passes, phases, X relabeling, merging, qubit remapping),
re-executed by tests/fused_emulator.py, reproduces the oracle -- no GPU needed."""

import numpy as np
import pytest

from oracle import svoracle as O
from paper_2403_02512_b200 import workloads
from paper_2403_02512_b200.ops import ARITY, Op
from tests.fused_emulator import plan_program, run_program


def rand_state(rng, n):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def random_op(rng, n):
    kinds = [k for k in ARITY if k not in ("Matrix", "ControlledMatrix")] + ["Matrix", "ControlledMatrix"]
    kind = kinds[int(rng.integers(len(kinds)))]
    nw, npar = ARITY[kind]
    if nw is None:
        nw = int(rng.integers(1, 3))
    nc = int(rng.integers(0, min(2, n - nw) + 1)) if rng.random() < 0.35 else 0
    qs = rng.choice(n, size=nw + nc, replace=False)
    m = None
    if kind in ("Matrix", "ControlledMatrix"):
        z = rng.normal(size=(1 << nw, 1 << nw)) + 1j * rng.normal(size=(1 << nw, 1 << nw))
        m = np.linalg.qr(z)[0]
    return Op(kind, tuple(int(q) for q in qs[:nw]), tuple(rng.uniform(-np.pi, np.pi, size=npar)),
              ctrls=tuple(int(q) for q in qs[nw:]), ctrl_values=tuple(int(v) for v in rng.integers(0, 2, size=nc)),
              inverse=bool(rng.random() < 0.2), matrix=m)


def check(n, ops, seed=0):
    rng = np.random.default_rng(seed)
    psi = rand_state(rng, n)
    ref = O.run_circuit(n, ops, psi)
    prog = plan_program(n, ops)
    got = run_program(prog, psi)
    assert np.abs(got - ref).max() < 1e-12
    return prog


@pytest.mark.parametrize("n", [13, 14])
def test_random_circuit_program(n):
    prog = check(n, workloads.random_circuit(n, 12, seed=n))
    assert any(k == "pass" for k, _ in prog["steps"])
    assert prog["perm"] != list(range(n))   # the in-tile relabeling moved qubits


@pytest.mark.parametrize("seed", range(6))
def test_every_kind_program(seed):
    rng = np.random.default_rng(seed)
    n = 13
    check(n, [random_op(rng, n) for _ in range(150)], seed)


def test_cnot_heavy_program_uses_xflip_and_remap():
    rng = np.random.default_rng(3)
    n = 14
    ops = []
    for _ in range(200):
        c, t = rng.choice(n, size=2, replace=False)
        ops.append(Op("CNOT", (int(c), int(t))))
        ops.append(Op(("RX", "RY", "RZ")[int(rng.integers(3))], (int(rng.integers(n)),), (float(rng.uniform(0, 6)),)))
    prog = check(n, ops)
    cases = {op["cs"] for op in prog["ops"]}
    assert cases & set(range(62, 66)), "thread-predicated X should use CS_XFLIP"


def test_structured_workloads_program():
    ops, _ = workloads.sel_config(12, 3, seed=1)
    check(12, ops)
    ops, _, _ = workloads.qaoa_maxcut(12, p=2, seed=2)
    check(12, ops)
    check(13, workloads.hardware_efficient_ansatz(13, layers=4, n_trainable=100, seed=4))


def test_parity_and_shear_cases_are_exercised():
    """IsingZZ becomes a parity phase (register mask + per-thread parity), unconditioned
    rotations become scaled 2-FMA rotations -- both re-executed against the oracle."""
    rng = np.random.default_rng(11)
    n = 14
    ops = [Op("H", (q,)) for q in range(n)]
    for _ in range(60):
        a, b = rng.choice(n, size=2, replace=False)
        ops.append(Op("IsingZZ", (int(a), int(b)), (float(rng.uniform(-3, 3)),)))
        ops.append(Op(("RX", "RY")[int(rng.integers(2))], (int(rng.integers(n)),), (float(rng.uniform(-6, 6)),)))
        if rng.random() < 0.3:
            ops.append(Op("CNOT", (int(a), int(b))))
    prog = check(n, ops)
    cases = [op["cs"] for op in prog["ops"]]
    assert any(106 <= c < 122 for c in cases), "IsingZZ should plan to CS_PARITY"
    assert any(122 <= c < 146 for c in cases), "rotations should plan to the scaled CS_TAN / CS_TAND forms"
    assert any(106 <= op["cs"] < 122 and op["xm"] for op in prog["ops"]), "some parity bits off the registers"


def test_wide_diagonal_matrix_program():
    """A 7-wire diagonal Matrix stays a DENSE primitive (DIAG tables hold <= 64 entries) and the
    planned program still reproduces the oracle."""
    rng = np.random.default_rng(5)
    n = 13
    m = np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, 128)))
    ops = [Op("H", (q,)) for q in range(n)] + [Op("Matrix", (12, 0, 4, 6, 2, 7, 1), matrix=m), Op("RX", (3,), (0.3,))]
    check(n, ops)


def test_scaled_rotations_tan_and_cot():
    """Unconditioned rotations plan to the scaled 2-FMA form (CS_TAN: R/cos for |phi| <= pi/4, R/sin
    beyond), the pass's product of dropped factors is absorbed into one op of the pass, and the
    program still reproduces the oracle (fused_plan.cpp absorb_pass_scale)."""
    n = 13
    prog = check(n, workloads.random_circuit(n, 20, seed=5))
    tans = [op["cs"] for op in prog["ops"] if 122 <= op["cs"] < 138]
    assert any((c - 122) % 4 < 2 for c in tans), "TAN form"
    assert any((c - 122) % 4 >= 2 for c in tans), "COT form"
    # RY on a bit a thread-predicated X may flip: CS_TAND (flipped threads apply R(-phi))
    prog = check(n, workloads.random_circuit(n, 30, seed=0), seed=1)
    assert any(138 <= op["cs"] < 146 for op in prog["ops"]), "TAND form"
    # near-pi rotations (RX(pi) = -iX-like): COT with kappa ~ 0, and exact multiples of pi/2
    ops = [Op("RX", (q,), (np.pi - 1e-9 * q,)) for q in range(n)] + \
          [Op("RY", (q,), (np.pi / 2,)) for q in range(n)] + workloads.random_circuit(n, 4, seed=1)
    check(n, ops, seed=2)
