"""CPU oracle for the B200 state-vector hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU reference. The product (``paper_2403_02512_b200``) never calls
it; there is no CPU fallback.

What it is: a numpy restatement of the reference's algorithm
(``/root/reference/pkg/src/svkit/state.py``) for gate application, plus
restatements of the SPEC-only modules the reference does not ship
(gate library SPEC.md:123-196, measurements SPEC.md:267-352, adjoint gradient
SPEC.md:354-422, sharded semantics SPEC.md:424-486). Each function cites the
reference line it follows.

Parity pinning: ``tests/golden/make_golden.py`` imports the real
``svkit.state`` from /root/reference (in the build container only) and writes
``tests/golden/state_golden.npz``; ``tests/test_oracle.py`` checks this oracle
bit-for-bit-ish (|d| < 1e-13) against those vectors, and against the SPEC
known-answer tests. The expval/adjoint layers have no executable reference
(SPEC only); their golden values are produced by running every gate through
the reference's own ``apply_matrix`` (see make_golden.py) and they are
cross-checked here by parameter-shift and finite differences.
"""

import numpy as np

BIT_WIDTH = 64                      # state.py:14
UINT_MAX = (1 << BIT_WIDTH) - 1     # state.py:15
MAX_QUBITS = 62                     # state.py:18


class OracleError(ValueError):
    pass


# ---------------------------------------------------------------------------
# statevector-core (state.py)
# ---------------------------------------------------------------------------

def zero_state(n_qubits):
    """|0...0> (state.py:34-47)."""
    if n_qubits < 1:
        raise OracleError("n_qubits must be >= 1")
    amps = np.zeros(1 << n_qubits, dtype=np.complex128)
    amps[0] = 1.0
    return amps


def get_masks(excluded_bit_offsets, n_qubits):
    """n_excluded+1 disjoint masks around the excluded offsets (state.py:128-151).

    Returns (masks, strides). masks[0] = bits below the lowest excluded offset,
    masks[i] = bits strictly between excluded offsets i-1 and i, last = bits
    above the highest, clipped to the n-bit window.
    """
    bits = sorted(excluded_bit_offsets)
    if len(set(bits)) != len(bits):
        raise OracleError("duplicate offsets")
    if any(not 0 <= b < n_qubits for b in bits):
        raise OracleError("offset out of range")
    window = (1 << n_qubits) - 1
    if not bits:
        return (window,), ()
    masks = [(1 << bits[0]) - 1]
    for lo, hi in zip(bits[:-1], bits[1:]):
        masks.append(((1 << hi) - 1) ^ ((1 << (lo + 1)) - 1))
    masks.append(window & ~((1 << (bits[-1] + 1)) - 1))
    return tuple(masks), tuple(1 << b for b in bits)


def expand(masks, ks):
    """Spread compact counters ``ks`` into the non-excluded bits (state.py:112-124)."""
    ks = np.asarray(ks, dtype=np.uint64)
    out = ks & np.uint64(masks[0])
    for i in range(1, len(masks)):
        out |= (ks << np.uint64(i)) & np.uint64(masks[i])
    return out


def alg1_pairs(n, q):
    """(i0, i1) index arrays of Alg. 1 (state.py:162-171)."""
    n, q = int(n), int(q)
    q_offset = n - q - 1
    stride = 1 << q_offset
    mask_high = (UINT_MAX << (q_offset + 1)) & UINT_MAX
    mask_low = 0 if q_offset == 0 else UINT_MAX >> (BIT_WIDTH - q_offset)  # state.py:166-167
    k = np.arange(1 << (n - 1), dtype=np.uint64)
    i0 = ((k << np.uint64(1)) & np.uint64(mask_high)) | (k & np.uint64(mask_low))
    return i0, i0 | np.uint64(stride)


def alg2_pairs(n, ctrls, q, ctrl_values=None):
    """(i0, i1) arrays of Alg. 2 with prescribed control values (state.py:192-226)."""
    n, q = int(n), int(q)
    ctrls = tuple(int(c) for c in ctrls)
    values = (1,) * len(ctrls) if not ctrl_values else tuple(int(v) for v in ctrl_values)
    if len(set(ctrls)) != len(ctrls) or q in ctrls or len(values) != len(ctrls):
        raise OracleError("bad controls")
    q_offset = n - q - 1
    ctrl_offsets = [n - 1 - c for c in ctrls]
    masks, _ = get_masks(sorted(ctrl_offsets + [q_offset]), n)
    on_bits = 0
    for off, v in zip(ctrl_offsets, values):   # values align with ctrls as given, state.py:214-217
        if v:
            on_bits |= 1 << off
    k = np.arange(1 << (n - 1 - len(ctrls)), dtype=np.uint64)
    i0 = expand(masks, k) | np.uint64(on_bits)
    return i0, i0 | np.uint64(1 << q_offset)


def apply_single_qubit(amps, n, q, m):
    """Alg. 1 with the coefficient interaction given as a 2x2 matrix (state.py:154-171)."""
    i0, i1 = alg1_pairs(n, q)
    a0, a1 = amps[i0].copy(), amps[i1].copy()
    amps[i0] = m[0, 0] * a0 + m[0, 1] * a1
    amps[i1] = m[1, 0] * a0 + m[1, 1] * a1


def apply_controlled_single_qubit(amps, n, ctrls, q, m, ctrl_values=None):
    """Alg. 2 with the interaction given as a 2x2 matrix (state.py:192-226)."""
    i0, i1 = alg2_pairs(n, ctrls, q, ctrl_values)
    a0, a1 = amps[i0].copy(), amps[i1].copy()
    amps[i0] = m[0, 0] * a0 + m[0, 1] * a1
    amps[i1] = m[1, 0] * a0 + m[1, 1] * a1


def wire_addresses(n, wires):
    """(2^w, 2^(n-w)) address table, wires[0] = MSB of the row index (state.py:238-257)."""
    n, wires = int(n), [int(x) for x in wires]
    w = len(wires)
    offsets = [n - 1 - q for q in wires]
    masks, _ = get_masks(sorted(offsets), n)
    base = expand(masks, np.arange(1 << (n - w), dtype=np.uint64))
    rows = np.zeros(1 << w, dtype=np.uint64)
    for j, o in enumerate(offsets):
        sel = (np.arange(1 << w) >> (w - 1 - j)) & 1
        rows |= sel.astype(np.uint64) << np.uint64(o)
    return rows[:, None] | base[None, :]


def apply_matrix(amps, n, wires, matrix):
    """Dense 2^w x 2^w contraction on ordered wires, in place (state.py:278-303).

    Gather -> M @ sub -> scatter, the reference's <=4-wire path (state.py:260-264);
    the >4-wire transpose path (state.py:267-275) computes the same contraction.
    """
    n, wires = int(n), tuple(int(x) for x in wires)
    if len(set(wires)) != len(wires) or any(not 0 <= w < n for w in wires):
        raise OracleError("bad wires")
    matrix = np.asarray(matrix, dtype=np.complex128)
    if matrix.shape != (1 << len(wires),) * 2:
        raise OracleError("matrix shape")
    addr = wire_addresses(n, wires)
    amps[addr] = matrix @ amps[addr]


# ---------------------------------------------------------------------------
# gate-library (conventions SURVEY Appendix A)
# ---------------------------------------------------------------------------

_I2 = np.eye(2, dtype=np.complex128)
_X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
_Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
PAULI = {"I": _I2, "X": _X, "Y": _Y, "Z": _Z}


def _sub_rotation(dim, i, j, theta):
    """exp(-i theta/2 sigma_y) in span{|i>,|j>} of a dim-dim identity."""
    m = np.eye(dim, dtype=np.complex128)
    c, s = np.cos(theta / 2), np.sin(theta / 2)
    m[i, i] = c
    m[i, j] = -s
    m[j, i] = s
    m[j, j] = c
    return m


def matrix_of(name, params=()):
    """Unitary of a named gate. Rotations exp(-i theta/2 P)."""
    p = list(params)
    if name == "I":
        return _I2.copy()
    if name in ("X", "Y", "Z"):
        return PAULI[name].copy()
    if name == "H":
        return np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2)
    if name == "S":
        return np.diag([1, 1j]).astype(np.complex128)
    if name == "T":
        return np.diag([1, np.exp(1j * np.pi / 4)])
    if name == "Phase":
        return np.diag([1, np.exp(1j * p[0])])
    if name in ("RX", "RY", "RZ"):
        P = PAULI[name[1]]
        return np.cos(p[0] / 2) * _I2 - 1j * np.sin(p[0] / 2) * P
    if name == "Rot":
        # Rot(phi, theta, omega) == RZ(phi) . RY(theta) . RZ(omega) as matrices
        return matrix_of("RZ", [p[0]]) @ matrix_of("RY", [p[1]]) @ matrix_of("RZ", [p[2]])
    if name == "CNOT":
        m = np.eye(4, dtype=np.complex128)
        m[2:, 2:] = _X
        return m
    if name == "CZ":
        return np.diag([1, 1, 1, -1]).astype(np.complex128)
    if name == "SWAP":
        return np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]
    if name in ("IsingXX", "IsingYY", "IsingZZ"):
        P = PAULI[name[5]]
        PP = np.kron(P, P)
        return np.cos(p[0] / 2) * np.eye(4) - 1j * np.sin(p[0] / 2) * PP    # Eq. 1
    if name == "IsingXY":
        G = np.kron(_X, _X) + np.kron(_Y, _Y)
        return _expm_herm(G, 0.25 * p[0])
    if name == "SingleExcitation":
        return _sub_rotation(4, 1, 2, p[0])                     # span{|01>,|10>}, SPEC.md:123 / PAPER.md:147
    if name == "DoubleExcitation":
        return _sub_rotation(16, 3, 12, p[0])                   # span{|0011>,|1100>}
    raise OracleError(f"no matrix for {name}")


def _expm_herm(G, alpha):
    """exp(i alpha G) for Hermitian G via eigendecomposition."""
    w, v = np.linalg.eigh(G)
    return (v * np.exp(1j * alpha * w)) @ v.conj().T


def generator_of(name):
    """(G, prefactor) with gate(theta) = exp(i prefactor theta G)."""
    if name in ("RX", "RY", "RZ"):
        return PAULI[name[1]].copy(), -0.5
    if name == "Phase":
        return np.diag([0, 1]).astype(np.complex128), 1.0
    if name in ("IsingXX", "IsingYY", "IsingZZ"):
        P = PAULI[name[5]]
        return np.kron(P, P), -0.5
    if name == "IsingXY":
        return np.kron(_X, _X) + np.kron(_Y, _Y), 0.25
    if name == "SingleExcitation":
        g = np.zeros((4, 4), dtype=np.complex128)
        g[1, 2], g[2, 1] = -1j, 1j
        return g, -0.5
    if name == "DoubleExcitation":
        g = np.zeros((16, 16), dtype=np.complex128)
        g[3, 12], g[12, 3] = -1j, 1j
        return g, -0.5
    raise OracleError(f"{name} has no single-parameter generator")


def _controlled(m, n_ctrls, ctrl_values):
    """Block matrix acting as ``m`` where the control bits equal ``ctrl_values``."""
    if n_ctrls == 0:
        return m
    d = m.shape[0]
    on = 0
    for v in ctrl_values:
        on = (on << 1) | int(v)
    full = np.eye(d << n_ctrls, dtype=np.complex128)
    full[on * d:(on + 1) * d, on * d:(on + 1) * d] = m
    return full


def base_matrix(op, params=None):
    """Target-wire unitary of an op (no controls), honouring ``inverse``."""
    params = op.params if params is None else params
    if op.name in ("Matrix", "ControlledMatrix"):
        m = np.asarray(op.matrix, dtype=np.complex128)
    else:
        m = matrix_of(op.name, params)
    return m.conj().T if op.inverse else m


def apply_op(amps, n, op, params=None):
    """Apply one op record: 1q (+ctrls) via Alg. 1/2, everything else via apply_matrix."""
    m = base_matrix(op, params)
    ctrls = tuple(op.ctrls)
    vals = tuple(op.ctrl_values) if op.ctrl_values else (1,) * len(ctrls)
    if len(op.wires) == 1 and not ctrls:
        apply_single_qubit(amps, n, op.wires[0], m)
    elif len(op.wires) == 1:
        apply_controlled_single_qubit(amps, n, ctrls, op.wires[0], m, vals)
    else:
        apply_matrix(amps, n, ctrls + tuple(op.wires), _controlled(m, len(ctrls), vals))


def run_circuit(n, ops, state=None):
    amps = zero_state(n) if state is None else np.array(state, dtype=np.complex128)
    for op in ops:
        apply_op(amps, n, op)
    return amps


# ---------------------------------------------------------------------------
# measurements
# ---------------------------------------------------------------------------

def apply_pauli_word(amps, n, factors):
    """Out-of-place P|psi> for a Pauli word [(wire, P), ...]."""
    out = np.array(amps, dtype=np.complex128)
    for w, p in factors:
        if p != "I":
            apply_single_qubit(out, n, w, PAULI[p])
    return out


def apply_observable(amps, n, obs):
    """Out-of-place O|psi> (the lambda = O psi step of SPEC.md:373)."""
    if hasattr(obs, "indptr"):   # SparseHermitian: CSR over logical indices
        amps = np.asarray(amps)
        out = np.zeros_like(amps)
        for r in range(len(obs.indptr) - 1):
            lo, hi = obs.indptr[r], obs.indptr[r + 1]
            out[r] = np.dot(obs.data[lo:hi], amps[obs.indices[lo:hi]])
        return out
    if hasattr(obs, "factors"):
        return apply_pauli_word(amps, n, obs.factors)
    if hasattr(obs, "coeffs"):
        out = np.zeros_like(amps)
        for c, t in zip(obs.coeffs, obs.terms):
            out += c * apply_pauli_word(amps, n, t.factors)
        return out
    out = np.array(amps, dtype=np.complex128)
    apply_matrix(out, n, obs.wires, obs.matrix)
    return out


def expval(amps, n, obs):
    """<psi|O|psi>: Hamiltonian = sum_t c_t <P_t>."""
    if hasattr(obs, "coeffs"):
        return float(sum(c * expval(amps, n, t) for c, t in zip(obs.coeffs, obs.terms)))
    return float(np.vdot(amps, apply_observable(amps, n, obs)).real)


def probabilities(amps, n, wires=None):
    """Marginal probabilities over ``wires`` (all wires if None), wires[0] = MSB."""
    p = np.abs(np.asarray(amps)) ** 2
    if wires is None:
        return p
    wires = list(wires)
    t = p.reshape((2,) * n)
    rest = tuple(q for q in range(n) if q not in wires)
    m = t.sum(axis=rest) if rest else t
    kept = sorted(wires)
    return np.transpose(m, [kept.index(w) for w in wires]).reshape(-1)


def variance(amps, n, obs):
    """<O^2> - <O>^2, O^2 formed by applying O twice."""
    amps = np.asarray(amps)
    lam = apply_observable(amps, n, obs)
    e = np.vdot(amps, lam).real
    return float(np.vdot(lam, lam).real - e * e)


def _splitmix64(x):
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def sample(amps, n, shots, seed=0, wires=None):
    """Outcome indices of ``shots`` draws by the fixed inverse-CDF procedure
    the library documents (include/svb200.h, sv_sample): sequential prefix sums C of the
    marginal probabilities, u_i = splitmix64(seed + (i+1) * golden) >> 11 scaled by 2^-53,
    outcome = first b with C[b] > u_i * C[-1]."""
    if shots < 1:
        raise OracleError("shots must be >= 1")
    c = np.cumsum(probabilities(amps, n, wires))
    m = (1 << 64) - 1
    u = np.array([(_splitmix64((seed + (i + 1) * 0x9E3779B97F4A7C15) & m) >> 11) for i in range(shots)],
                 dtype=np.float64) * (1.0 / 9007199254740992.0) * c[-1]
    return np.minimum(np.searchsorted(c, u, side="right"), len(c) - 1).astype(np.int64)


# ---------------------------------------------------------------------------
# adjoint-gradient (formula SURVEY Appendix A)
# ---------------------------------------------------------------------------

def lower_op(op):
    """Expand Rot into RZ(omega), RY(theta), RZ(phi) in application order.

    Returns a list of (name, wires, param, ctrls, ctrl_values, inverse, trainable, column_key)
    single-parameter pieces for the adjoint sweep.
    """
    if op.name != "Rot":
        return [op]
    phi, theta, omega = op.params
    tr = op.trainable or (False,) * 3
    from types import SimpleNamespace as NS
    seq = [("RZ", omega, tr[2], 2), ("RY", theta, tr[1], 1), ("RZ", phi, tr[0], 0)]
    if op.inverse:
        seq = seq[::-1]
    return [NS(name=nm, wires=op.wires, params=(a,), ctrls=op.ctrls, ctrl_values=op.ctrl_values,
               inverse=op.inverse, matrix=None, trainable=(t,), _rot_param=k) for nm, a, t, k in seq]


def _generator_full(op):
    """Generator G on ctrls+wires (controls become a projector) and prefactor c."""
    G, c = generator_of(op.name)
    if op.inverse:
        c = -c
    vals = tuple(op.ctrl_values) if op.ctrl_values else (1,) * len(op.ctrls)
    if op.ctrls:
        on = 0
        for v in vals:
            on = (on << 1) | int(v)
        d = G.shape[0]
        full = np.zeros((d << len(op.ctrls),) * 2, dtype=np.complex128)
        full[on * d:(on + 1) * d, on * d:(on + 1) * d] = G
        G = full
    return G, c


def adjoint_jacobian(n, ops, observables, state=None):
    """Jacobian [n_obs x n_trainable] by one forward pass + reverse sweep.

    d<O>/d theta_k = -2 c Im<lambda_k|G_k|psi_k>; columns ordered by (op, param)
    with Rot params in (phi, theta, omega) order. Returns (jac, expvals).
    """
    # column bookkeeping in circuit order
    cols = {}
    for i, op in enumerate(ops):
        for p, t in enumerate(op.trainable or ()):
            if t:
                if op.name not in ("Phase", "RX", "RY", "RZ", "Rot", "IsingXX", "IsingXY", "IsingYY",
                                   "IsingZZ", "SingleExcitation", "DoubleExcitation"):
                    raise OracleError(f"{op.name} is not differentiable")
                cols[(i, p)] = len(cols)
    pieces = []
    for i, op in enumerate(ops):
        for piece in lower_op(op):
            pidx = getattr(piece, "_rot_param", 0)
            trainable = bool(piece.trainable and piece.trainable[0])
            pieces.append((piece, cols[(i, pidx)] if trainable else None))
    psi = run_circuit(n, [p for p, _ in pieces], state)
    lams = [apply_observable(psi, n, o) for o in observables]
    expvals = np.array([np.vdot(psi, l).real for l in lams])
    jac = np.zeros((len(observables), len(cols)))
    for piece, col in reversed(pieces):
        if col is not None:
            G, c = _generator_full(piece)
            mu = psi.copy()
            apply_matrix(mu, n, tuple(piece.ctrls) + tuple(piece.wires), G)
            for k, lam in enumerate(lams):
                jac[k, col] = -2.0 * c * np.vdot(lam, mu).imag
        inv = _inverse_piece(piece)
        apply_op(psi, n, inv)
        for lam in lams:
            apply_op(lam, n, inv)
    return jac, expvals


def _inverse_piece(op):
    from types import SimpleNamespace as NS
    return NS(name=op.name, wires=op.wires, params=op.params, ctrls=op.ctrls,
              ctrl_values=op.ctrl_values, inverse=not op.inverse, matrix=op.matrix, trainable=())


def _param_circuit_expvals(n, ops, observables, state, col, delta):
    """Expectation values with trainable column ``col`` shifted by ``delta``."""
    shifted = []
    k = 0
    for op in ops:
        params = list(op.params)
        for p, t in enumerate(op.trainable or ()):
            if t:
                if k == col:
                    params[p] += delta
                k += 1
        from types import SimpleNamespace as NS
        shifted.append(NS(name=op.name, wires=op.wires, params=tuple(params), ctrls=op.ctrls,
                          ctrl_values=op.ctrl_values, inverse=op.inverse, matrix=op.matrix,
                          trainable=op.trainable))
    psi = run_circuit(n, shifted, state)
    return np.array([expval(psi, n, o) for o in observables])


def parameter_shift_jacobian(n, ops, observables, state=None):
    """(f(theta+pi/2) - f(theta-pi/2))/2 per column. Valid for Pauli-generator gates."""
    ncol = sum(sum(op.trainable or ()) for op in ops)
    jac = np.zeros((len(observables), ncol))
    for c in range(ncol):
        jac[:, c] = 0.5 * (_param_circuit_expvals(n, ops, observables, state, c, np.pi / 2)
                           - _param_circuit_expvals(n, ops, observables, state, c, -np.pi / 2))
    return jac


def finite_diff_jacobian(n, ops, observables, state=None, h=1e-6):
    """Central finite differences (h = 1e-6)."""
    ncol = sum(sum(op.trainable or ()) for op in ops)
    jac = np.zeros((len(observables), ncol))
    for c in range(ncol):
        jac[:, c] = (_param_circuit_expvals(n, ops, observables, state, c, h)
                     - _param_circuit_expvals(n, ops, observables, state, c, -h)) / (2 * h)
    return jac


# ---------------------------------------------------------------------------
# sharded-sv semantics
# ---------------------------------------------------------------------------

def shard(amps, n_shards):
    """Contiguous split; global qubits are the top log2(n_shards) bits."""
    if n_shards < 1 or n_shards & (n_shards - 1) or n_shards > len(amps):
        raise OracleError("n_shards must be a power of two <= 2^n")
    return [s.copy() for s in np.split(np.asarray(amps), n_shards)]


def gather(shards):
    return np.concatenate(shards)
