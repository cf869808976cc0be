// Gate library and op lowering (host side of libsvb200).
//
// gate-library: matrix_of / generator_of for the GateKind
// vocabulary of SPEC.md:129, rotations exp(-i theta/2 P),
// IsingXX per Eq. 1, Rot(phi,theta,omega) = RZ(phi) RY(theta)
// RZ(omega) as matrices, T = diag(1, e^{i pi/4}),
// Phase(phi) = diag(1, e^{i phi}), Single/DoubleExcitation
// rotations in span{|01>,|10>} / span{|0011>,|1100>}.
//
// Lowering turns each op into PAIR / DIAG / DENSE primitives on logical bit
// offsets (offset = n-1-q: qubit 0 is the MSB, state.py:1-5); a PAIR is the
// Alg. 1 / Alg. 2 pair loop (state.py:154-226) with the control pattern folded
// into (fmask, fval) exactly like get_masks + on_bits (state.py:212-225).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>

#include "sv_internal.h"

namespace {

const cplx I1(0.0, 1.0);

int arity_wires(int kind) {
  switch (kind) {
    case SV_GATE_CNOT: case SV_GATE_CZ: case SV_GATE_SWAP: case SV_GATE_ISINGXX:
    case SV_GATE_ISINGXY: case SV_GATE_ISINGYY: case SV_GATE_ISINGZZ:
    case SV_GATE_SINGLE_EXCITATION:
      return 2;
    case SV_GATE_DOUBLE_EXCITATION:
      return 4;
    case SV_GATE_MATRIX: case SV_GATE_CONTROLLED_MATRIX:
      return -1;
    default:
      return 1;
  }
}

int arity_params(int kind) {
  switch (kind) {
    case SV_GATE_PHASE: case SV_GATE_RX: case SV_GATE_RY: case SV_GATE_RZ:
    case SV_GATE_ISINGXX: case SV_GATE_ISINGXY: case SV_GATE_ISINGYY: case SV_GATE_ISINGZZ:
    case SV_GATE_SINGLE_EXCITATION: case SV_GATE_DOUBLE_EXCITATION:
      return 1;
    case SV_GATE_ROT:
      return 3;
    default:
      return 0;
  }
}

std::string tuple_str(const int32_t* v, int n) {
  std::ostringstream s;
  s << "(";
  for (int i = 0; i < n; ++i) s << (i ? ", " : "") << v[i];
  if (n == 1) s << ",";
  s << ")";
  return s.str();
}

std::vector<cplx> eye(int d) {
  std::vector<cplx> m(size_t(d) * d, 0.0);
  for (int i = 0; i < d; ++i) m[size_t(i) * d + i] = 1.0;
  return m;
}

std::vector<cplx> matmul(const std::vector<cplx>& a, const std::vector<cplx>& b, int d) {
  std::vector<cplx> c(size_t(d) * d, 0.0);
  for (int i = 0; i < d; ++i)
    for (int k = 0; k < d; ++k) {
      cplx aik = a[size_t(i) * d + k];
      if (aik == 0.0) continue;
      for (int j = 0; j < d; ++j) c[size_t(i) * d + j] += aik * b[size_t(k) * d + j];
    }
  return c;
}

std::vector<cplx> dagger(const std::vector<cplx>& a, int d) {
  std::vector<cplx> c(size_t(d) * d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) c[size_t(j) * d + i] = std::conj(a[size_t(i) * d + j]);
  return c;
}

std::vector<cplx> kron(const std::vector<cplx>& a, int da, const std::vector<cplx>& b, int db) {
  int d = da * db;
  std::vector<cplx> c(size_t(d) * d);
  for (int i = 0; i < da; ++i)
    for (int j = 0; j < da; ++j)
      for (int k = 0; k < db; ++k)
        for (int l = 0; l < db; ++l)
          c[size_t(i * db + k) * d + (j * db + l)] = a[size_t(i) * da + j] * b[size_t(k) * db + l];
  return c;
}

std::vector<cplx> pauli(char p) {
  switch (p) {
    case 'X': return {0.0, 1.0, 1.0, 0.0};
    case 'Y': return {0.0, -I1, I1, 0.0};
    case 'Z': return {1.0, 0.0, 0.0, -1.0};
    default: return {1.0, 0.0, 0.0, 1.0};
  }
}

// exp(-i theta/2 P) = cos(theta/2) I - i sin(theta/2) P
std::vector<cplx> rotation(const std::vector<cplx>& P, int d, double theta) {
  std::vector<cplx> m = eye(d);
  double c = std::cos(theta / 2), s = std::sin(theta / 2);
  for (size_t i = 0; i < m.size(); ++i) m[i] = c * m[i] - I1 * s * P[i];
  return m;
}

std::vector<cplx> sub_rotation(int d, int i, int j, double theta) {
  std::vector<cplx> m = eye(d);
  double c = std::cos(theta / 2), s = std::sin(theta / 2);
  m[size_t(i) * d + i] = c;
  m[size_t(i) * d + j] = -s;
  m[size_t(j) * d + i] = s;
  m[size_t(j) * d + j] = c;
  return m;
}

// generator G and prefactor c with gate(theta) = exp(i c theta G)
bool generator_of(int kind, std::vector<cplx>& G, double& c) {
  switch (kind) {
    case SV_GATE_RX: G = pauli('X'); c = -0.5; return true;
    case SV_GATE_RY: G = pauli('Y'); c = -0.5; return true;
    case SV_GATE_RZ: G = pauli('Z'); c = -0.5; return true;
    case SV_GATE_PHASE: G = {0.0, 0.0, 0.0, 1.0}; c = 1.0; return true;
    case SV_GATE_ISINGXX: G = kron(pauli('X'), 2, pauli('X'), 2); c = -0.5; return true;
    case SV_GATE_ISINGYY: G = kron(pauli('Y'), 2, pauli('Y'), 2); c = -0.5; return true;
    case SV_GATE_ISINGZZ: G = kron(pauli('Z'), 2, pauli('Z'), 2); c = -0.5; return true;
    case SV_GATE_ISINGXY: {
      G = kron(pauli('X'), 2, pauli('X'), 2);
      auto yy = kron(pauli('Y'), 2, pauli('Y'), 2);
      for (size_t i = 0; i < G.size(); ++i) G[i] += yy[i];
      c = 0.25;
      return true;
    }
    case SV_GATE_SINGLE_EXCITATION:
      G.assign(16, 0.0); G[1 * 4 + 2] = -I1; G[2 * 4 + 1] = I1; c = -0.5; return true;
    case SV_GATE_DOUBLE_EXCITATION:
      G.assign(256, 0.0); G[3 * 16 + 12] = -I1; G[12 * 16 + 3] = I1; c = -0.5; return true;
    default:
      return false;
  }
}

// physical bit position of wire q: logical offset n-1-q mapped through the shard layout
inline int off(int n, int q, const int* phys) { return phys ? phys[n - 1 - q] : n - 1 - q; }

// Build a prim from a 2^k matrix on logical wires (wires[0] = MSB), plus controls.
Prim make_prim(const std::vector<int>& wires, const std::vector<cplx>& m, int n,
               const std::vector<int>& ctrls, const std::vector<int>& cvals, const int* phys) {
  Prim p = make_dense_prim(wires, m, n, ctrls, cvals, phys);
  classify_prim(p);
  return p;
}

}  // namespace

// Raise ValidationError / UnsupportedOperationError exactly where the reference does
// (state.py:95-97, 200-207, 229-235, 291-295).
void validate_op(const sv_op& op, int n) {
  if (op.kind < 0 || op.kind >= SV_GATE_COUNT) sv_fail(SV_ERR_VALIDATION, "unknown gate kind " + std::to_string(op.kind));
  int nw = arity_wires(op.kind);
  if (nw > 0 && op.n_wires != nw)
    sv_fail(SV_ERR_VALIDATION, "gate kind " + std::to_string(op.kind) + " acts on " + std::to_string(nw) +
                                   " wires, got " + std::to_string(op.n_wires));
  if (op.n_wires < 1 || op.n_wires > 30) sv_fail(SV_ERR_VALIDATION, "bad number of wires");
  if (op.n_ctrls < 0 || op.n_ctrls > 62) sv_fail(SV_ERR_VALIDATION, "bad number of controls");
  if (!op.wires || (op.n_ctrls && !op.ctrls)) sv_fail(SV_ERR_VALIDATION, "null wire array");
  for (int i = 0; i < op.n_wires; ++i)
    if (op.wires[i] < 0 || op.wires[i] >= n)
      sv_fail(SV_ERR_VALIDATION, "wire " + std::to_string(op.wires[i]) + " out of range for " + std::to_string(n) +
                                     "-qubit register");
  for (int i = 0; i < op.n_wires; ++i)
    for (int j = i + 1; j < op.n_wires; ++j)
      if (op.wires[i] == op.wires[j]) sv_fail(SV_ERR_VALIDATION, "duplicate wires: " + tuple_str(op.wires, op.n_wires));
  for (int i = 0; i < op.n_ctrls; ++i) {
    if (op.ctrls[i] < 0 || op.ctrls[i] >= n)
      sv_fail(SV_ERR_VALIDATION, "control " + std::to_string(op.ctrls[i]) + " out of range for " + std::to_string(n) +
                                     "-qubit register");
    for (int j = i + 1; j < op.n_ctrls; ++j)
      if (op.ctrls[i] == op.ctrls[j]) sv_fail(SV_ERR_VALIDATION, "duplicate control qubits: " + tuple_str(op.ctrls, op.n_ctrls));
    for (int j = 0; j < op.n_wires; ++j)
      if (op.ctrls[i] == op.wires[j])
        sv_fail(SV_ERR_VALIDATION, "target qubit " + std::to_string(op.wires[j]) + " overlaps controls " +
                                       tuple_str(op.ctrls, op.n_ctrls));
    if (op.ctrl_values && op.ctrl_values[i] != 0 && op.ctrl_values[i] != 1)
      sv_fail(SV_ERR_VALIDATION, "control values must be bits");
  }
  if ((op.kind == SV_GATE_MATRIX || op.kind == SV_GATE_CONTROLLED_MATRIX) && !op.matrix)
    sv_fail(SV_ERR_VALIDATION, "matrix kind without a matrix");
  int np = arity_params(op.kind);
  if (op.trainable_mask & ~((1 << np) - 1))
    sv_fail(SV_ERR_UNSUPPORTED, "gate kind " + std::to_string(op.kind) + " has no trainable parameter here");
}

std::vector<cplx> gate_matrix(int kind, const double* p, int n_wires, const double* matrix) {
  switch (kind) {
    case SV_GATE_I: return eye(2);
    case SV_GATE_X: return pauli('X');
    case SV_GATE_Y: return pauli('Y');
    case SV_GATE_Z: return pauli('Z');
    case SV_GATE_H: {
      double r = 1.0 / std::sqrt(2.0);
      return {r, r, r, -r};
    }
    case SV_GATE_S: return {1.0, 0.0, 0.0, I1};
    case SV_GATE_T: return {1.0, 0.0, 0.0, std::exp(I1 * (M_PI / 4))};
    case SV_GATE_PHASE: return {1.0, 0.0, 0.0, std::exp(I1 * p[0])};
    case SV_GATE_RX: return rotation(pauli('X'), 2, p[0]);
    case SV_GATE_RY: return rotation(pauli('Y'), 2, p[0]);
    case SV_GATE_RZ: return rotation(pauli('Z'), 2, p[0]);
    case SV_GATE_ROT: {
      double z1[1] = {p[0]}, y[1] = {p[1]}, z2[1] = {p[2]};
      return matmul(matmul(gate_matrix(SV_GATE_RZ, z1, 1, nullptr), gate_matrix(SV_GATE_RY, y, 1, nullptr), 2),
                    gate_matrix(SV_GATE_RZ, z2, 1, nullptr), 2);
    }
    case SV_GATE_CNOT: {
      auto m = eye(4);
      m[10] = 0.0; m[11] = 1.0; m[14] = 1.0; m[15] = 0.0;
      return m;
    }
    case SV_GATE_CZ: {
      auto m = eye(4);
      m[15] = -1.0;
      return m;
    }
    case SV_GATE_SWAP: {
      std::vector<cplx> m(16, 0.0);
      m[0] = 1.0; m[1 * 4 + 2] = 1.0; m[2 * 4 + 1] = 1.0; m[15] = 1.0;
      return m;
    }
    case SV_GATE_ISINGXX: return rotation(kron(pauli('X'), 2, pauli('X'), 2), 4, p[0]);
    case SV_GATE_ISINGYY: return rotation(kron(pauli('Y'), 2, pauli('Y'), 2), 4, p[0]);
    case SV_GATE_ISINGZZ: return rotation(kron(pauli('Z'), 2, pauli('Z'), 2), 4, p[0]);
    case SV_GATE_ISINGXY: {
      // exp(i phi/4 (XX + YY)): identity on |00>,|11>; [[c, i s],[i s, c]] on {|01>,|10>}
      auto m = eye(4);
      double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
      m[1 * 4 + 1] = c; m[1 * 4 + 2] = I1 * s; m[2 * 4 + 1] = I1 * s; m[2 * 4 + 2] = c;
      return m;
    }
    case SV_GATE_SINGLE_EXCITATION: return sub_rotation(4, 1, 2, p[0]);
    case SV_GATE_DOUBLE_EXCITATION: return sub_rotation(16, 3, 12, p[0]);
    case SV_GATE_MATRIX:
    case SV_GATE_CONTROLLED_MATRIX: {
      size_t d = size_t(1) << n_wires;
      std::vector<cplx> m(d * d);
      for (size_t i = 0; i < d * d; ++i) m[i] = cplx(matrix[2 * i], matrix[2 * i + 1]);
      return m;
    }
  }
  sv_fail(SV_ERR_UNSUPPORTED, "unknown gate kind");
}

Prim make_dense_prim(const std::vector<int>& wires, const std::vector<cplx>& m, int n,
                     const std::vector<int>& ctrls, const std::vector<int>& cvals, const int* phys) {
  Prim p;
  p.type = PRIM_DENSE;
  int k = int(wires.size());
  if (k > 16) sv_fail(SV_ERR_UNSUPPORTED, "dense matrices on more than 16 wires are not supported");
  std::vector<int> offs(k);
  for (int j = 0; j < k; ++j) offs[j] = off(n, wires[j], phys);
  std::vector<int> sorted = offs;
  std::sort(sorted.begin(), sorted.end());
  p.nb = k;
  for (int j = 0; j < k; ++j) p.pos[j] = sorted[j];
  // matrix index bit (k-1-j) <-> offs[j]   ==>   new index bit i <-> sorted[i]
  std::vector<int> old_bit_of_new(k);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j)
      if (offs[j] == sorted[i]) old_bit_of_new[i] = k - 1 - j;
  size_t d = size_t(1) << k;
  std::vector<size_t> perm(d);
  for (size_t r = 0; r < d; ++r) {
    size_t o = 0;
    for (int i = 0; i < k; ++i)
      if ((r >> i) & 1) o |= size_t(1) << old_bit_of_new[i];
    perm[r] = o;
  }
  p.m.resize(d * d);
  for (size_t r = 0; r < d; ++r)
    for (size_t c = 0; c < d; ++c) p.m[r * d + c] = m[perm[r] * d + perm[c]];
  for (int j = 0; j < k; ++j) p.fmask |= 1ull << p.pos[j];
  for (size_t i = 0; i < ctrls.size(); ++i) {
    int o = off(n, ctrls[i], phys);
    p.fmask |= 1ull << o;
    if (cvals[i]) p.fval |= 1ull << o;
  }
  return p;
}

// Specialise a DENSE prim (positions ascending, fmask includes targets with value 0):
//   diagonal        -> DIAG (single non-unit entry folded into fmask/fval);
//   2-dim subspace  -> PAIR (Alg. 1/2 pair loop);
//   identity        -> skip.
void classify_prim(Prim& p) {
  if (p.type != PRIM_DENSE) return;
  int k = p.nb;
  size_t d = size_t(1) << k;
  bool diag = true;
  std::vector<int> moved;   // basis states whose row/col differ from identity
  for (size_t r = 0; r < d; ++r) {
    bool dev = false;
    for (size_t c = 0; c < d; ++c) {
      cplx v = p.m[r * d + c];
      cplx e = (r == c) ? cplx(1.0) : cplx(0.0);
      if (r != c && v != 0.0) diag = false;
      if (v != e || p.m[c * d + r] != e) dev = true;
    }
    if (dev) moved.push_back(int(r));
  }
  u64 tmask = 0;
  for (int j = 0; j < k; ++j) tmask |= 1ull << p.pos[j];
  auto pattern = [&](size_t r) {
    u64 v = 0;
    for (int j = 0; j < k; ++j)
      if ((r >> j) & 1) v |= 1ull << p.pos[j];
    return v;
  };
  if (moved.empty()) {
    p.skip = true;
    return;
  }
  if (diag) {
    if (moved.size() == 1) {
      cplx v = p.m[size_t(moved[0]) * d + moved[0]];
      p.type = PRIM_DIAG;
      p.fval |= pattern(moved[0]);
      p.nb = 0;
      p.m.assign(1, v);
      return;
    }
    if (k > 6) return;   // DIAG tables hold <= 64 entries; wider diagonals stay DENSE
    std::vector<cplx> t(d);
    for (size_t r = 0; r < d; ++r) t[r] = p.m[r * d + r];
    p.type = PRIM_DIAG;
    p.fmask &= ~tmask;
    p.m = t;
    return;
  }
  if (moved.size() == 2) {
    size_t u = moved[0], v = moved[1];
    std::vector<cplx> m2 = {p.m[u * d + u], p.m[u * d + v], p.m[v * d + u], p.m[v * d + v]};
    p.type = PRIM_PAIR;
    p.fval |= pattern(u);
    p.xmask = pattern(u) ^ pattern(v);
    p.nb = 0;
    p.m = m2;
    return;
  }
}

Prim adjoint_prim(const Prim& p) {
  Prim q = p;
  if (p.type == PRIM_DIAG) {
    for (auto& v : q.m) v = std::conj(v);
  } else {
    int d = (p.type == PRIM_PAIR) ? 2 : (1 << p.nb);
    q.m = dagger(p.m, d);
  }
  return q;
}

std::vector<Piece> lower_op(const sv_op& op, int n, int& next_column, bool need_gen, const int* phys) {
  std::vector<Piece> out;
  std::vector<int> wires(op.wires, op.wires + op.n_wires);
  std::vector<int> ctrls(op.ctrls ? op.ctrls : nullptr, op.ctrls ? op.ctrls + op.n_ctrls : nullptr);
  std::vector<int> cvals(op.n_ctrls, 1);
  if (op.ctrl_values)
    for (int i = 0; i < op.n_ctrls; ++i) cvals[i] = op.ctrl_values[i];
  int np = arity_params(op.kind);
  // Jacobian columns of this op, in parameter order
  int col[3] = {-1, -1, -1};
  for (int i = 0; i < np; ++i)
    if (op.trainable_mask & (1 << i)) col[i] = next_column++;

  auto add_piece = [&](int kind, const double* params, int column) {
    Piece pc;
    std::vector<cplx> U = gate_matrix(kind, params, op.n_wires, op.matrix);
    int d = 1 << op.n_wires;
    if (op.inverse) U = dagger(U, d);
    pc.fwd = make_prim(wires, U, n, ctrls, cvals, phys);
    pc.inv = adjoint_prim(pc.fwd);
    if (column >= 0 && need_gen) {
      std::vector<cplx> G;
      double c;
      if (!generator_of(kind, G, c)) sv_fail(SV_ERR_UNSUPPORTED, "gate kind " + std::to_string(kind) + " is not differentiable");
      pc.has_gen = true;
      pc.gen.g = make_dense_prim(wires, G, n, ctrls, cvals, phys);
      pc.gen.prefactor = op.inverse ? -c : c;
      pc.gen.column = column;
    }
    out.push_back(pc);
  };

  if (op.kind == SV_GATE_I && op.trainable_mask == 0) return out;
  if (op.kind == SV_GATE_ROT) {
    // Rot(phi, theta, omega) = RZ(phi) RY(theta) RZ(omega): RZ(omega) is applied first
    double phi[1] = {op.params[0]}, th[1] = {op.params[1]}, om[1] = {op.params[2]};
    struct { int kind; double* p; int c; } seq[3] = {{SV_GATE_RZ, om, col[2]}, {SV_GATE_RY, th, col[1]}, {SV_GATE_RZ, phi, col[0]}};
    if (op.inverse) std::swap(seq[0], seq[2]);
    for (auto& s : seq) add_piece(s.kind, s.p, s.c);
    return out;
  }
  add_piece(op.kind, op.params, col[0]);
  return out;
}

// Factor the first table entry out of every unrestricted DIAG prim (RZ = e^{-i t/2} diag(1, e^{i t}),
// IsingZZ, ...) and fold the product of those scalars into the matrix of one uncontrolled
// 1-qubit PAIR / DENSE prim (each amplitude passes through it exactly once).  The remaining
// table then has a unit entry, so single-bit diagonals touch half of the amplitudes.  Exact up
// to fp64 rounding of the divisions (|d| ~ 1e-16).
void fold_diag_phases(std::vector<Prim>& prims) {
  cplx phase(1.0, 0.0);
  for (auto& p : prims) {
    if (p.skip || p.type != PRIM_DIAG || p.fmask != 0 || p.nb == 0) continue;
    const cplx f = p.m[0];
    if (f == cplx(1.0, 0.0)) continue;
    phase *= f;
    for (size_t i = 1; i < p.m.size(); ++i) p.m[i] /= f;
    p.m[0] = 1.0;
    if (p.nb == 1) {   // [1, t] -> single entry on bit = 1
      p.fmask = p.fval = 1ull << p.pos[0];
      p.m = {p.m[1]};
      p.nb = 0;
    }
  }
  if (phase == cplx(1.0, 0.0)) return;
  for (auto& p : prims) {
    if (p.skip) continue;
    const bool whole_pair = p.type == PRIM_PAIR && popcount64(p.xmask) == 1 && p.fmask == p.xmask;
    u64 tm = 0;
    for (int j = 0; j < p.nb; ++j) tm |= 1ull << p.pos[j];
    const bool whole_dense = p.type == PRIM_DENSE && p.fmask == tm;
    if (whole_pair || whole_dense) {
      for (auto& v : p.m) v *= phase;
      return;
    }
  }
  Prim s;
  s.type = PRIM_DIAG;
  s.m = {phase};
  prims.push_back(s);
}

// Resolve bits that live on the shard index (physical position >= nl) for this rank:
// controls / fixed bits become a predicate (skip when unmet), DIAG table bits become a
// per-rank constant -- no communication (SURVEY.md §8(e) "no-comm cases").
void resolve_global(Prim& p, int nl, int rank) {
  if (p.skip) return;
  u64 local = (nl >= 64) ? ~0ull : ((1ull << nl) - 1);
  u64 gm = p.fmask & ~local;
  for (int b = nl; b < 64 && gm; ++b) {
    if (!((gm >> b) & 1)) continue;
    int rb = (rank >> (b - nl)) & 1;
    int need = int((p.fval >> b) & 1);
    if (rb != need) {
      p.skip = true;
      return;
    }
    gm &= ~(1ull << b);
  }
  p.fmask &= local;
  p.fval &= local;
  if (p.type == PRIM_PAIR && (p.xmask & ~local)) sv_fail(SV_ERR_DEVICE, "internal: pair target on a global qubit");
  if (p.type == PRIM_DENSE || p.type == PRIM_GEN) {
    for (int j = 0; j < p.nb; ++j)
      if (p.pos[j] >= nl) sv_fail(SV_ERR_DEVICE, "internal: dense target on a global qubit");
  }
  if ((p.type == PRIM_DIAG || p.type == PRIM_GEND) && p.nb > 0) {
    int keep[16], nk = 0;
    int fixed_bits = 0;  // table index bits pinned by the rank
    int fixed_vals = 0;
    for (int j = 0; j < p.nb; ++j) {
      if (p.pos[j] >= nl) {
        fixed_bits |= 1 << j;
        if ((rank >> (p.pos[j] - nl)) & 1) fixed_vals |= 1 << j;
      } else {
        keep[nk++] = j;
      }
    }
    if (!fixed_bits) return;
    std::vector<cplx> t(size_t(1) << nk);
    for (size_t r = 0; r < t.size(); ++r) {
      int idx = fixed_vals;
      for (int i = 0; i < nk; ++i)
        if ((r >> i) & 1) idx |= 1 << keep[i];
      t[r] = p.m[idx];
    }
    int newpos[16];
    for (int i = 0; i < nk; ++i) newpos[i] = p.pos[keep[i]];
    for (int i = 0; i < nk; ++i) p.pos[i] = newpos[i];
    p.nb = nk;
    p.m = t;
  }
}
