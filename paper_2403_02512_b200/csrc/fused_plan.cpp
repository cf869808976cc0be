// Host planner of the K7 fusion engine: pass construction, register-phase scheduling, gate
// merging, in-tile qubit relabeling and device-op emission (program format: fused.h; kernel:
// fused.cu).
//
// Commutation is decided per bit: a primitive acts on each bit of its support either Z-like
// (diagonal: controls, diagonal-table bits), X-like (a single-target 2x2 of the form aI + bX,
// e.g. RX or the X of a CNOT) or generally.  Two primitives commute when every shared bit is
// Z-like in both or X-like in both -- so RZ slides past CNOT controls and RX past CNOT targets.
#include <algorithm>
#include <functional>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <iterator>
#include <map>
#include <mutex>
#include <string>

#include "fused.h"
#include "prim_util.h"

namespace fused {

// tile bits of a pass (2^b amplitudes staged per CTA); SVB200_TILE_BITS (9..12) for experiments
// physical bits every tile contains (2^LB-amplitude contiguous runs); SVB200_LOW_BITS (2..3)
int low_bits() {
  static const int lb = getenv("SVB200_LOW_BITS") ? std::max(2, std::min(3, atoi(getenv("SVB200_LOW_BITS")))) : 3;
  return lb;
}

// Low physical bits every tile contains (SVB200_TILE_LOW, 3..9): a tile is then 2^LBT-amplitude
// contiguous runs, which is what keeps HBM efficient -- one fused pass streams at 97 % of the copy
// peak when its tile holds bits 3..11 but at 66-71 % when the tile's other bits are all high
// (benchmarks/tile_locality.py: scattered 128-byte lines from many tiles hit DRAM pages out of
// order).  The in-tile relabeling then moves the next gates' qubits onto these low positions.
int tile_low_bits() {
  static const int lb = getenv("SVB200_TILE_LOW") ? std::max(3, std::min(9, atoi(getenv("SVB200_TILE_LOW")))) : 3;
  return lb;
}

int tile_bits() {
  static const int b = getenv("SVB200_TILE_BITS") ? std::max(9, std::min(kMaxB, atoi(getenv("SVB200_TILE_BITS")))) : kMaxB;
  return b;
}
namespace {

// planner view of a primitive: commutation classes (prim_util.h) + fusability
struct Req : PrimReq {
  bool fusable = true;
};

Req requirements(const Prim& p) {
  Req r;
  static_cast<PrimReq&>(r) = prim_requirements(p);
  if (p.type == PRIM_PAIR)
    r.fusable = popcount64(p.xmask) <= kRB;
  else if (p.type == PRIM_DIAG || p.type == PRIM_GEND)
    r.fusable = p.nb <= 6;
  else
    r.fusable = p.nb <= 2;   // DENSE (<= 2 targets) and GEN (<= 2 targets + the psi/lambda bit)
  return r;
}

inline bool commute(const Req& a, const Req& b) { return prims_commute(a, b); }
using Deferred = DeferredSet;
inline void relabel(Prim& p, const int* perm) { relabel_prim(p, perm); }

int mtype_of(const std::vector<cplx>& m) {
  auto re = [](cplx c) { return c.imag() == 0.0; };
  auto im = [](cplx c) { return c.real() == 0.0; };
  if (m[0] == 0.0 && m[3] == 0.0 && m[1] == 1.0 && m[2] == 1.0) return MT_X;
  if (re(m[0]) && re(m[1]) && re(m[2]) && re(m[3])) return MT_REAL;
  if (re(m[0]) && re(m[3]) && im(m[1]) && im(m[2])) return MT_RXLIKE;
  return MT_GENERAL;
}

// choose extra register positions so each bank class {p mod 3} keeps a free thread position
// (avoid: positions to keep off the registers when possible -- the epoch's warp bits)
void fill_regs(std::vector<int>& reg, int b, const std::vector<int>& avoid = {}) {
  auto cls_free = [&](int c, const std::vector<int>& R) {
    for (int p = c; p < b; p += 3)
      if (std::find(R.begin(), R.end(), p) == R.end() && std::find(avoid.begin(), avoid.end(), p) == avoid.end())
        return true;
    return false;
  };
  for (int p = b - 1; p >= 0 && int(reg.size()) < kRB; --p) {
    if (std::find(reg.begin(), reg.end(), p) != reg.end()) continue;
    if (std::find(avoid.begin(), avoid.end(), p) != avoid.end()) continue;
    std::vector<int> trial = reg;
    trial.push_back(p);
    if (cls_free(0, trial) && cls_free(1, trial) && cls_free(2, trial)) reg = trial;
  }
  for (int p = b - 1; p >= 0 && int(reg.size()) < kRB; --p)
    if (std::find(reg.begin(), reg.end(), p) == reg.end()) reg.push_back(p);
}

// Thread-index bits of a phase.  Lanes 0..2 take one non-register position of each residue class
// mod 3 (the swizzle then spreads a 16-byte wavefront over all banks); among the candidates, and
// for the remaining bits, positions the phase's ops test as predicates (controls, diagonal
// patterns: `use`) go to the high, warp-uniform thread bits, so those predicates -- and the
// per-thread X flips they drive -- do not split warps.
// warp: when non-empty (b = 12), the tile positions of the warp-index bits thr[5..7], in order --
// kept from the previous phase so that the phase change stays inside each warp (see build_program).
void make_phase_thr(FPhase& F, const std::vector<int>& reg, int b, const int* use, const std::vector<int>& warp = {}) {
  for (int k = 0; k < kRB; ++k) F.reg[k] = (uint8_t)reg[k];
  auto is_reg = [&](int p) { return std::find(reg.begin(), reg.end(), p) != reg.end(); };
  auto is_warp = [&](int p) { return std::find(warp.begin(), warp.end(), p) != warp.end(); };
  std::vector<int> thr;
  for (int c = 0; c < 3; ++c) {
    int best = -1;
    for (int p = c; p < b; p += 3)
      if (!is_reg(p) && !is_warp(p) && (best < 0 || use[p] < use[best])) best = p;
    if (best >= 0) thr.push_back(best);
  }
  std::vector<int> rest;
  for (int p = 0; p < b; ++p)
    if (!is_reg(p) && !is_warp(p) && std::find(thr.begin(), thr.end(), p) == thr.end()) rest.push_back(p);
  std::stable_sort(rest.begin(), rest.end(), [&](int x, int y) { return use[x] < use[y]; });
  thr.insert(thr.end(), rest.begin(), rest.end());
  thr.insert(thr.end(), warp.begin(), warp.end());
  for (int j = 0; j < b - kRB; ++j) F.thr[j] = (uint8_t)thr[j];
}

// Warp-local phase changes.  A 12-bit tile is 4 register bits x 5 lane bits x 3 warp bits; when two
// consecutive phases put the SAME tile positions on the warp bits, every amplitude stays inside its
// warp across the change, so the shared-memory round trip needs only __syncwarp, not a CTA barrier:
// the warps of a CTA then drift apart and one warp's round trip overlaps other warps' FP64 work
// (a CTA-wide barrier per phase serialises the two).  An epoch's warp positions must hold every
// predicate position of its phases that is not a register (thread predicates on lanes would split
// warps); among such choices the one that lasts for the most following phases wins.  Returns {}
// when the phase's predicates do not fit three warp bits or no choice leaves a lane of each
// residue class mod 3.
bool lanes_ok(const std::vector<int>& reg, const std::vector<int>& warp, int b) {
  for (int c = 0; c < 3; ++c) {
    bool free = false;
    for (int p = c; p < b; p += 3)
      if (std::find(reg.begin(), reg.end(), p) == reg.end() && std::find(warp.begin(), warp.end(), p) == warp.end())
        free = true;
    if (!free) return false;
  }
  return true;
}

std::vector<int> choose_warp_bits(const std::vector<int>& reg_now, const std::vector<u64>& future_dense,
                                  const std::vector<u64>& future_pred, int b) {
  u64 rmask = 0;
  for (int p : reg_now) rmask |= 1ull << p;
  const u64 need = future_pred.empty() ? 0 : (future_pred[0] & ~rmask);
  if (popcount64(need) > 3) return {};
  std::vector<int> base, cand;
  for (int p = 0; p < b; ++p) {
    if ((need >> p) & 1) base.push_back(p);
    else if (!((rmask >> p) & 1)) cand.push_back(p);
  }
  auto run = [&](const std::vector<int>& w) {
    u64 wm = 0;
    for (int p : w) wm |= 1ull << p;
    int r = 0;
    for (size_t j = 0; j < future_dense.size(); ++j) {
      if ((future_dense[j] & wm) || (future_pred[j] & ~future_dense[j] & ~wm)) break;
      ++r;
    }
    return r;
  };
  std::vector<int> best;
  int best_run = -1;
  const size_t m = 3 - base.size();
  std::vector<size_t> idx(m);
  std::function<void(size_t, size_t)> rec = [&](size_t start, size_t depth) {
    if (depth == m) {
      std::vector<int> w = base;
      for (size_t i : idx) w.push_back(cand[i]);
      if (!lanes_ok(reg_now, w, b)) return;
      const int r = run(w);
      if (r > best_run) {
        best_run = r;
        best = w;
      }
      return;
    }
    for (size_t i = start; i < cand.size(); ++i) {
      idx[depth] = i;
      rec(i + 1, depth + 1);
    }
  };
  rec(0, 0);
  return best;
}

// A diagonal table that is 1 on even-parity indices and one constant d on odd ones (IsingZZ
// after phase folding, Z..Z-string rotations).
bool parity_table(const Prim& p) {
  if (p.nb < 1 || p.m.size() != (size_t(1) << p.nb) || p.m[0] != cplx(1.0, 0.0)) return false;
  const cplx d = p.m[1];
  for (size_t i = 0; i < p.m.size(); ++i)
    if (p.m[i] != ((__builtin_popcountll(i) & 1) ? d : cplx(1.0, 0.0))) return false;
  return true;
}

// Register bits an op mixes (acts on non-diagonally), flips, or reads as a whole (bra-kets): a
// diagonal op on any other register bit commutes with it.
int nondiag_regs(const FOp& o) {
  const int cs = o.cs;
  int m = o.fk;   // an attached thread-predicated X flips its bit before the op
  if ((cs >= CS_PAIR1 && cs < CS_PAIR1 + 16) || (cs >= CS_PAIR1D && cs < CS_PAIR1D + 16)) m |= 1 << o.k;
  else if (cs >= CS_SHEAR && cs < CS_SHEAR + 16) m |= 1 << ((cs - CS_SHEAR) / 4);
  else if (cs >= CS_TAN && cs < CS_TAN + 16) m |= 1 << ((cs - CS_TAN) / 4);
  else if (cs >= CS_TAND && cs < CS_TAND + 8) m |= 1 << ((cs - CS_TAND) / 2);
  else if (cs >= CS_XFLIP && cs < CS_XFLIP + 4) m |= 1 << (cs - CS_XFLIP);
  else if (cs >= CS_PAIRGR && cs < CS_PAIRG + 15) m |= cs < CS_PAIRG ? cs - CS_PAIRGR + 1 : cs - CS_PAIRG + 1;
  else if (cs >= CS_DENSE2 && cs < CS_DENSE2 + 6) m |= (1 << (o.xr & 15)) | (1 << (o.xr >> 4));
  else if (cs >= CS_GEN1) m |= 15;
  return m & 15;
}

// Diagonal grouping (pass compiler only): the unpredicated PHASE1 ops of a phase commute with every
// op that touches their bit only diagonally, so each may float inside its window (between the ops
// before and after it that act on its bit non-diagonally).  Windows are covered greedily by as few
// points as possible (sorted by window end); the ops sharing a point become one register diagonal
// (CS_RDIAG: a[r] *= t[r], one complex product per affected register).  m ops on distinct bits then
// cost 4 FP64 ops on (1 - 2^-m) of the amplitudes instead of 2m per amplitude.  The affected-register
// mask is structure (kernel text), the table values (kernel parameters).
void group_phase_diagonals(Program& prog, int first) {
  const int n = int(prog.ops.size()) - first;
  std::vector<int> cand, lo, hi;
  std::vector<int> nd(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    const FOp& o = prog.ops[size_t(first + i)];
    const bool c = o.cs >= CS_PHASE1 && o.cs < CS_PHASE1 + 8 && o.pm == 0 && o.fk == 0;
    nd[size_t(i)] = c ? 0 : nondiag_regs(o);
    if (c) cand.push_back(i);
  }
  if (cand.size() < 2) return;
  for (int i : cand) {
    const int k = (prog.ops[size_t(first + i)].cs - CS_PHASE1) / 2;
    int l = i - 1, h = i + 1;
    while (l >= 0 && !((nd[size_t(l)] >> k) & 1)) --l;
    while (h < n && !((nd[size_t(h)] >> k) & 1)) ++h;
    lo.push_back(l);   // may be placed right before any op index p with l < p <= h (p = n: the end)
    hi.push_back(h);
  }
  std::vector<int> order(cand.size()), point(cand.size(), -1);
  for (size_t j = 0; j < cand.size(); ++j) order[j] = int(j);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return hi[size_t(x)] < hi[size_t(y)]; });
  for (int j : order) {
    if (point[size_t(j)] >= 0) continue;
    const int p = hi[size_t(j)];
    for (int q : order)
      if (point[size_t(q)] < 0 && lo[size_t(q)] < p && p <= hi[size_t(q)]) point[size_t(q)] = p;
  }
  // rebuild the phase: every non-candidate op in order, each point's group inserted before op p
  std::vector<FOp> out;
  out.reserve(size_t(n));
  std::vector<char> is_cand(size_t(n), 0);
  for (int i : cand) is_cand[size_t(i)] = 1;
  auto emit_group = [&](int p) {
    std::vector<int> mem;
    for (size_t j = 0; j < cand.size(); ++j)
      if (point[j] == p) mem.push_back(cand[j]);
    if (mem.empty()) return;
    if (mem.size() == 1) {
      out.push_back(prog.ops[size_t(first + mem[0])]);
      return;
    }
    FOp g = prog.ops[size_t(first + mem[0])];
    cplx tab[16];
    for (int r = 0; r < 16; ++r) tab[r] = cplx(1.0, 0.0);
    u64 aff = 0;   // structure only: a product that happens to be 1 still counts
    for (int i : mem) {
      const FOp& o = prog.ops[size_t(first + i)];
      const int k = (o.cs - CS_PHASE1) / 2, v = (o.cs - CS_PHASE1) % 2;
      for (int r = 0; r < 16; ++r)
        if (((r >> k) & 1) == v) {
          tab[r] *= cplx(o.c[0].x, o.c[0].y);
          aff |= 1ull << r;
        }
    }
    g.kind = FK_DIAGG;
    g.cs = CS_RDIAG;
    g.xm = aff;
    g.tab = int(prog.coef.size());
    for (int r = 0; r < 16; ++r) prog.coef.push_back(make_double2(tab[r].real(), tab[r].imag()));
    out.push_back(g);
  };
  for (int i = 0; i <= n; ++i) {
    emit_group(i);
    if (i < n && !is_cand[size_t(i)]) out.push_back(prog.ops[size_t(first + i)]);
  }
  prog.ops.resize(size_t(first));
  prog.ops.insert(prog.ops.end(), out.begin(), out.end());
}

// Emit the device ops of one phase.  Unconditional X on a register bit is not executed: it is
// absorbed into a flip mask F (logical register index j lives in register j ^ F); later ops of
// the phase are rewritten for F and the phase's store offsets apply it.  Thread-predicated X
// becomes CS_XFLIP (per-thread relabel) and later ops on that bit use the *D cases.  Returns F.
int emit_ops(Program& prog, const std::vector<Prim>& prims, const std::vector<int>& list, const int* tile_pos_of,
             const std::vector<int>& reg) {
  // phys bit -> register index (or -1)
  auto reg_of_phys = [&](int phys) -> int {
    int tp = tile_pos_of[phys];
    if (tp < 0) return -1;
    for (int k = 0; k < kRB; ++k)
      if (reg[k] == tp) return k;
    return -1;
  };
  int F = 0;   // uniform flips (applied here, on the host)
  int D = 0;   // register bits that may carry a per-thread flip (handled by the kernel)
  static const bool shear_on = !(getenv("SVB200_SHEAR") && std::string(getenv("SVB200_SHEAR")) == "0");
  static const bool tan_on = !(getenv("SVB200_TAN") && std::string(getenv("SVB200_TAN")) == "0");
  const bool stable = jit_enabled();
  const int op_first = int(prog.ops.size());
  // A thread-predicated X is not an op of its own: it rides on the next op of the phase (the
  // kernel toggles the flip before that op), saving one dispatch; only a second X arriving
  // before that op, or one left at the end of the phase, is emitted standalone (CS_XFLIP).
  bool pend = false;
  FOp pend_op;
  auto push_op = [&](FOp& o) {
    if (pend && o.cs >= CS_XFLIP && o.cs < CS_XFLIP + 4) {
      prog.ops.push_back(pend_op);   // two flips in a row: the first stands alone
      pend = false;
    }
    if (pend) {
      o.fpm = pend_op.pm;
      o.fpv = pend_op.pv;
      o.fk = 1 << pend_op.k;
      pend = false;
    }
    prog.ops.push_back(o);
  };
  int neg = 0;   // unconditioned rotations emitted as -R(phi'): the phase owes the state a factor (-1)^neg
  for (int i : list) {
    const Prim& p = prims[i];
    FOp op;
    std::memset(&op, 0, sizeof(op));
    // split the fixed pattern into register / non-register parts
    u64 fm = p.fmask;
    for (int bpos = 0; bpos < 64 && fm; ++bpos) {
      if (!((fm >> bpos) & 1)) continue;
      fm &= ~(1ull << bpos);
      const int k = reg_of_phys(bpos);
      const int v = int((p.fval >> bpos) & 1);
      if (k >= 0) {
        op.cm |= uint8_t(1 << k);
        if (v) op.cv |= uint8_t(1 << k);
      } else {
        op.pm |= 1ull << bpos;
        if (v) op.pv |= 1ull << bpos;
      }
    }
    op.cv ^= uint8_t(F & op.cm);   // physical register = logical ^ F
    op.tab = int(prog.coef.size());
    if (p.type == PRIM_GEND) {
      // diagonal generator: table bits anywhere (like DIAGG), only the psi/lambda bit t in registers
      int t = -1;
      for (int bpos = 0; bpos < 64; ++bpos)
        if ((p.xmask >> bpos) & 1) t = reg_of_phys(bpos);
      op.slot = int(prog.gen_slot_of.size());
      prog.gen_slot_of.push_back(p.slot);
      op.nt = uint8_t(p.nb);
      int tflip = 0;
      for (int j = 0; j < p.nb; ++j) {
        const int k = reg_of_phys(p.pos[j]);
        op.treg[j] = k >= 0 ? uint8_t(k) : uint8_t(0xFF);
        op.tphys[j] = uint8_t(p.pos[j]);
        if (k >= 0 && ((F >> k) & 1)) tflip |= 1 << j;
      }
      for (size_t tt = 0; tt < p.m.size(); ++tt) {
        const cplx c = p.m[tt ^ size_t(tflip)];
        prog.coef.push_back(make_double2(c.real(), c.imag()));
      }
      op.v = uint8_t(t);
      op.cs = CS_GEND + t;
      push_op(op);
      continue;
    }
    if (p.type == PRIM_GEN) {
      // adjoint bra-ket: targets and the psi/lambda bit t are register bits; the slot is assigned
      // by build_program (op.slot = index into prog.gen_slot_of, rebased per pass)
      int t = -1;
      for (int bpos = 0; bpos < 64; ++bpos)
        if ((p.xmask >> bpos) & 1) t = reg_of_phys(bpos);
      op.slot = int(prog.gen_slot_of.size());
      prog.gen_slot_of.push_back(p.slot);
      if (p.nb == 1) {
        const int k = reg_of_phys(p.pos[0]);
        std::vector<cplx> g = p.m;
        if ((F >> k) & 1) g = {p.m[3], p.m[2], p.m[1], p.m[0]};   // logical |0> lives in the bit-1 register
        op.cm &= uint8_t(~(1 << k));
        op.cv &= uint8_t(~(1 << k));
        op.k = uint8_t(k);
        op.v = uint8_t(t);
        op.cs = CS_GEN1 + k * 4 + t;
        for (int j = 0; j < 4; ++j) {
          prog.coef.push_back(make_double2(g[j].real(), g[j].imag()));
          op.c[j] = prog.coef.back();
        }
      } else {
        int k0 = reg_of_phys(p.pos[0]), k1 = reg_of_phys(p.pos[1]);
        std::vector<cplx> m = p.m;
        if (k0 > k1) {
          std::swap(k0, k1);
          const int sw[4] = {0, 2, 1, 3};
          for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) m[r * 4 + c] = p.m[sw[r] * 4 + sw[c]];
        }
        const int f = ((F >> k0) & 1) | (((F >> k1) & 1) << 1);
        const uint8_t tb = uint8_t((1 << k0) | (1 << k1));
        op.cm &= uint8_t(~tb);
        op.cv &= uint8_t(~tb);
        op.xr = uint8_t(k0 | (k1 << 4));
        static const uint8_t pairs[6] = {0x10, 0x20, 0x30, 0x21, 0x31, 0x32};
        const int pidx = int(std::find(pairs, pairs + 6, op.xr) - pairs);
        op.v = uint8_t(t);
        op.cs = CS_GEN2 + pidx * 4 + t;
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 4; ++c) {
            const cplx v = m[(r ^ f) * 4 + (c ^ f)];
            prog.coef.push_back(make_double2(v.real(), v.imag()));
          }
      }
      push_op(op);
      continue;
    }
    if (p.type == PRIM_PAIR) {
      for (int bpos = 0; bpos < 64; ++bpos)
        if ((p.xmask >> bpos) & 1) op.xr |= uint8_t(1 << reg_of_phys(bpos));
      const int mt = mtype_of(p.m);
      const bool single = popcount64(op.xr) == 1 && op.cm == op.xr;
      if (single && mt == MT_X && op.pm == 0) {   // unconditional X: relabel, no data movement
        F ^= op.xr;
        continue;
      }
      if (single && mt == MT_X) {                 // thread-predicated X: per-thread relabel
        op.kind = FK_PAIR1;
        op.k = uint8_t(__builtin_ctz(op.xr));
        op.cs = CS_XFLIP + op.k;
        D |= op.xr;
        if (pend) prog.ops.push_back(pend_op);
        pend_op = op;
        pend = true;
        continue;
      }
      std::vector<cplx> m = p.m;
      if (single && (op.cv & op.xr)) {            // i0 sits on the bit-1 register: swap roles
        m = {p.m[3], p.m[2], p.m[1], p.m[0]};
        op.cv = 0;
      }
      if (single && op.cv == 0) {
        op.kind = FK_PAIR1;
        op.k = uint8_t(__builtin_ctz(op.xr));
        op.mtype = uint8_t(mtype_of(m));
      } else {
        op.kind = FK_PAIRG;
        // MT_X stays visible (register-controlled X): the pass compiler turns it into register
        // renaming instead of FP64 arithmetic; the interpreter runs it as the real 2x2 it is
        op.mtype = uint8_t(mt == MT_X ? MT_X : (mt == MT_REAL ? MT_REAL : MT_GENERAL));
      }
      for (int j = 0; j < 4; ++j) prog.coef.push_back(make_double2(m[j].real(), m[j].imag()));
    } else if (p.type == PRIM_DIAG && p.nb == 0 && popcount64(op.cm) <= 1) {
      if (op.cm == 0) {
        op.kind = FK_SCALAR;
      } else {
        op.kind = FK_PHASE1;
        op.k = uint8_t(__builtin_ctz(op.cm));
        op.v = uint8_t(op.cv ? 1 : 0);
      }
      prog.coef.push_back(make_double2(p.m[0].real(), p.m[0].imag()));
    } else if (p.type == PRIM_DIAG && op.cm == 0 && parity_table(p)) {
      // phase d on the odd-parity half of the table bits: register bits form the case mask,
      // the rest enter through the thread's physical base (xm); uniform flips fix the offset v
      op.kind = FK_PARITY;
      int M = 0, v = 0;
      for (int j = 0; j < p.nb; ++j) {
        const int k = reg_of_phys(p.pos[j]);
        if (k >= 0) {
          M |= 1 << k;
          v ^= (F >> k) & 1;
        } else {
          op.xm |= 1ull << p.pos[j];
        }
      }
      op.v = uint8_t(v);
      op.cs = CS_PARITY + M;
      prog.coef.push_back(make_double2(p.m[1].real(), p.m[1].imag()));
      op.c[0] = prog.coef.back();
      push_op(op);
      continue;
    } else if (p.type == PRIM_DIAG) {
      op.kind = FK_DIAGG;
      op.nt = uint8_t(p.nb);
      int tflip = 0;
      for (int j = 0; j < p.nb; ++j) {
        const int k = reg_of_phys(p.pos[j]);
        op.treg[j] = k >= 0 ? uint8_t(k) : uint8_t(0xFF);
        op.tphys[j] = uint8_t(p.pos[j]);
        if (k >= 0 && ((F >> k) & 1)) tflip |= 1 << j;
      }
      for (size_t t = 0; t < p.m.size(); ++t) {
        const cplx c = p.m[t ^ size_t(tflip)];
        prog.coef.push_back(make_double2(c.real(), c.imag()));
      }
    } else {
      op.kind = FK_DENSE2;
      int k0 = reg_of_phys(p.pos[0]), k1 = reg_of_phys(p.pos[1]);
      // matrix index bit 0 <-> pos[0] (ascending physical); kernel wants bit 0 <-> lower register index
      std::vector<cplx> m = p.m;
      if (k0 > k1) {
        std::swap(k0, k1);
        const int sw[4] = {0, 2, 1, 3};
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 4; ++c) m[r * 4 + c] = p.m[sw[r] * 4 + sw[c]];
      }
      const int f = ((F >> k0) & 1) | (((F >> k1) & 1) << 1);
      std::vector<cplx> mf(16);
      for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) mf[r * 4 + c] = m[(r ^ f) * 4 + (c ^ f)];
      op.xr = uint8_t(k0 | (k1 << 4));
      const uint8_t tb = uint8_t((1 << k0) | (1 << k1));   // targets are enumerated by the kernel
      op.cm &= uint8_t(~tb);
      op.cv &= uint8_t(~tb);
      for (auto& c : mf) prog.coef.push_back(make_double2(c.real(), c.imag()));
    }
    const bool dyn = ((D >> op.k) & 1) != 0;
    if (shear_on && op.kind == FK_PAIR1 && (op.mtype == MT_REAL || op.mtype == MT_RXLIKE)) {
      // rotation R(phi) = [[c, -s], [s, c]] (RY type) or [[c, -is], [-is, c]] (RX type)?
      cplx m[4];
      for (int j = 0; j < 4; ++j) m[j] = cplx(prog.coef[op.tab + j].x, prog.coef[op.tab + j].y);
      const bool rx = op.mtype == MT_RXLIKE;
      const bool rot = rx ? (m[0] == m[3] && m[1] == m[2]) : (m[0] == m[3] && m[1] == -m[2]);
      double c = m[0].real(), sn = rx ? -m[1].imag() : m[2].real();
      // the runtime pass compiler keys kernels on structure, so there the choice may not depend on
      // the angle: conditioned rotations always keep the 2x2 form
      if (rot && (op.pm == 0 || (c >= 0.0 && !stable))) {
        if (c < 0.0) {   // R(phi) = -R(phi -+ pi): the sign is global for an unconditioned op
          c = -c;
          sn = -sn;
          neg ^= 1;
        }
        if (stable && tan_on) {
          // scaled form (2 FMAs per real pair): R/c for |phi| <= pi/4, else R/s; the factor is
          // owed to the state until absorb_pass_scale folds the pass's product into one op
          bool cot = std::fabs(sn) > c;
          // hysteresis: the form is structure (part of the generated kernel), so a re-plan of the
          // same circuit with new angles keeps the previous plan's form while its coefficient stays
          // within kTanBand (|phi| <= 68 deg as TAN, >= 22 deg as COT) -- no recompilation for
          // small parameter updates; beyond the band the pass is recompiled once for the new form
          const size_t idx = prog.tan_forms.size();
          if (idx < prog.tan_hint.size()) {
            const bool hc = prog.tan_hint[idx] != 0;
            if (hc != cot && std::fabs(hc ? c / sn : sn / c) <= kTanBand) cot = hc;
          }
          prog.tan_forms.push_back(cot ? 1 : 0);
          // RX type is symmetric under a per-thread flip; RY type on a flippable bit: CS_TAND
          op.cs = (!rx && dyn) ? CS_TAND + op.k * 2 + (cot ? 1 : 0) : CS_TAN + op.k * 4 + (rx ? 1 : 0) + (cot ? 2 : 0);
          op.c[0] = make_double2(cot ? c / sn : sn / c, cot ? sn : c);
          op.c[1] = make_double2(c, 0.0);
          op.c[2] = make_double2(sn, rx ? 1.0 : 0.0);
          push_op(op);
          continue;
        }
        op.cs = CS_SHEAR + op.k * 4 + (rx ? SH_RX : (dyn ? SH_RYD : SH_RY));   // RX is symmetric under flips
        op.c[0] = make_double2(-sn / (1.0 + c), sn);
        op.c[1] = make_double2(c, 0.0);   // (c, s) kept for a later conversion back to the 2x2 form
        op.c[2] = make_double2(sn, rx ? 1.0 : 0.0);
        push_op(op);
        continue;
      }
    }
    switch (op.kind) {
      case FK_PAIR1: op.cs = (dyn ? CS_PAIR1D : CS_PAIR1) + op.k * 4 + op.mtype; break;
      case FK_PHASE1: op.cs = (dyn ? CS_PHASE1D : CS_PHASE1) + op.k * 2 + op.v; break;
      case FK_SCALAR: op.cs = CS_SCALAR; break;
      case FK_PAIRG: op.cs = (op.mtype == MT_REAL || op.mtype == MT_X ? CS_PAIRGR : CS_PAIRG) + op.xr - 1; break;
      case FK_DIAGG: op.cs = CS_DIAGG; break;
      default: {
        static const uint8_t pairs[6] = {0x10, 0x20, 0x30, 0x21, 0x31, 0x32};
        op.cs = CS_DENSE2 + int(std::find(pairs, pairs + 6, op.xr) - pairs);
      }
    }
    if (op.kind != FK_DIAGG && op.kind != FK_DENSE2) {   // hot kinds carry their coefficients inline
      const int nc = (op.kind == FK_PAIR1 || op.kind == FK_PAIRG) ? 4 : 1;
      for (int j = 0; j < nc; ++j) op.c[j] = prog.coef[op.tab + j];
    }
    push_op(op);
  }
  if (pend) prog.ops.push_back(pend_op);
  prog.owed_neg ^= neg;   // resolved once per program (absorb_rotation_signs)
  if (stable) group_phase_diagonals(prog, op_first);
  return F;
}

// Unconditioned rotations emitted as -R(phi') leave the state owing a global factor -1 per such
// rotation.  A global sign commutes with everything (and cancels in every psi/lambda bra-ket, both
// halves carry it), so the program's net sign is absorbed ONCE, into the coefficients of any
// unconditioned 2x2 / scalar op of the program; only a program without one turns its last
// unconditioned shear back into a 2x2 carrying the sign.  With the runtime pass compiler the
// choice must not depend on the angles (kernels are keyed on structure), so the conversion then
// happens whether the owed sign is +1 or -1.
void absorb_rotation_signs(Program& prog, bool stable) {
  const double sg = prog.owed_neg ? -1.0 : 1.0;
  auto absorber = [](const FOp& o) {
    if (o.pm != 0) return false;
    if (o.cs == CS_SCALAR) return true;
    const bool p1 = (o.cs >= CS_PAIR1 && o.cs < CS_PAIR1 + 16) || (o.cs >= CS_PAIR1D && o.cs < CS_PAIR1D + 16);
    return p1 && o.mtype != MT_X && (o.cs % 4) != 3;
  };
  for (FOp& o : prog.ops)
    if (absorber(o)) {
      if (sg < 0) {
        const int nc = o.cs == CS_SCALAR ? 1 : 4;
        for (int j = 0; j < nc; ++j) {
          o.c[j] = make_double2(-o.c[j].x, -o.c[j].y);
          prog.coef[o.tab + j] = o.c[j];
        }
      }
      prog.owed_neg = 0;
      return;
    }
  if (!(sg < 0 || stable)) return;
  for (int oi = int(prog.ops.size()) - 1; oi >= 0; --oi) {
    FOp& o = prog.ops[oi];
    if (o.pm != 0 || o.cs < CS_SHEAR || o.cs >= CS_SHEAR + 16) continue;
    const double c = o.c[1].x, sn = o.c[2].x;
    const bool rx = o.c[2].y != 0.0;
    const int k = (o.cs - CS_SHEAR) / 4;
    // RX-type 2x2s are symmetric under a per-thread flip of their bit; RY-type ones on a flipped
    // bit (SH_RYD) need the *D form
    const bool dyn = (o.cs - CS_SHEAR) % 4 == SH_RYD;
    std::array<cplx, 4> mm;
    if (rx)
      mm = {cplx(c, 0), cplx(0, -sn), cplx(0, -sn), cplx(c, 0)};     // [[c, -is], [-is, c]]
    else
      mm = {cplx(c, 0), cplx(-sn, 0), cplx(sn, 0), cplx(c, 0)};      // [[c, -s], [s, c]]
    o.tab = int(prog.coef.size());
    for (int j = 0; j < 4; ++j) {
      prog.coef.push_back(make_double2(sg * mm[j].real(), sg * mm[j].imag()));
      o.c[j] = prog.coef.back();
    }
    o.mtype = uint8_t(rx ? MT_RXLIKE : MT_REAL);
    o.cs = (dyn ? CS_PAIR1D : CS_PAIR1) + k * 4 + o.mtype;
    prog.owed_neg = 0;
    return;
  }
  if (sg < 0) sv_fail(SV_ERR_DEVICE, "internal: unabsorbed rotation sign");
}

// Form memory of the scaled rotations, per circuit structure (see emit_ops): the last plan's
// TAN/COT choice of every scaled rotation, in emission order.
std::mutex g_tan_mu;
std::map<u64, std::vector<uint8_t>> g_tan_forms;

u64 structure_key(int nl, const std::vector<Prim>& prims, bool remap, bool pin_top) {
  u64 h = 1469598103934665603ull;
  auto mix = [&](u64 v) {
    h ^= v;
    h *= 1099511628211ull;
  };
  mix(u64(nl) | (u64(remap) << 8) | (u64(pin_top) << 9));
  for (const Prim& p : prims) {
    mix(u64(p.type) | (u64(p.nb) << 8) | (u64(p.m.size()) << 16));
    mix(p.fmask);
    mix(p.fval);
    mix(p.xmask);
    for (int t = 0; t < p.nb; ++t) mix(u64(p.pos[t]));
  }
  return h;
}

// Scaled rotations (CS_TAN) apply R/f with f = cos(phi) or sin(phi): after them the stored state
// is the true one divided by the product of their factors.  The pass restores it before its store:
// the product S is multiplied into one unconditioned op of the pass that takes any coefficient
// (a SCALAR or a non-X PAIR1 on every amplitude), or else the pass's last scaled rotation goes back
// to the full 2x2 form carrying S.  The choice depends only on op kinds (structure), never on
// values, so generated kernels stay keyed on structure.  A bra-ket op in between sees psi and
// lambda both scaled by the running factor r: its result is corrected by 1 / r^2 on the host
// (Program::gen_scale).  Factors are >= 1/sqrt(2) each, so S stays far from underflow within a
// pass.
void absorb_pass_scale(Program& prog, const FPassArgs& A) {
  auto is_tan = [](const FOp& o) { return o.cs >= CS_TAN && o.cs < CS_TAND + 8; };
  double S = 1.0;
  int last = -1, absorber = -1;
  for (int oi = A.op_begin; oi < A.op_end; ++oi) {
    const FOp& o = prog.ops[oi];
    if (is_tan(o)) {
      S *= o.c[0].y;
      last = oi;
    } else if (absorber < 0 && o.pm == 0 && o.cs < CS_GEN1) {
      const bool p1 = (o.cs >= CS_PAIR1 && o.cs < CS_PAIR1 + 16) || (o.cs >= CS_PAIR1D && o.cs < CS_PAIR1D + 16);
      if (o.cs == CS_SCALAR || (p1 && o.mtype != MT_X && (o.cs % 4) != 3)) absorber = oi;
    }
  }
  if (last < 0) return;
  double Sx = 1.0;   // product of the factors of every scaled rotation but the last (no division)
  for (int oi = A.op_begin; oi < A.op_end; ++oi)
    if (oi != last && is_tan(prog.ops[oi])) Sx *= prog.ops[oi].c[0].y;
  const bool convert = absorber < 0;
  if (convert) {
    // the last scaled rotation becomes the full rotation times the other rotations' factors
    FOp& o = prog.ops[last];
    const double c = o.c[1].x, sn = o.c[2].x;
    const bool rx = o.c[2].y != 0.0;
    const bool dyn = o.cs >= CS_TAND;
    const int k = dyn ? (o.cs - CS_TAND) / 2 : (o.cs - CS_TAN) / 4;
    std::array<cplx, 4> mm;
    if (rx) mm = {cplx(c, 0), cplx(0, -sn), cplx(0, -sn), cplx(c, 0)};
    else mm = {cplx(c, 0), cplx(-sn, 0), cplx(sn, 0), cplx(c, 0)};
    o.tab = int(prog.coef.size());
    for (int j = 0; j < 4; ++j) {
      prog.coef.push_back(make_double2(Sx * mm[j].real(), Sx * mm[j].imag()));
      o.c[j] = prog.coef.back();
    }
    o.mtype = uint8_t(rx ? MT_RXLIKE : MT_REAL);
    o.kind = FK_PAIR1;
    o.cs = (dyn ? CS_PAIR1D : CS_PAIR1) + k * 4 + o.mtype;
    absorber = last;
  } else {
    FOp& o = prog.ops[absorber];
    const int nc = o.cs == CS_SCALAR ? 1 : 4;
    for (int j = 0; j < nc; ++j) {
      o.c[j] = make_double2(S * o.c[j].x, S * o.c[j].y);
      prog.coef[o.tab + j] = o.c[j];
    }
  }
  // running factor of the stored state at each bra-ket
  if (prog.gen_scale.size() < prog.gen_slot_of.size()) prog.gen_scale.resize(prog.gen_slot_of.size(), 1.0);
  double r = 1.0;
  for (int oi = A.op_begin; oi < A.op_end; ++oi) {
    const FOp& o = prog.ops[oi];
    if (is_tan(o)) r /= o.c[0].y;
    else if (oi == absorber) r *= convert ? Sx : S;
    else if (o.cs >= CS_GEN1) prog.gen_scale[size_t(A.gen_base + o.slot)] = 1.0 / (r * r);
  }
}

// Can prim i be folded into prim j (j runs right before i on every bit i touches)?
bool mergeable(const Prim& j, const Prim& i) {
  if (j.type != i.type || j.fmask != i.fmask || j.fval != i.fval) return false;
  if (i.type == PRIM_PAIR) return j.xmask == i.xmask && popcount64(i.xmask) == 1;
  if (i.type == PRIM_DIAG) {
    if (i.nb != j.nb) return false;
    for (int t = 0; t < i.nb; ++t)
      if (i.pos[t] != j.pos[t]) return false;
    return true;
  }
  return false;
}

// Merging two rotations about different axes yields a general 2x2 (16 FP64 ops per amplitude
// pair) where the two rotations cost 12 (two 3-shear rotations): only merge a PAIR into a PAIR
// when the product is no more general than the more general of the two.
bool merge_pays(const Prim& j, const Prim& i) {
  if (i.type != PRIM_PAIR) return true;
  const std::vector<cplx> a = i.m, b = j.m;
  const std::vector<cplx> m = {a[0] * b[0] + a[1] * b[2], a[0] * b[1] + a[1] * b[3], a[2] * b[0] + a[3] * b[2],
                               a[2] * b[1] + a[3] * b[3]};
  auto general = [](const std::vector<cplx>& x) { return mtype_of(x) == MT_GENERAL; };
  return !general(m) || general(a) || general(b);
}

void merge_into(Prim& j, const Prim& i) {
  if (i.type == PRIM_PAIR) {   // apply j then i: M = Mi * Mj
    const std::vector<cplx> a = i.m, b = j.m;
    j.m = {a[0] * b[0] + a[1] * b[2], a[0] * b[1] + a[1] * b[3], a[2] * b[0] + a[3] * b[2], a[2] * b[1] + a[3] * b[3]};
  } else {
    for (size_t t = 0; t < j.m.size(); ++t) j.m[t] *= i.m[t];
  }
}

// List-schedule a pass's prims into register phases.  Prims are reordered only past prims
// they commute with; each phase picks up to 4 register bits and runs every ready prim whose
// dense bits fit, to a fixpoint.  A prim that immediately follows a compatible prim on all of
// its bits is multiplied into it (one op instead of two).
// Returns (register-bit mask in physical positions, prims in execution order) per phase.
std::vector<std::pair<u64, std::vector<int>>> schedule_phases(std::vector<Prim>& prims, const std::vector<int>& list,
                                                              int64_t& merged) {
  const int L = int(list.size());
  std::vector<Req> rq(L);
  for (int i = 0; i < L; ++i) rq[i] = requirements(prims[list[i]]);
  std::vector<int> npred(L, 0);
  std::vector<std::vector<int>> succ(L);
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < i; ++j)
      if (!commute(rq[i], rq[j])) {
        succ[j].push_back(i);
        npred[i]++;
      }
  std::vector<char> done(L, 0);
  int ndone = 0;
  std::vector<std::vector<int>> preds;   // built on first use by the register-set search
  std::vector<std::pair<u64, std::vector<int>>> phases;
  while (ndone < L) {
    u64 R = 0;
    std::vector<int> order;
    int last_on[64];   // per bit: index (into list) of the last op of this phase touching it
    for (int b = 0; b < 64; ++b) last_on[b] = -1;
    for (;;) {
      bool progress = false;
      for (int i = 0; i < L; ++i) {
        if (done[i] || npred[i] != 0) continue;
        if ((rq[i].dense & ~R) != 0) continue;
        done[i] = 1;
        ++ndone;
        for (int s : succ[i]) npred[s]--;
        progress = true;
        // merge into the op that last touched all of this prim's bits, if compatible
        int cand = -2;
        for (int b = 0; b < 64; ++b)
          if ((rq[i].support >> b) & 1) {
            if (cand == -2) cand = last_on[b];
            else if (cand != last_on[b]) cand = -1;
          }
        static const bool merge_on = !(getenv("SVB200_MERGE") && std::string(getenv("SVB200_MERGE")) == "0");
        if (merge_on && cand >= 0 && rq[cand].support == rq[i].support &&
            mergeable(prims[list[cand]], prims[list[i]]) && merge_pays(prims[list[cand]], prims[list[i]])) {
          merge_into(prims[list[cand]], prims[list[i]]);
          ++merged;
          continue;
        }
        order.push_back(list[i]);
        for (int b = 0; b < 64; ++b)
          if ((rq[i].support >> b) & 1) last_on[b] = i;
      }
      if (progress) continue;
      // stuck with an empty register set (a new phase): choose the whole set at once -- every subset
      // of at most kRB of the bits the remaining ops need densely, scored by the ops it lets this
      // phase run (transitively; predecessors precede in list order, so one ordered sweep
      // simulates it); ties keep the smaller set, then the first found
      static const bool search = !(getenv("SVB200_PHASE_SEARCH") && std::string(getenv("SVB200_PHASE_SEARCH")) == "0");
      if (search && R == 0) {
        u64 need = 0;
        for (int i = 0; i < L; ++i)
          if (!done[i]) need |= rq[i].dense;
        std::vector<int> bits;
        for (int b = 0; b < 64; ++b)
          if ((need >> b) & 1) bits.push_back(b);
        if (!bits.empty() && bits.size() <= 16) {
          if (preds.empty()) {
            preds.assign(L, {});
            for (int j = 0; j < L; ++j)
              for (int s : succ[j]) preds[s].push_back(j);
          }
          // ops a register set lets a phase run after the ops in `base` (transitively, one sweep)
          const int nb = int(bits.size());
          std::vector<u64> sets;
          for (u64 m = 1; m < (1ull << nb); ++m) {
            if (popcount64(m) > kRB) continue;
            u64 Rm = 0;
            for (int t = 0; t < nb; ++t)
              if ((m >> t) & 1) Rm |= 1ull << bits[t];
            sets.push_back(Rm);
          }
          auto run = [&](const std::vector<char>& base, u64 Rm, std::vector<char>& sim) {
            int g = 0;
            for (int i = 0; i < L; ++i) {
              sim[i] = base[i];
              if (base[i] || (rq[i].dense & ~Rm)) continue;
              bool ok = true;
              for (int j : preds[i])
                if (!sim[j]) {
                  ok = false;
                  break;
                }
              if (ok) {
                sim[i] = 1;
                ++g;
              }
            }
            return g;
          };
          std::vector<char> sim(L), sim2(L);
          std::vector<std::pair<int, int>> first;   // (ops, set index)
          for (size_t k = 0; k < sets.size(); ++k) first.push_back({run(done, sets[k], sim), int(k)});
          std::stable_sort(first.begin(), first.end(), [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
            if (x.first != y.first) return x.first > y.first;
            return popcount64(sets[size_t(x.second)]) < popcount64(sets[size_t(y.second)]);
          });
          // SVB200_PHASE_BEAM=k > 1: two-phase lookahead over the k best first sets (ops of this phase +
          // the best next phase); measured 172 -> 170 phases on the bench circuit for 2.5x planning time
          static const int beam = getenv("SVB200_PHASE_BEAM") ? std::max(1, atoi(getenv("SVB200_PHASE_BEAM"))) : 1;
          u64 bestR = 0;
          int bestg = -1, bestg1 = -1;
          for (int c = 0; c < int(first.size()) && c < beam && first[size_t(c)].first > 0; ++c) {
            const u64 R1 = sets[size_t(first[size_t(c)].second)];
            const int g1 = run(done, R1, sim);
            int g2 = 0;
            if (beam > 1)
              for (u64 R2 : sets) g2 = std::max(g2, run(sim, R2, sim2));
            if (g1 + g2 > bestg || (g1 + g2 == bestg && g1 > bestg1)) {
              bestg = g1 + g2;
              bestg1 = g1;
              bestR = R1;
            }
          }
          bestg = bestg1;
          if (bestg > 0) {
            R = bestR;
            continue;
          }
        }
      }
      // stuck: widen the register set by the ready op whose bits unlock the most work in this
      // phase (simulated: ops that become runnable, transitively), first ready op on ties
      static const bool greedy = getenv("SVB200_PHASE_GREEDY") && std::string(getenv("SVB200_PHASE_GREEDY")) == "1";
      int pick = -1, best = -1;
      std::vector<int> np2;
      std::vector<char> dn2;
      for (int i = 0; i < L; ++i) {
        if (done[i] || npred[i] != 0 || popcount64(R | rq[i].dense) > kRB) continue;
        if (greedy) {
          pick = i;
          break;
        }
        const u64 R2 = R | rq[i].dense;
        np2 = npred;
        dn2 = done;
        int gain = 0;
        for (bool again = true; again;) {
          again = false;
          for (int j = 0; j < L; ++j) {
            if (dn2[j] || np2[j] != 0 || (rq[j].dense & ~R2) != 0) continue;
            dn2[j] = 1;
            ++gain;
            for (int s2 : succ[j]) np2[s2]--;
            again = true;
          }
        }
        // prefer more unlocked work per new register bit
        const int cost = popcount64(rq[i].dense & ~R);
        const int score = cost ? gain * 4 / cost : gain * 16;
        if (score > best) {
          best = score;
          pick = i;
        }
      }
      if (pick < 0) break;
      R |= rq[pick].dense;
    }
    phases.push_back({R, order});
  }
  return phases;
}

}  // namespace

// One planning run with tail-deferral threshold defer_k (0: off) and the scaled-rotation form hints.
Program build_program_k(int nl, const std::vector<Prim>& prims_in, bool remap, bool pin_top, int defer_k,
                        const std::vector<uint8_t>& hint) {
  Program prog;
  std::vector<Prim> P = prims_in;
  prog.n_prims_in = int64_t(P.size());
  prog.tan_hint = hint;
  const int b = std::min(tile_bits(), nl);
  const int LB = std::min(low_bits(), nl);   // physical bits the direct store's 8-lane groups cover
  const int LBT = std::max(LB, std::min(tile_low_bits(), b - 3));   // physical bits every tile contains
  const u64 low = (1ull << LBT) - 1;
  std::vector<int> perm_total(nl);
  for (int p = 0; p < nl; ++p) perm_total[p] = p;
  std::vector<Req> req(P.size());
  for (size_t i = 0; i < P.size(); ++i) req[i] = requirements(P[i]);
  std::vector<int> remaining(P.size());
  for (size_t i = 0; i < P.size(); ++i) remaining[i] = int(i);
  while (!remaining.empty()) {
    const int p0 = remaining[0];
    if (!req[p0].fusable || nl < 5) {
      prog.steps.push_back({false, int(prog.singles.size())});
      prog.singles.push_back(P[p0]);
      remaining.erase(remaining.begin());
      continue;
    }
    // ---- choose the pass: greedy over the dependency order, from several starting points ----
    // Candidate s: the first s remaining prims may only join if they fit the bits chosen so far
    // (the register set grows from prim s onward); the candidate taking the most prims wins
    // (s = 0 is the plain greedy pass).
    u64 B = low;
    std::vector<int> take, rest;
    {
      static const int n_starts = getenv("SVB200_PASS_STARTS") ? std::max(1, atoi(getenv("SVB200_PASS_STARTS"))) : 48;
      std::vector<size_t> starts = {0};
      for (size_t k = 1; k < remaining.size() && int(starts.size()) < n_starts; ++k)
        if (req[remaining[k]].dense & ~low) starts.push_back(k);
      size_t best_taken = 0;
      static const int pass_score = getenv("SVB200_PASS_SCORE") ? atoi(getenv("SVB200_PASS_SCORE")) : 0;
      struct Cand {
        u64 Bc;
        std::vector<int> tk, rs;
      };
      std::vector<Cand> cands;
      for (size_t s0 : starts) {
        u64 Bc = low;
        Deferred defc;
        std::vector<int> tk, rs;
        int ng = 0;
        for (size_t k = 0; k < remaining.size(); ++k) {
          const int i = remaining[k];
          const Req& r = req[i];
          const bool gen = P[i].type == PRIM_GEN || P[i].type == PRIM_GEND;
          const bool grow_ok = k >= s0 ? popcount64(Bc | r.dense) <= b : (r.dense & ~Bc) == 0;
          const bool ok = r.fusable && int(tk.size()) < kMaxSmemOps && !defc.blocks(r) && grow_ok &&
                          (!gen || ng < kMaxGens);
          if (ok) {
            Bc |= r.dense;
            tk.push_back(i);
            ng += gen ? 1 : 0;
          } else {
            defc.add(r);
            rs.push_back(i);
          }
        }
        if (pass_score > 0) {
          cands.push_back({Bc, std::move(tk), std::move(rs)});
          continue;
        }
        if (tk.size() > best_taken) {
          best_taken = tk.size();
          B = Bc;
          take.swap(tk);
          rest.swap(rs);
        }
      }
      if (pass_score > 0) {
        // SVB200_PASS_SCORE=k: schedule the k largest candidates (on a copy: scheduling merges
        // prims) and keep the one with the most prims per cost (phases + 1.8 for the pass itself)
        std::stable_sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) { return x.tk.size() > y.tk.size(); });
        double best_score = -1.0;
        size_t best_i = 0;
        for (size_t ci = 0; ci < cands.size() && int(ci) < pass_score; ++ci) {
          std::vector<Prim> Pc = P;
          int64_t mg = 0;
          const auto sc = schedule_phases(Pc, cands[ci].tk, mg);
          const double score = double(cands[ci].tk.size()) / (double(sc.size()) + 1.8);
          if (score > best_score) {
            best_score = score;
            best_i = ci;
          }
        }
        B = cands[best_i].Bc;
        take.swap(cands[best_i].tk);
        rest.swap(cands[best_i].rs);
      }
    }
    for (int p = 0; p < nl && popcount64(B) < b; ++p) B |= 1ull << p;   // fill: longest contiguous runs
    // ---- emit ----
    FPassArgs A;
    std::memset(&A, 0, sizeof(A));
    A.b = b;
    A.nthr = b - kRB;
    int tile_pos_of[64];
    for (int i = 0; i < 64; ++i) tile_pos_of[i] = -1;
    int j = 0;
    for (int p = 0; p < nl; ++p)
      if ((B >> p) & 1) {
        A.tpos[j] = (unsigned char)p;
        tile_pos_of[p] = j++;
      }
    A.n_tiles = 1ull << (nl - b);
    A.phase_begin = int(prog.phases.size());
    A.gen_base = int(prog.gen_slot_of.size());
    auto sched = schedule_phases(P, take, prog.n_prims_merged);
    // Tail deferral: a last phase holding only a few ops costs a whole shared-memory round trip
    // (and often the op-free store phase after it); when more passes follow anyway, its ops move to
    // the next pass, whose first phases usually hold their bits.  Nothing left in this pass depends
    // on them (they were scheduled last), and ops merged into them stay merged.
    static const bool defer_loop = getenv("SVB200_DEFER_LOOP") && std::string(getenv("SVB200_DEFER_LOOP")) == "1";
    while (defer_k > 0 && sched.size() >= 2 && !rest.empty() && int(sched.back().second.size()) <= defer_k) {
      std::vector<int> back = sched.back().second;
      sched.pop_back();
      std::sort(back.begin(), back.end());
      std::vector<int> merged;
      std::merge(rest.begin(), rest.end(), back.begin(), back.end(), std::back_inserter(merged));
      rest.swap(merged);
      if (!defer_loop) break;
    }
    std::vector<u64> dense_tile(sched.size(), 0);   // register (dense) tile positions per phase
    std::vector<u64> pred_tile(sched.size(), 0);    // tile positions its ops test per thread
    for (size_t k = 0; k < sched.size(); ++k) {
      for (int p = 0; p < 64; ++p)
        if ((sched[k].first >> p) & 1) dense_tile[k] |= 1ull << tile_pos_of[p];
      for (int i : sched[k].second) {
        for (int p = 0; p < 64; ++p)
          if (((P[i].fmask >> p) & 1) && tile_pos_of[p] >= 0) pred_tile[k] |= 1ull << tile_pos_of[p];
        if (P[i].type == PRIM_DIAG)
          for (int j = 0; j < P[i].nb; ++j)
            if (tile_pos_of[P[i].pos[j]] >= 0) pred_tile[k] |= 1ull << tile_pos_of[P[i].pos[j]];
      }
    }
    // SVB200_WARP_LOCAL=1 (off by default): on the 30-qubit bench circuit only 15 of 141 phase
    // changes qualify once predicates must stay off the lanes, and the run measured 0.43 s vs 0.41 s
    static const bool warp_local = getenv("SVB200_WARP_LOCAL") && std::string(getenv("SVB200_WARP_LOCAL")) == "1";
    std::vector<int> W;   // warp-bit positions of the current epoch
    // Group-local phase changes: tile positions no phase of the pass needs as a register stay on the
    // top thread bits for the whole pass (at most two, highest first), so each 128-thread half (one
    // fixed bit) or 64-thread quarter (two) of the CTA holds the same amplitudes in every phase and
    // its round trips synchronise only that group (named barrier, fused_jit.cpp) -- the groups
    // drift apart and one group's round trip overlaps the others' arithmetic.
    std::vector<int> fixed;
    static const bool group_on = !(getenv("SVB200_GROUP_BAR") && std::string(getenv("SVB200_GROUP_BAR")) == "0");
    if (group_on && b == kMaxB && !warp_local) {
      u64 used = 0;
      for (u64 d : dense_tile) used |= d;
      for (int p = b - 1; p >= 3 && fixed.size() < 2; --p)
        if (!((used >> p) & 1)) fixed.push_back(p);
      std::reverse(fixed.begin(), fixed.end());   // make_phase_thr puts them last, in this order
    }
    for (size_t k = 0; k < sched.size(); ++k) {
      const auto& ph = sched[k];
      std::vector<int> R;
      for (int p = 0; p < 64; ++p)
        if ((ph.first >> p) & 1) R.push_back(tile_pos_of[p]);
      int use[kMaxB] = {0};   // predicate tests per tile position in this phase
      for (int i : ph.second) {
        for (int p = 0; p < 64; ++p)
          if (((P[i].fmask >> p) & 1) && tile_pos_of[p] >= 0) ++use[tile_pos_of[p]];
        if (P[i].type == PRIM_DIAG)   // table bits off the registers are per-thread inputs too
          for (int j = 0; j < P[i].nb; ++j)
            if (tile_pos_of[P[i].pos[j]] >= 0) ++use[tile_pos_of[P[i].pos[j]]];
      }
      if (warp_local && b == kMaxB) {
        u64 wm = 0;
        for (int p : W) wm |= 1ull << p;
        // the epoch continues if its warp positions stay off this phase's registers and hold all of
        // its off-register predicates, and the register filler can avoid them
        bool keep = !W.empty() && !(dense_tile[k] & wm) && !(pred_tile[k] & ~dense_tile[k] & ~wm);
        if (keep) {
          std::vector<int> Rf = R;
          fill_regs(Rf, b, W);
          for (int p : W) keep = keep && std::find(Rf.begin(), Rf.end(), p) == Rf.end();
          keep = keep && lanes_ok(Rf, W, b);
        }
        if (!keep)
          W = choose_warp_bits(R, std::vector<u64>(dense_tile.begin() + long(k), dense_tile.end()),
                               std::vector<u64>(pred_tile.begin() + long(k), pred_tile.end()), b);
        fill_regs(R, b, W);
        for (int p : W)
          if (std::find(R.begin(), R.end(), p) != R.end()) W.clear();
        if (!W.empty() && !lanes_ok(R, W, b)) W.clear();
      } else if (!fixed.empty()) {
        std::vector<int> Rf = R;
        fill_regs(Rf, b, fixed);
        bool ok = lanes_ok(Rf, fixed, b);
        for (int p : fixed) ok = ok && std::find(Rf.begin(), Rf.end(), p) == Rf.end();
        if (ok) {
          // keep the group bits only if no predicate position is pushed onto a lane by them
          FPhase A0, A1;
          std::vector<int> R0 = R;
          fill_regs(R0, b);
          make_phase_thr(A0, R0, b, use);
          make_phase_thr(A1, Rf, b, use, fixed);
          int u0 = 0, u1 = 0;
          for (int j = 0; j < 5; ++j) {
            u0 += use[A0.thr[j]] ? 1 : 0;
            u1 += use[A1.thr[j]] ? 1 : 0;
          }
          ok = u1 <= u0;
        }
        if (ok) {
          R = Rf;
          W = fixed;
        } else {
          fill_regs(R, b);
          W.clear();
        }
      } else {
        fill_regs(R, b);
      }
      FPhase F;
      std::memset(&F, 0, sizeof(F));
      make_phase_thr(F, R, b, use, W);
      F.op_begin = int(prog.ops.size());
      F.flip = uint8_t(emit_ops(prog, P, ph.second, tile_pos_of, R));
      F.op_end = int(prog.ops.size());
      prog.phases.push_back(F);
    }
    A.n_phases = int(prog.phases.size()) - A.phase_begin;
    A.op_begin = A.n_phases ? prog.phases[A.phase_begin].op_begin : int(prog.ops.size());
    A.op_end = int(prog.ops.size());
    A.n_gen = int(prog.gen_slot_of.size()) - A.gen_base;
    bool full = false;
    for (int oi = A.op_begin; oi < A.op_end; ++oi) {
      FOp& o = prog.ops[oi];
      if (o.cs >= CS_GEN1) o.slot -= A.gen_base;   // pass-local accumulator slot
      full |= (o.cs < CS_GEN1 && (o.kind == FK_DIAGG || o.kind == FK_DENSE2 ||
                                  (o.kind == FK_PAIRG && o.mtype == MT_GENERAL))) ||
              (o.cs >= CS_GEN2 && o.cs < CS_GEND);
    }
    absorb_pass_scale(prog, A);
    // ---- in-tile relabeling: bring the qubits the next gates target onto physical bits 0..2 ----
    int sigma[64];
    for (int p = 0; p < 64; ++p) sigma[p] = p;
    if (remap && !rest.empty() && b > LBT) {
      int next_use[64];
      for (int p = 0; p < 64; ++p) next_use[p] = 1 << 30;
      for (size_t k = 0; k < rest.size(); ++k) {
        u64 d = req[rest[k]].dense;
        for (int p = 0; p < 64 && d; ++p)
          if ((d >> p) & 1) {
            if (next_use[p] > int(k)) next_use[p] = int(k);
            d &= ~(1ull << p);
          }
      }
      std::vector<int> cand;   // tile positions sorted by next use (earliest first), low bits win ties
      for (int t = 0; t < b; ++t)
        if (!(pin_top && A.tpos[t] == nl - 1)) cand.push_back(A.tpos[t]);
      std::stable_sort(cand.begin(), cand.end(), [&](int x, int y) {
        if (next_use[x] != next_use[y]) return next_use[x] < next_use[y];
        return x < y;
      });
      static const bool sort_all = !(getenv("SVB200_REMAP_SORT") && std::string(getenv("SVB200_REMAP_SORT")) == "0");
      // The positions sent to physical bits 0..2 become the last phase's lanes (direct store).  A
      // quarter-warp's 16-byte loads are conflict-free only when its three lane positions cover all
      // residues mod 3 (the swizzle folds tile position p into chunk bit p mod 3), so among the
      // soonest-needed candidates take three with distinct residues that the last phase neither
      // holds in registers nor tests as predicates.
      static const bool lane_res = !(getenv("SVB200_LANE_RESIDUE") && std::string(getenv("SVB200_LANE_RESIDUE")) == "0");
      if (lane_res && sort_all && A.n_phases > 0 && cand.size() >= 3 && LB == 3) {
        const FPhase& Lp = prog.phases[A.phase_begin + A.n_phases - 1];
        u64 predp = 0;   // physical positions the last phase tests per thread
        for (int oi = Lp.op_begin; oi < Lp.op_end; ++oi) {
          const FOp& o = prog.ops[oi];
          predp |= o.pm | o.fpm | o.xm;
          for (int j = 0; j < o.nt; ++j)
            if (o.treg[j] == 0xFF) predp |= 1ull << o.tphys[j];
        }
        std::vector<int> pick;
        int used = 0;
        for (int x : cand) {
          const int t = tile_pos_of[x];
          bool reg = false;
          for (int k = 0; k < kRB; ++k) reg |= Lp.reg[k] == t;
          if (reg || ((predp >> x) & 1) || ((used >> (t % 3)) & 1)) continue;
          used |= 1 << (t % 3);
          pick.push_back(x);
          if (pick.size() == 3) break;
        }
        if (pick.size() == 3) {
          std::vector<int> reordered(pick.begin(), pick.end());
          for (int x : cand)
            if (std::find(pick.begin(), pick.end(), x) == pick.end()) reordered.push_back(x);
          cand.swap(reordered);
        }
      }
      if (sort_all) {
        // every tile position, not only 0..LBT-1: the qubits needed soonest take the lowest
        // physical positions of the tile, the ones needed last the highest.  Low positions are
        // where tiles stream well; a tile holding several of the very top bits of a large state
        // (16-64 GiB strides) streams up to 6x slower (33-qubit QAOA: 296 vs 46-89 ms per pass).
        std::vector<int> slots(cand.begin(), cand.end());
        std::sort(slots.begin(), slots.end());
        for (size_t i = 0; i < cand.size(); ++i) sigma[cand[i]] = slots[i];
      } else {
        std::vector<int> want(cand.begin(), cand.begin() + LBT);   // physical positions to move onto 0..LBT-1
        std::vector<int> out_low, in_high;
        for (int l = 0; l < LBT; ++l)
          if (std::find(want.begin(), want.end(), l) == want.end()) out_low.push_back(l);
        for (int x : want)
          if (x >= LBT) in_high.push_back(x);
        for (size_t s = 0; s < in_high.size(); ++s) {   // swap(out_low[s], in_high[s])
          sigma[in_high[s]] = out_low[s];
          sigma[out_low[s]] = in_high[s];
        }
      }
    }
    std::vector<int> q_low, q_rest;
    for (int t = 0; t < b; ++t) {
      A.tpos_st[t] = (unsigned char)sigma[A.tpos[t]];
      if (A.tpos_st[t] < LB) q_low.push_back(t);
      else q_rest.push_back(t);
    }
    std::sort(q_low.begin(), q_low.end(), [&](int x, int y) { return A.tpos_st[x] < A.tpos_st[y]; });
    int qi = 0;
    for (int t : q_low) A.q[qi++] = (unsigned char)t;
    for (int t : q_rest) A.q[qi++] = (unsigned char)t;
    // Direct store: the tile positions that land on physical bits 0..2 become the last phase's
    // lane bits (those that are not its register bits; none may carry one of its predicates, which
    // would split warps).  An 8-lane group then holds one 128-byte run (or a run split over two
    // registers), so the generated kernel stores the last phase's registers
    // straight to HBM (no shared-memory round trip) and refills the tile buffer with the next
    // tile while the last phase computes (fused_jit.cpp).
    A.direct = 0;
    if (A.n_phases > 0 && int(q_low.size()) == LB) {
      FPhase& L = prog.phases[A.phase_begin + A.n_phases - 1];
      bool ok = true;
      u64 lowld = 0;
      std::vector<int> lanes;   // q_low positions that are thread bits of the last phase
      for (int t : q_low) {
        lowld |= 1ull << A.tpos[t];
        bool reg = false;
        for (int k = 0; k < kRB; ++k) reg |= L.reg[k] == t;
        if (!reg) lanes.push_back(t);
      }
      for (int oi = L.op_begin; oi < L.op_end && ok; ++oi) {
        const FOp& o = prog.ops[oi];
        if ((o.pm | o.fpm | o.xm) & lowld) ok = false;
        for (int j = 0; j < o.nt; ++j)
          if (o.treg[j] == 0xFF && ((lowld >> o.tphys[j]) & 1)) ok = false;
      }
      static const bool store_phase = !(getenv("SVB200_STORE_PHASE") && std::string(getenv("SVB200_STORE_PHASE")) == "0");
      if (ok && lanes.size() >= 2) {
        // a low store bit held in a register splits the thread's 128-byte run over two stores of
        // full 32-byte sectors (still merged in L2); lanes carry the others
        std::vector<int> thr(lanes.begin(), lanes.end());
        for (int j = 0; j < b - kRB; ++j)
          if (std::find(lanes.begin(), lanes.end(), int(L.thr[j])) == lanes.end()) thr.push_back(L.thr[j]);
        for (int j = 0; j < b - kRB; ++j) L.thr[j] = uint8_t(thr[j]);
        A.direct = 1;
      } else if (store_phase && b == kMaxB) {
        // The last phase holds two or more of the store's low bits in registers (or tests them
        // as predicates): its stores would write 16-32 bytes per 128-byte line per instruction,
        // which streams several times slower (a 33-qubit QAOA pass: 296 ms vs ~50).  Append an
        // op-free phase whose lanes ARE those bits: one more shared-memory round trip, and the pass
        // keeps its coalesced direct store and its overlapped next-tile load.
        FPhase E;
        std::memset(&E, 0, sizeof(E));
        std::vector<int> R;
        for (int k = 0; k < kRB; ++k)
          if (std::find(q_low.begin(), q_low.end(), int(L.reg[k])) == q_low.end()) R.push_back(L.reg[k]);
        fill_regs(R, b, q_low);
        bool clash = false;
        for (int t : q_low) clash |= std::find(R.begin(), R.end(), t) != R.end();
        if (!clash) {
          int use0[kMaxB] = {0};
          make_phase_thr(E, R, b, use0);
          std::vector<int> thr(q_low.begin(), q_low.end());
          for (int j = 0; j < b - kRB; ++j)
            if (std::find(q_low.begin(), q_low.end(), int(E.thr[j])) == q_low.end()) thr.push_back(E.thr[j]);
          for (int j = 0; j < b - kRB; ++j) E.thr[j] = uint8_t(thr[j]);
          E.op_begin = E.op_end = int(prog.ops.size());
          E.flip = 0;
          prog.phases.push_back(E);
          A.n_phases += 1;
          A.direct = 1;
        }
      }
    }
    bool moved = false;
    for (int p = 0; p < nl; ++p) moved |= sigma[p] != p;
    if (moved) {
      for (int i : rest) {
        relabel(P[i], sigma);
        req[i] = requirements(P[i]);
      }
      for (int p = 0; p < nl; ++p) perm_total[p] = sigma[perm_total[p]];
    }
    prog.steps.push_back({true, int(prog.passes.size())});
    prog.full.push_back(full ? 1 : 0);
    prog.passes.push_back(A);
    remaining.swap(rest);
  }
  prog.perm = perm_total;
  for (auto& A : prog.passes) A.n_gen_total = int(prog.gen_slot_of.size());
  prog.gen_scale.resize(prog.gen_slot_of.size(), 1.0);
  absorb_rotation_signs(prog, jit_enabled());
  return prog;
}

// Tail-deferral threshold chosen per circuit structure (see build_program; guarded by g_tan_mu).
static std::map<u64, int> g_defer_choice;

// Plan a program.  Pass construction is greedy and sensitive to where passes end, so the first plan
// of a circuit structure is built with several tail-deferral thresholds and the cheapest is kept,
// by a cost model fitted to the bench circuit's measured pass times: a pass costs ~1.8 phases (its
// HBM stream + tile load/store), a phase one shared-memory round trip plus its arithmetic.  The
// choice is remembered per structure (like the rotation forms), so re-plans with new parameter
// values plan once.  SVB200_DEFER_TAIL=k pins the threshold.
Program build_program(int nl, const std::vector<Prim>& prims_in, bool remap, bool pin_top) {
  const u64 skey = structure_key(nl, prims_in, remap, pin_top);
  std::vector<uint8_t> hint;
  int chosen = -1;
  {
    std::lock_guard<std::mutex> lk(g_tan_mu);
    auto it = g_tan_forms.find(skey);
    if (it != g_tan_forms.end()) hint = it->second;
    auto jt = g_defer_choice.find(skey);
    if (jt != g_defer_choice.end()) chosen = jt->second;
  }
  static const int forced = getenv("SVB200_DEFER_TAIL") ? std::max(0, atoi(getenv("SVB200_DEFER_TAIL"))) : -1;
  if (forced >= 0) chosen = forced;
  Program prog;
  if (chosen >= 0) {
    prog = build_program_k(nl, prims_in, remap, pin_top, chosen, hint);
  } else {
    double best = 1e300;
    for (int k : {3, 2, 1, 0}) {
      Program cand = build_program_k(nl, prims_in, remap, pin_top, k, hint);
      const double cost = 1.8 * double(cand.passes.size()) + double(cand.phases.size()) + double(cand.singles.size());
      if (cost < best) {
        best = cost;
        chosen = k;
        prog = std::move(cand);
      }
    }
  }
  std::lock_guard<std::mutex> lk(g_tan_mu);
  if (g_tan_forms.size() > 4096) g_tan_forms.clear();
  if (g_defer_choice.size() > 4096) g_defer_choice.clear();
  if (!prog.tan_forms.empty()) g_tan_forms[skey] = prog.tan_forms;
  g_defer_choice[skey] = chosen;
  return prog;
}


void serialize_program(const Program& prog, int nl, std::vector<int64_t>& I, std::vector<double>& Dv) {
  I.clear();
  Dv.clear();
  auto put_c = [&](const double2& c) {
    Dv.push_back(c.x);
    Dv.push_back(c.y);
  };
  I.push_back(1);   // format version
  I.push_back(nl);
  I.push_back(int64_t(prog.steps.size()));
  for (const Step& s : prog.steps) {
    I.push_back(s.fused ? 1 : 0);
    if (s.fused) {
      const FPassArgs& A = prog.passes[s.index];
      I.push_back(A.b);
      for (int t = 0; t < A.b; ++t) I.push_back(A.tpos[t]);
      for (int t = 0; t < A.b; ++t) I.push_back(A.tpos_st[t]);
      for (int t = 0; t < A.b; ++t) I.push_back(A.q[t]);
      I.push_back(A.phase_begin);
      I.push_back(A.n_phases);
    } else {
      const Prim& p = prog.singles[s.index];
      I.push_back(p.type);
      I.push_back(int64_t(p.fmask));
      I.push_back(int64_t(p.fval));
      I.push_back(int64_t(p.xmask));
      I.push_back(p.nb);
      for (int t = 0; t < p.nb; ++t) I.push_back(p.pos[t]);
      I.push_back(int64_t(Dv.size()) / 2);
      I.push_back(int64_t(p.m.size()));
      for (auto& c : p.m) {
        Dv.push_back(c.real());
        Dv.push_back(c.imag());
      }
    }
  }
  I.push_back(int64_t(prog.phases.size()));
  for (const FPhase& F : prog.phases) {
    for (int k = 0; k < kRB; ++k) I.push_back(F.reg[k]);
    I.push_back(F.flip);
    for (int t = 0; t < kMaxB; ++t) I.push_back(F.thr[t]);
    I.push_back(F.op_begin);
    I.push_back(F.op_end);
  }
  I.push_back(int64_t(prog.ops.size()));
  for (const FOp& o : prog.ops) {
    I.push_back(int64_t(o.pm));
    I.push_back(int64_t(o.pv));
    I.push_back(int64_t(o.xm));
    I.push_back(int64_t(o.fpm));
    I.push_back(int64_t(o.fpv));
    I.push_back(o.fk);
    I.push_back(o.cs);
    I.push_back(o.cm);
    I.push_back(o.cv);
    I.push_back(o.k);
    I.push_back(o.v);
    I.push_back(o.xr);
    I.push_back(o.nt);
    I.push_back(o.mtype);
    for (int t = 0; t < 6; ++t) I.push_back(o.treg[t]);
    for (int t = 0; t < 6; ++t) I.push_back(o.tphys[t]);
    I.push_back(o.tab);
    I.push_back(int64_t(Dv.size()) / 2);   // inline coefficients
    for (int t = 0; t < 4; ++t) put_c(o.c[t]);
  }
  I.push_back(int64_t(Dv.size()) / 2);     // coefficient table offset
  I.push_back(int64_t(prog.coef.size()));
  for (auto& c : prog.coef) put_c(c);
  for (int p = 0; p < nl; ++p) I.push_back(prog.perm[p]);
}

}  // namespace fused

void plan_program_serialized(int n_qubits, const std::vector<Prim>& prims, std::vector<int64_t>& ints,
                             std::vector<double>& dbls) {
  static const bool remap = !(getenv("SVB200_REMAP") && std::string(getenv("SVB200_REMAP")) == "0");
  const fused::Program prog = fused::build_program(n_qubits, prims, remap);
  fused::serialize_program(prog, n_qubits, ints, dbls);
}

// Host-only: plan, then compile every pass with the runtime pass compiler (no GPU needed: NVRTC
// emits sm_100a cubins; they are loaded on first launch).  out4 = {passes, passes with a generated
// kernel, kernels compiled so far in this process, their total compile time in microseconds}.
void plan_compile(int nl, const std::vector<Prim>& prims, bool two, int64_t* out4) {
  using namespace fused;
  Program prog = build_program(nl, prims, true, two);
  jit_prepare(prog, two);
  int64_t with = 0;
  for (const JitPass& jp : prog.jit) with += jp.kernel ? 1 : 0;
  int64_t compiled = 0, us = 0, cached = 0;
  jit_stats(&compiled, &us, &cached);
  out4[0] = int64_t(prog.passes.size());
  out4[1] = with;
  out4[2] = compiled;
  out4[3] = us;
}

// FP64 floating-point operations the fused program performs per amplitude of the state (DFMA = 2,
// DMUL / DADD = 1), counted from the op cases as the device code executes them on a thread's 16
// amplitudes (register-pattern subsets scale the pair / group counts); for the roofline report.
double program_fp64_flops_per_amp(const fused::Program& prog) {
  using namespace fused;
  double f = 0.0;   // per thread (16 amplitudes)
  auto subset = [](int cm, int fixed) {   // fraction of register patterns an op's (cm, cv) selects
    return 1.0 / double(1 << __builtin_popcount(cm & ~fixed & 15));
  };
  for (const FOp& o : prog.ops) {
    const int cs = o.cs;
    if (cs >= CS_SHEAR && cs < CS_SHEAR + 16) f += 8 * 6 * 2;
    else if (cs >= CS_TAN && cs < CS_TAND + 8) f += 8 * 4 * 2;
    else if (cs == CS_RDIAG) f += 6.0 * __builtin_popcountll(o.xm);
    else if ((cs >= CS_PAIR1 && cs < CS_PAIR1 + 16) || (cs >= CS_PAIR1D && cs < CS_PAIR1D + 16))
      f += o.mtype == MT_GENERAL ? 8 * 28 : (o.mtype == MT_X ? 0 : 8 * 12);
    else if ((cs >= CS_PHASE1 && cs < CS_PHASE1 + 8) || (cs >= CS_PHASE1D && cs < CS_PHASE1D + 8)) f += 8 * 6;
    else if (cs == CS_SCALAR) f += 16 * 6;
    else if (cs >= CS_PARITY && cs < CS_PARITY + 16) f += 8 * 6;
    else if (cs >= CS_PAIRGR && cs < CS_PAIRGR + 15) f += o.mtype == MT_X ? 0.0 : 16 * 12 / 2.0 * subset(o.cm, o.xr);
    else if (cs >= CS_PAIRG && cs < CS_PAIRG + 15) f += 16 * 28 / 2.0 * subset(o.cm, o.xr);
    else if (cs == CS_DIAGG) f += 16 * 6 * subset(o.cm, 0);
    else if (cs >= CS_DENSE2 && cs < CS_DENSE2 + 6) f += 4 * 16 * 8 * subset(o.cm, 0);
    else if (cs >= CS_GEN1 && cs < CS_GEN2) f += 4 * 2 * 24 + 20;
    else if (cs >= CS_GEN2 && cs < CS_GEND) f += 2 * 4 * (16 * 8 + 8) + 20;
    else if (cs >= CS_GEND && cs < CS_GEND + 4) f += 8 * 8 + 20;
  }
  return f / 16.0;
}

PlanStats plan_stats(int nl, const std::vector<Prim>& prims) {
  using namespace fused;
  PlanStats s;
  s.ops = int64_t(prims.size());
  if (nl < 5) {
    s.passes = s.ops;
    return s;
  }
  Program prog = build_program(nl, prims, true);
  s.passes = int64_t(prog.steps.size());
  s.tile_bits = std::min(tile_bits(), nl);
  s.phases = int64_t(prog.phases.size());
  s.fp64_flops_per_amp = program_fp64_flops_per_amp(prog);
  return s;
}
