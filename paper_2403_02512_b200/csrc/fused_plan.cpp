// Host planner of the K7 fusion engine: pass construction, register-phase scheduling and
// device-op emission (see fused.h for the program format and fused.cu for the kernel).
#include <algorithm>
#include <cstring>

#include "fused.h"

namespace fused {

struct Req {
  u64 dense = 0;     // bits that must be register bits
  u64 support = 0;   // every bit the prim reads
  bool diag = false;
  bool fusable = true;
};

Req requirements(const Prim& p) {
  Req r;
  if (p.type == PRIM_PAIR) {
    r.dense = p.xmask;
    r.support = p.fmask | p.xmask;
    r.fusable = popcount64(p.xmask) <= kRB;
  } else if (p.type == PRIM_DIAG) {
    r.diag = true;
    r.support = p.fmask;
    for (int j = 0; j < p.nb; ++j) r.support |= 1ull << p.pos[j];
    r.fusable = p.nb <= 6;
  } else {
    for (int j = 0; j < p.nb; ++j) r.dense |= 1ull << p.pos[j];
    r.support = p.fmask | r.dense;
    r.fusable = p.nb <= 2;
  }
  return r;
}

std::vector<PassPlan> plan_passes(int nl, const std::vector<Prim>& prims, int b) {
  std::vector<Req> req(prims.size());
  for (size_t i = 0; i < prims.size(); ++i) req[i] = requirements(prims[i]);
  std::vector<int> remaining(prims.size());
  for (size_t i = 0; i < prims.size(); ++i) remaining[i] = int(i);
  std::vector<PassPlan> out;
  const u64 low = (1ull << std::min(3, nl)) - 1;
  const size_t window = 4096;
  while (!remaining.empty()) {
    const int p0 = remaining[0];
    if (!req[p0].fusable || nl < 5) {
      PassPlan s;
      s.single = p0;
      out.push_back(s);
      remaining.erase(remaining.begin());
      continue;
    }
    PassPlan pp;
    pp.fused = true;
    u64 B = low;
    u64 def_nd = 0, def_d = 0;
    std::vector<int> rest;
    for (size_t k = 0; k < remaining.size(); ++k) {
      const int i = remaining[k];
      const Req& r = req[i];
      bool ok = k < window && r.fusable && int(pp.prims.size()) < kMaxSmemOps;   // op records fit in smem
      if (ok) {
        const u64 blocked = r.diag ? (r.support & def_nd) : (r.support & (def_nd | def_d));
        ok = blocked == 0 && popcount64(B | r.dense) <= b;
      }
      if (ok) {
        B |= r.dense;
        pp.prims.push_back(i);
      } else {
        if (r.diag)
          def_d |= r.support;
        else
          def_nd |= r.support;
        rest.push_back(i);
      }
    }
    // fill the tile up to b bits with the lowest unused positions (longer contiguous runs)
    for (int p = 0; p < nl && popcount64(B) < b; ++p) B |= 1ull << p;
    pp.tile_bits = B;
    out.push_back(pp);
    remaining.swap(rest);
  }
  return out;
}

int mtype_of(const std::vector<cplx>& m) {
  auto re = [](cplx c) { return c.imag() == 0.0; };
  auto im = [](cplx c) { return c.real() == 0.0; };
  if (m[0] == 0.0 && m[3] == 0.0 && m[1] == 1.0 && m[2] == 1.0) return MT_X;
  if (re(m[0]) && re(m[1]) && re(m[2]) && re(m[3])) return MT_REAL;
  if (re(m[0]) && re(m[3]) && im(m[1]) && im(m[2])) return MT_RXLIKE;
  return MT_GENERAL;
}

// choose extra register positions so each bank class {p mod 3} keeps a free thread position
void fill_regs(std::vector<int>& reg, int b) {
  auto cls_free = [&](int c, const std::vector<int>& R) {
    for (int p = c; p < b; p += 3)
      if (std::find(R.begin(), R.end(), p) == R.end()) return true;
    return false;
  };
  for (int p = b - 1; p >= 0 && int(reg.size()) < kRB; --p) {
    if (std::find(reg.begin(), reg.end(), p) != reg.end()) continue;
    std::vector<int> trial = reg;
    trial.push_back(p);
    if (cls_free(0, trial) && cls_free(1, trial) && cls_free(2, trial)) reg = trial;
  }
  for (int p = b - 1; p >= 0 && int(reg.size()) < kRB; --p)
    if (std::find(reg.begin(), reg.end(), p) == reg.end()) reg.push_back(p);
}

void make_phase_thr(FPhase& F, const std::vector<int>& reg, int b) {
  for (int k = 0; k < kRB; ++k) F.reg[k] = (uint8_t)reg[k];
  std::vector<int> thr;
  for (int c = 0; c < 3; ++c)
    for (int p = c; p < b; p += 3)
      if (std::find(reg.begin(), reg.end(), p) == reg.end()) {
        thr.push_back(p);
        break;
      }
  for (int p = 0; p < b; ++p)
    if (std::find(reg.begin(), reg.end(), p) == reg.end() && std::find(thr.begin(), thr.end(), p) == thr.end())
      thr.push_back(p);
  for (int j = 0; j < b - kRB; ++j) F.thr[j] = (uint8_t)thr[j];
}

// Emit the device ops of one phase.  Unconditional X on a register bit is not executed: it is
// absorbed into a flip mask F (logical register index j lives in register j ^ F); later ops of
// the phase are rewritten for F and the phase's store offsets apply it.  Returns F.
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
        prog.ops.push_back(op);
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
        op.mtype = uint8_t((mt == MT_X || mt == MT_REAL) ? MT_REAL : MT_GENERAL);
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
    switch (op.kind) {
      case FK_PAIR1: op.cs = (dyn ? CS_PAIR1D : CS_PAIR1) + op.k * 4 + op.mtype; break;
      case FK_PHASE1: op.cs = (dyn ? CS_PHASE1D : CS_PHASE1) + op.k * 2 + op.v; break;
      case FK_SCALAR: op.cs = CS_SCALAR; break;
      case FK_PAIRG: op.cs = (op.mtype == MT_REAL ? CS_PAIRGR : CS_PAIRG) + op.xr - 1; break;
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
    prog.ops.push_back(op);
  }
  return F;
}

// List-schedule a pass's prims into register phases.  Prims may be reordered only past prims
// they commute with (disjoint support, or both diagonal); each phase picks up to 4 register
// bits and runs every ready prim whose dense bits fit, to a fixpoint.
// Returns (register-bit mask in physical positions, prims in execution order) per phase.
std::vector<std::pair<u64, std::vector<int>>> schedule_phases(const std::vector<Prim>& prims,
                                                              const std::vector<int>& list) {
  const int L = int(list.size());
  std::vector<Req> rq(L);
  for (int i = 0; i < L; ++i) rq[i] = requirements(prims[list[i]]);
  // remaining-predecessor counts and successor lists of the conflict DAG
  std::vector<int> npred(L, 0);
  std::vector<std::vector<int>> succ(L);
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < i; ++j) {
      const bool commute = (rq[i].diag && rq[j].diag) || (rq[i].support & rq[j].support) == 0;
      if (!commute) {
        succ[j].push_back(i);
        npred[i]++;
      }
    }
  std::vector<char> done(L, 0);
  int ndone = 0;
  std::vector<std::pair<u64, std::vector<int>>> phases;
  while (ndone < L) {
    u64 R = 0;
    std::vector<int> order;
    for (;;) {
      bool progress = false;
      for (int i = 0; i < L; ++i) {
        if (done[i] || npred[i] != 0) continue;
        if ((rq[i].dense & ~R) != 0) continue;
        done[i] = 1;
        ++ndone;
        order.push_back(list[i]);
        for (int s : succ[i]) npred[s]--;
        progress = true;
      }
      if (progress) continue;
      int pick = -1;
      for (int i = 0; i < L; ++i)
        if (!done[i] && npred[i] == 0 && popcount64(R | rq[i].dense) <= kRB) {
          pick = i;
          break;
        }
      if (pick < 0) break;
      R |= rq[pick].dense;
    }
    phases.push_back({R, order});
  }
  return phases;
}

Program build_program(int nl, const std::vector<Prim>& prims, std::vector<PassPlan>& plan) {
  Program prog;
  const int b = std::min(kMaxB, nl);
  plan = plan_passes(nl, prims, b);
  for (auto& pp : plan) {
    if (!pp.fused) continue;
    FPassArgs A;
    std::memset(&A, 0, sizeof(A));
    A.b = b;
    A.nthr = b - kRB;
    int tile_pos_of[64];
    for (int i = 0; i < 64; ++i) tile_pos_of[i] = -1;
    int j = 0;
    for (int p = 0; p < nl; ++p)
      if ((pp.tile_bits >> p) & 1) {
        A.tpos[j] = (unsigned char)p;
        tile_pos_of[p] = j++;
      }
    A.n_tiles = 1ull << (nl - b);
    A.phase_begin = int(prog.phases.size());
    for (auto& ph : schedule_phases(prims, pp.prims)) {
      std::vector<int> R;
      for (int p = 0; p < 64; ++p)
        if ((ph.first >> p) & 1) R.push_back(tile_pos_of[p]);
      fill_regs(R, b);
      FPhase F;
      std::memset(&F, 0, sizeof(F));
      make_phase_thr(F, R, b);
      F.op_begin = int(prog.ops.size());
      F.flip = uint8_t(emit_ops(prog, prims, ph.second, tile_pos_of, R));
      F.op_end = int(prog.ops.size());
      prog.phases.push_back(F);
    }
    A.n_phases = int(prog.phases.size()) - A.phase_begin;
    A.op_begin = A.n_phases ? prog.phases[A.phase_begin].op_begin : int(prog.ops.size());
    A.op_end = int(prog.ops.size());
    bool full = false;
    for (int ph = A.phase_begin; ph < A.phase_begin + A.n_phases; ++ph)
      for (int oi = prog.phases[ph].op_begin; oi < prog.phases[ph].op_end; ++oi) {
        const FOp& o = prog.ops[oi];
        full |= o.kind == FK_DIAGG || o.kind == FK_DENSE2 || (o.kind == FK_PAIRG && o.mtype == MT_GENERAL);
      }
    prog.full.push_back(full ? 1 : 0);
    prog.passes.push_back(A);
  }
  return prog;
}

}  // namespace fused

PlanStats plan_stats(int nl, const std::vector<Prim>& prims) {
  using namespace fused;
  PlanStats s;
  s.ops = int64_t(prims.size());
  if (nl < 5) {
    s.passes = s.ops;
    return s;
  }
  std::vector<PassPlan> plan;
  Program prog = build_program(nl, prims, plan);
  s.passes = int64_t(plan.size());
  s.tile_bits = std::min(kMaxB, nl);
  s.phases = int64_t(prog.phases.size());
  return s;
}
