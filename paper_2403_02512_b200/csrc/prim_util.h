// Scheduling helpers shared by the fusion planner (fused_plan.cpp) and the sharded driver
// (api.cpp run_ops): per-bit commutation classes of a primitive and bit relabeling.
//
// Commutation is decided per bit: a primitive acts on each bit of its support either Z-like
// (diagonal: controls, diagonal-table bits), X-like (a single-target 2x2 of the form aI + bX,
// e.g. RX or the X of a CNOT) or generally.  Two primitives commute when every shared bit is
// Z-like in both or X-like in both -- so RZ slides past CNOT controls and RX past CNOT targets.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "sv_internal.h"

struct PrimReq {
  u64 dense = 0;     // bits the primitive's non-diagonal action needs local / in registers
  u64 support = 0;   // every bit it reads
  u64 zb = 0, xb = 0;
  bool diag = false;
};

inline bool prim_is_xlike(const std::vector<cplx>& m) { return m.size() == 4 && m[0] == m[3] && m[1] == m[2]; }

// SVB200_GEN_SEL_GENERAL=1: the round-1 rule (the psi/lambda bit as a general action), for A/B
inline bool gen_sel_general() {
  static const bool on = getenv("SVB200_GEN_SEL_GENERAL") && std::string(getenv("SVB200_GEN_SEL_GENERAL")) == "1";
  return on;
}

inline PrimReq prim_requirements(const Prim& p) {
  PrimReq r;
  if (p.type == PRIM_PAIR) {
    r.dense = p.xmask;
    r.support = p.fmask | p.xmask;
    r.zb = p.fmask & ~p.xmask;
    if (popcount64(p.xmask) == 1 && prim_is_xlike(p.m)) r.xb = p.xmask;
  } else if (p.type == PRIM_DIAG) {
    r.diag = true;
    r.support = p.fmask;
    for (int j = 0; j < p.nb; ++j) r.support |= 1ull << p.pos[j];
    r.zb = r.support;
  } else if (p.type == PRIM_GEND) {
    // diagonal generator: Z-like everywhere; the psi/lambda bit must be a register bit (dense)
    r.support = p.fmask | p.xmask;
    for (int j = 0; j < p.nb; ++j) r.support |= 1ull << p.pos[j];
    r.dense = p.xmask;
    r.zb = r.support & ~(gen_sel_general() ? p.xmask : 0ull);
  } else if (p.type == PRIM_GEN) {
    // reads psi and lambda on its targets (general) across the psi/lambda bit; controls Z-like
    for (int j = 0; j < p.nb; ++j) r.dense |= 1ull << p.pos[j];
    r.dense |= p.xmask;
    r.support = p.fmask | r.dense;
    r.zb = p.fmask & ~r.dense;
    // A bra-ket only reads the state and no gate acts on the psi/lambda bit, so for commutation
    // that bit is Z-like: bra-kets commute with each other and with gates on other qubits (a
    // unitary V on both arrays that commutes with G leaves <lambda|G|psi> unchanged).  Treating
    // it as a general action chained every bra-ket to the previous one: one deferred bra-ket
    // blocked all later ones and ended the pass (reverse sweeps took ~3x the forward's passes).
    if (!gen_sel_general()) r.zb |= p.xmask;
  } else {
    for (int j = 0; j < p.nb; ++j) r.dense |= 1ull << p.pos[j];
    r.support = p.fmask | r.dense;
    r.zb = p.fmask & ~r.dense;
  }
  return r;
}

inline bool prims_commute(const PrimReq& a, const PrimReq& b) {
  const u64 shared = a.support & b.support;
  return (shared & ~((a.zb & b.zb) | (a.xb & b.xb))) == 0;
}

// union of the per-bit action classes of primitives deferred past a point of the schedule
struct DeferredSet {
  u64 z = 0, x = 0, g = 0;
  void add(const PrimReq& r) {
    z |= r.zb;
    x |= r.xb;
    g |= r.support & ~(r.zb | r.xb);
  }
  // would r fail to commute with some deferred primitive?
  bool blocks(const PrimReq& r) const {
    const u64 rg = r.support & ~(r.zb | r.xb);
    return (r.support & g) || (r.zb & x) || (r.xb & z) || (rg & (z | x));
  }
};

inline u64 permute_mask(u64 m, const int* perm) {
  u64 o = 0;
  for (int b = 0; b < 64 && m; ++b)
    if ((m >> b) & 1) {
      o |= 1ull << perm[b];
      m &= ~(1ull << b);
    }
  return o;
}

// relabel the bits of a prim (bit b -> perm[b]); positions stay ascending, tables follow
inline void relabel_prim(Prim& p, const int* perm) {
  p.fmask = permute_mask(p.fmask, perm);
  p.fval = permute_mask(p.fval, perm);
  p.xmask = permute_mask(p.xmask, perm);
  if (p.nb == 0) return;
  const int k = p.nb;
  int np[16], order[16];
  for (int j = 0; j < k; ++j) {
    np[j] = perm[p.pos[j]];
    order[j] = j;
  }
  std::sort(order, order + k, [&](int x, int y) { return np[x] < np[y]; });
  int rank[16];   // old index bit j -> new index bit rank[j]
  for (int i = 0; i < k; ++i) {
    rank[order[i]] = i;
    p.pos[i] = np[order[i]];
  }
  const size_t d = size_t(1) << k;
  auto map_idx = [&](size_t r) {
    size_t o = 0;
    for (int j = 0; j < k; ++j)
      if ((r >> j) & 1) o |= size_t(1) << rank[j];
    return o;
  };
  std::vector<cplx> m(p.m.size());
  if (p.type == PRIM_DIAG || p.type == PRIM_GEND) {
    for (size_t r = 0; r < d; ++r) m[map_idx(r)] = p.m[r];
  } else {
    for (size_t r = 0; r < d; ++r)
      for (size_t c = 0; c < d; ++c) m[map_idx(r) * d + map_idx(c)] = p.m[r * d + c];
  }
  p.m = m;
}
