// K7: gate-fusion tile engine.
//
// One "pass" streams the whole shard through shared memory once: each CTA stages a tile of
// 2^b amplitudes (b <= 12, 64 KiB) whose index bits are the pass's tile bits B (always the
// three lowest physical bits -> 128-byte contiguous runs, plus any high bits the pass's gates
// need), applies a whole list of gates to the tile, and writes it back: a run of G gates costs
// one HBM read + write of the state instead of G (north_star: "a gate-fusion kernel stages
// 2^k-amplitude blocks in shared memory so runs of low-qubit gates take one HBM pass").
//
// Inside a tile, work proceeds in "phases": every thread holds 16 amplitudes in registers,
// indexed by 4 register bits R (tile positions); dense targets of the phase's gates must be in
// R, while controls and diagonal gates may sit on ANY bit (register, thread or tile-outer bit:
// they are predicates / per-thread constants).  Switching R costs one shared-memory round trip.
// Shared memory is XOR-swizzled so every phase's 16-byte accesses are bank-conflict free.
//
// The host planner (bottom of this file) greedily builds passes over the dependency order of
// the primitive list (prims only move past prims they commute with: disjoint support, or both
// diagonal) and splits each pass into phases.
#include <algorithm>
#include <cstring>

#include "sv_internal.h"

namespace {

constexpr int kMaxB = 12;        // tile bits (2^12 amps = 64 KiB)
constexpr int kRB = 4;           // register bits per thread (16 amplitudes)
constexpr int kRegs = 1 << kRB;

// op kinds; the *1 kinds are fast paths whose register predicate is compile-time
enum FKind : uint8_t {
  FK_PAIR1 = 0,   // 2x2 on register bit k, no register-side control
  FK_PAIRG = 1,   // 2x2 on register xmask xr with register pattern (cm, cv)
  FK_PHASE1 = 2,  // a *= d where register bit k == v (no other register-side pattern)
  FK_SCALAR = 3,  // a *= d on all 16 amplitudes (pattern only on thread / outer bits)
  FK_DIAGG = 4,   // table lookup diagonal, general
  FK_DENSE2 = 5,  // 4x4 on register bits (k0 < k1) = xr & 15, xr >> 4
};
enum MType : uint8_t { MT_GENERAL = 0, MT_REAL = 1, MT_RXLIKE = 2, MT_X = 3 };

struct __align__(16) FOp {
  u64 pm, pv;            // fixed pattern on non-register bits (tested on the thread's physical base)
  uint8_t kind, mtype;
  uint8_t xr;            // PAIRG: register-space xmask; DENSE2: k0 | (k1 << 4)
  uint8_t cm, cv;        // register-space pattern (PAIRG includes i0's pattern on xr)
  uint8_t nt;            // DIAGG: table bits
  uint8_t k, v;          // PAIR1 / PHASE1: register bit and value
  uint8_t treg[6];       // DIAGG: register bit of table bit j, or 0xFF
  uint8_t tphys[6];      // DIAGG: physical position of table bit j when not a register bit
  int tab;               // offset into the coefficient array
  int pad[2];
};
static_assert(sizeof(FOp) == 48, "FOp layout");

struct FPhase {
  uint8_t reg[kRB];      // tile positions held in registers
  uint8_t flip;          // absorbed X gates: logical register index j is stored in register j ^ flip
  uint8_t thr[kMaxB];    // tile positions of thread-index bits (b - 4 of them; lanes 0..2 first)
  int op_begin, op_end;
};

struct FPassArgs {
  int b;                 // tile bits
  int nthr;              // b - kRB
  unsigned char tpos[kMaxB];   // physical positions of tile bits (ascending)
  int n_outer_ins;
  u64 n_tiles;
  int phase_begin, n_phases;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// XOR swizzle of a tile index: linear over GF(2), so swz(a ^ b) == swz(a) ^ swz(b)
__device__ __forceinline__ int swz(int s) { return s ^ (((s >> 3) ^ (s >> 6) ^ (s >> 9)) & 7); }

// In-place friendly forms: every product that needs an OLD value is formed first, then the
// final FMAs overwrite x0 / x1.  This lets ptxas keep a[] in fixed registers across the op
// dispatch (the naive form costs ~4 register moves per amplitude per op at the switch merge).
template <int MT>
__device__ __forceinline__ void pair_upd(double2& x0, double2& x1, const double2 m0, const double2 m1, const double2 m2,
                                         const double2 m3) {
  if (MT == MT_X) {
    const double2 t = x0;
    x0 = x1;
    x1 = t;
  } else if (MT == MT_REAL) {
    const double px = m1.x * x1.x, py = m1.x * x1.y, qx = m2.x * x0.x, qy = m2.x * x0.y;
    x0.x = fma(m0.x, x0.x, px);
    x0.y = fma(m0.x, x0.y, py);
    x1.x = fma(m3.x, x1.x, qx);
    x1.y = fma(m3.x, x1.y, qy);
  } else if (MT == MT_RXLIKE) {   // m0, m3 real; m1, m2 imaginary: (i b)(x + i y) = -b y + i b x
    const double px = -m1.y * x1.y, py = m1.y * x1.x, qx = -m2.y * x0.y, qy = m2.y * x0.x;
    x0.x = fma(m0.x, x0.x, px);
    x0.y = fma(m0.x, x0.y, py);
    x1.x = fma(m3.x, x1.x, qx);
    x1.y = fma(m3.x, x1.y, qy);
  } else {
    const double2 p = cmul(m1, x1), q = cmul(m2, x0);
    x0 = cfma(m0, x0, p);
    x1 = cfma(m3, x1, q);
  }
}

// a *= d in place (cross products first)
__device__ __forceinline__ void cmul_ip(double2& a, const double2 d) {
  const double t1 = a.y * d.y, t2 = a.x * d.y;
  a.x = fma(a.x, d.x, -t1);
  a.y = fma(a.y, d.x, t2);
}

// fast path: every (r, r | 1<<K) pair, no register-side predicate
template <int K, int MT>
__device__ __forceinline__ void pair1(double2 (&a)[kRegs], const double2* __restrict__ c) {
  double2 m0, m1, m2, m3;
  if (MT != MT_X) {
    m0 = c[0]; m1 = c[1]; m2 = c[2]; m3 = c[3];
  }
#pragma unroll
  for (int r = 0; r < kRegs; ++r)
    if (!((r >> K) & 1)) pair_upd<MT>(a[r], a[r | (1 << K)], m0, m1, m2, m3);
}

// general pair: xmask XR in register space, runtime register pattern (cm, cv)
template <int XR, int MT>
__device__ __forceinline__ void pairg(double2 (&a)[kRegs], const double2* __restrict__ c, int cm, int cv) {
  double2 m0, m1, m2, m3;
  if (MT != MT_X) {
    m0 = c[0]; m1 = c[1]; m2 = c[2]; m3 = c[3];
  }
#pragma unroll
  for (int r = 0; r < kRegs; ++r)
    if ((r & cm) == cv) pair_upd<MT>(a[r], a[r ^ XR], m0, m1, m2, m3);
}

template <int K, int V>
__device__ __forceinline__ void phase1(double2 (&a)[kRegs], const double2 d) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r)
    if (((r >> K) & 1) == V) cmul_ip(a[r], d);
}

template <int K0, int K1>
__device__ __forceinline__ void dense2(double2 (&a)[kRegs], const double2* __restrict__ M, int cm, int cv) {
  constexpr int B0 = 1 << K0, B1 = 1 << K1;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r & (B0 | B1)) != 0) continue;
    if ((r & cm) != cv) continue;
    const int idx[4] = {r, r | B0, r | B1, r | B0 | B1};   // matrix index bit 0 <-> K0, bit 1 <-> K1
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = a[idx[q]];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) acc = cfma(M[q * 4 + cc], v[cc], acc);
      a[idx[q]] = acc;
    }
  }
}

__device__ __forceinline__ void diagg(double2 (&a)[kRegs], const FOp& op, const double2* __restrict__ coef,
                                      u64 phys_base) {
  // table index = tconst | sum_k bit_k(r) * w_k   (w_k built without dynamic register indexing)
  int tconst = 0, w0 = 0, w1 = 0, w2 = 0, w3 = 0;
  for (int j = 0; j < op.nt; ++j) {
    const int rg = op.treg[j];
    const int bit = 1 << j;
    if (rg == 0xFF) tconst |= int((phys_base >> op.tphys[j]) & 1ull) << j;
    w0 |= (rg == 0) ? bit : 0;
    w1 |= (rg == 1) ? bit : 0;
    w2 |= (rg == 2) ? bit : 0;
    w3 |= (rg == 3) ? bit : 0;
  }
  const int cm = op.cm, cv = op.cv;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r & cm) != cv) continue;
    const int t = tconst | ((r & 1) ? w0 : 0) | ((r & 2) ? w1 : 0) | ((r & 4) ? w2 : 0) | ((r & 8) ? w3 : 0);
    cmul_ip(a[r], coef[op.tab + t]);
  }
}

#define PAIR1_CASE(K)                                            \
  case K * 4 + MT_GENERAL: pair1<K, MT_GENERAL>(a, c); break;   \
  case K * 4 + MT_REAL: pair1<K, MT_REAL>(a, c); break;         \
  case K * 4 + MT_RXLIKE: pair1<K, MT_RXLIKE>(a, c); break;     \
  case K * 4 + MT_X: pair1<K, MT_X>(a, c); break;

#define PAIRG_CASE(XR)                                                              \
  case XR: if (!FULL || op.mtype == MT_X) pairg<XR, MT_X>(a, c, op.cm, op.cv);       \
           else pairg<XR, MT_GENERAL>(a, c, op.cm, op.cv); break;

// FULL = false compiles only the common kinds (PAIR1, PHASE1, SCALAR, X-type PAIRG): fewer live
// registers, no spills; passes that need DIAGG / DENSE2 / general PAIRG use the FULL kernel.
template <bool FULL>
__device__ __forceinline__ void apply_op(double2 (&a)[kRegs], const FOp& op, const double2* __restrict__ coef,
                                         u64 phys_base) {
  const double2* c = coef + op.tab;
  switch (op.kind) {
    case FK_PAIR1:
      switch (op.k * 4 + op.mtype) {
        PAIR1_CASE(0) PAIR1_CASE(1) PAIR1_CASE(2) PAIR1_CASE(3)
        default: break;
      }
      break;
    case FK_PHASE1: {
      const double2 d = c[0];
      switch (op.k * 2 + op.v) {
        case 0: phase1<0, 0>(a, d); break;
        case 1: phase1<0, 1>(a, d); break;
        case 2: phase1<1, 0>(a, d); break;
        case 3: phase1<1, 1>(a, d); break;
        case 4: phase1<2, 0>(a, d); break;
        case 5: phase1<2, 1>(a, d); break;
        case 6: phase1<3, 0>(a, d); break;
        case 7: phase1<3, 1>(a, d); break;
        default: break;
      }
      break;
    }
    case FK_SCALAR: {
      const double2 d = c[0];
#pragma unroll
      for (int r = 0; r < kRegs; ++r) cmul_ip(a[r], d);
      break;
    }
    case FK_PAIRG:
      switch (op.xr) {
        PAIRG_CASE(1) PAIRG_CASE(2) PAIRG_CASE(3) PAIRG_CASE(4) PAIRG_CASE(5) PAIRG_CASE(6) PAIRG_CASE(7)
        PAIRG_CASE(8) PAIRG_CASE(9) PAIRG_CASE(10) PAIRG_CASE(11) PAIRG_CASE(12) PAIRG_CASE(13)
        PAIRG_CASE(14) PAIRG_CASE(15)
        default: break;
      }
      break;
    case FK_DIAGG:
      if (FULL) diagg(a, op, coef, phys_base);
      break;
    case FK_DENSE2:
      if (FULL) switch (op.xr) {
        case 0x10: dense2<0, 1>(a, c, op.cm, op.cv); break;
        case 0x20: dense2<0, 2>(a, c, op.cm, op.cv); break;
        case 0x30: dense2<0, 3>(a, c, op.cm, op.cv); break;
        case 0x21: dense2<1, 2>(a, c, op.cm, op.cv); break;
        case 0x31: dense2<1, 3>(a, c, op.cm, op.cv); break;
        case 0x32: dense2<2, 3>(a, c, op.cm, op.cv); break;
        default: break;
      }
      break;
    default:
      break;
  }
}

// DB = true : one persistent CTA per SM, two tile buffers, tile t+grid prefetched during tile t.
// DB = false: two CTAs per SM (128 registers), one buffer each; CTAs overlap each other instead.
template <bool FULL, bool DB>
__global__ void __launch_bounds__(256, DB ? 1 : 2) k_fused(double2* __restrict__ state, const FPassArgs P,
                                                            const FPhase* __restrict__ phases,
                                                            const FOp* __restrict__ ops,
                                                            const double2* __restrict__ coef) {
  extern __shared__ double2 tile_mem[];   // DB: two tiles of 2^b amplitudes; else one
  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;            // 2^(b-4)
  // load slot i of this thread is tile index s = tid + nthreads * i
  u64 spread_tid = 0;
  for (int j = 0; j < P.nthr; ++j)
    if ((tid >> j) & 1) spread_tid |= 1ull << P.tpos[j];
  u64 hb[kRB];
#pragma unroll
  for (int j = 0; j < kRB; ++j) hb[j] = 1ull << P.tpos[P.nthr + j];
  const int swz_tid = swz(tid);
  int swz_hi[kRB];
#pragma unroll
  for (int j = 0; j < kRB; ++j) swz_hi[j] = swz(nthreads << j);
#define SPREAD_HI(i) ((((i) & 1) ? hb[0] : 0ull) | (((i) & 2) ? hb[1] : 0ull) | (((i) & 4) ? hb[2] : 0ull) | \
                      (((i) & 8) ? hb[3] : 0ull))
#define SWZ_HI(i) ((((i) & 1) ? swz_hi[0] : 0) ^ (((i) & 2) ? swz_hi[1] : 0) ^ (((i) & 4) ? swz_hi[2] : 0) ^ \
                   (((i) & 8) ? swz_hi[3] : 0))
  const int T = 1 << P.b;
  // tile index -> global base (insert zero bits at the tile positions)
  auto tile_base = [&](u64 t) {
    u64 base = t;
    for (int j = 0; j < P.b; ++j) {
      const int p = P.tpos[j];
      const u64 lo = base & ((1ull << p) - 1ull);
      base = ((base ^ lo) << 1) | lo;
    }
    return base;
  };
  // global -> shared (cp.async 16 B per amplitude, conflict-free through the swizzle), one group
  auto issue_load = [&](u64 t, double2* dst_buf) {
    const u64 gb = tile_base(t) | spread_tid;
#pragma unroll
    for (int i = 0; i < kRegs; ++i) {
      const double2* src = state + (gb | SPREAD_HI(i));
      const unsigned dst = (unsigned)__cvta_generic_to_shared(&dst_buf[swz_tid ^ SWZ_HI(i)]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // double buffer: tile t+grid streams in while tile t is being computed
  int cur = 0;
  if (DB && blockIdx.x < P.n_tiles) issue_load(blockIdx.x, tile_mem);
  for (u64 t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
    double2* tile = tile_mem + (DB ? cur * T : 0);
    if (!DB) {
      __syncthreads();   // previous tile fully stored before the buffer is refilled
      issue_load(t, tile_mem);
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    if (DB && t + gridDim.x < P.n_tiles) issue_load(t + gridDim.x, tile_mem + (cur ^ 1) * T);
    const u64 base = tile_base(t);
    const u64 gbase = base | spread_tid;
    for (int ph = 0; ph < P.n_phases; ++ph) {
      const FPhase& F = phases[P.phase_begin + ph];
      int sthr = 0;
      u64 phys_base = base;
      for (int j = 0; j < P.nthr; ++j)
        if ((tid >> j) & 1) {
          sthr |= 1 << F.thr[j];
          phys_base |= 1ull << P.tpos[F.thr[j]];
        }
      const int s0 = swz(sthr);
      const int W0 = swz(1 << F.reg[0]), W1 = swz(1 << F.reg[1]), W2 = swz(1 << F.reg[2]), W3 = swz(1 << F.reg[3]);
#define REG_OFF(r) (s0 ^ (((r) & 1) ? W0 : 0) ^ (((r) & 2) ? W1 : 0) ^ (((r) & 4) ? W2 : 0) ^ (((r) & 8) ? W3 : 0))
      double2 a[kRegs];
#pragma unroll
      for (int r = 0; r < kRegs; ++r) a[r] = tile[REG_OFF(r)];
      for (int oi = F.op_begin; oi < F.op_end; ++oi) {
        const FOp op = ops[oi];
        if ((phys_base & op.pm) != op.pv) continue;
        apply_op<FULL>(a, op, coef, phys_base);
      }
      {
        // register r holds logical index r ^ flip: store offset = swz(sthr) ^ W(r ^ flip) (W linear)
        const int fl = F.flip;
        const int sf = s0 ^ ((fl & 1) ? W0 : 0) ^ ((fl & 2) ? W1 : 0) ^ ((fl & 4) ? W2 : 0) ^ ((fl & 8) ? W3 : 0);
#pragma unroll
        for (int r = 0; r < kRegs; ++r)
          tile[sf ^ ((r & 1) ? W0 : 0) ^ ((r & 2) ? W1 : 0) ^ ((r & 4) ? W2 : 0) ^ ((r & 8) ? W3 : 0)] = a[r];
      }
      __syncthreads();
#undef REG_OFF
    }
    // shared -> global (this buffer is refilled only after the next iteration's barrier)
#pragma unroll
    for (int i = 0; i < kRegs; ++i) state[gbase | SPREAD_HI(i)] = tile[swz_tid ^ SWZ_HI(i)];
    cur ^= 1;
  }
#undef SPREAD_HI
#undef SWZ_HI
}

// ===========================================================================
// host planner
// ===========================================================================
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

struct PassPlan {
  bool fused = false;
  int single = -1;            // prim index when not fused
  u64 tile_bits = 0;
  std::vector<int> prims;     // in application order
};

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
      bool ok = k < window && r.fusable;
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

struct Program {
  std::vector<FPassArgs> passes;
  std::vector<char> full;          // pass needs the FULL kernel variant
  std::vector<int> pass_of;        // for singles: -1
  std::vector<FPhase> phases;
  std::vector<FOp> ops;
  std::vector<double2> coef;
};

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
  int F = 0;
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
        op.mtype = uint8_t(mt == MT_X ? MT_X : MT_GENERAL);
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
    bool full = false;
    for (int ph = A.phase_begin; ph < A.phase_begin + A.n_phases; ++ph)
      for (int oi = prog.phases[ph].op_begin; oi < prog.phases[ph].op_end; ++oi) {
        const FOp& o = prog.ops[oi];
        full |= o.kind == FK_DIAGG || o.kind == FK_DENSE2 || (o.kind == FK_PAIRG && o.mtype != MT_X);
      }
    prog.full.push_back(full ? 1 : 0);
    prog.passes.push_back(A);
  }
  return prog;
}

struct DevProgram {
  void* buf = nullptr;
  size_t cap = 0;
};
std::mutex g_prog_mu;
std::vector<std::pair<sv_handle*, DevProgram>> g_progs;

void* program_buffer(sv_handle* h, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_prog_mu);
  for (auto& e : g_progs)
    if (e.first == h) {
      if (e.second.cap < bytes) {
        CUDA_CHECK(cudaStreamSynchronize(h->stream));
        CUDA_CHECK(cudaFree(e.second.buf));
        e.second.cap = std::max(bytes, size_t(1) << 20);
        CUDA_CHECK(cudaMalloc(&e.second.buf, e.second.cap));
      }
      return e.second.buf;
    }
  DevProgram d;
  d.cap = std::max(bytes, size_t(1) << 20);
  CUDA_CHECK(cudaMalloc(&d.buf, d.cap));
  g_progs.push_back({h, d});
  return d.buf;
}

}  // namespace

void release_fused(sv_handle* h) {
  std::lock_guard<std::mutex> lk(g_prog_mu);
  for (size_t i = 0; i < g_progs.size(); ++i)
    if (g_progs[i].first == h) {
      cudaFree(g_progs[i].second.buf);
      g_progs.erase(g_progs.begin() + i);
      return;
    }
}

void apply_prims_fused(sv_handle* h, double2* state, const std::vector<Prim>& prims) {
  if (h->nl < 5) {
    for (const Prim& p : prims) launch_prim(h, state, p);
    return;
  }
  std::vector<PassPlan> plan;
  Program prog = build_program(h->nl, prims, plan);
  if (prog.passes.empty()) {
    for (const Prim& p : prims) launch_prim(h, state, p);
    return;
  }
  // upload phases | ops | coef in one copy (the buffer is only reused after a stream sync)
  const size_t b_ph = prog.phases.size() * sizeof(FPhase);
  const size_t b_op = prog.ops.size() * sizeof(FOp);
  const size_t b_cf = prog.coef.size() * sizeof(double2);
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t total = align(b_ph) + align(b_op) + align(b_cf);
  std::vector<char> host(total);
  std::memcpy(host.data(), prog.phases.data(), b_ph);
  std::memcpy(host.data() + align(b_ph), prog.ops.data(), b_op);
  std::memcpy(host.data() + align(b_ph) + align(b_op), prog.coef.data(), b_cf);
  CUDA_CHECK(cudaStreamSynchronize(h->stream));   // previous program may still be in use
  char* dbuf = (char*)program_buffer(h, total);
  CUDA_CHECK(cudaMemcpyAsync(dbuf, host.data(), total, cudaMemcpyHostToDevice, h->stream));
  const FPhase* d_ph = (const FPhase*)dbuf;
  const FOp* d_op = (const FOp*)(dbuf + align(b_ph));
  const double2* d_cf = (const double2*)(dbuf + align(b_ph) + align(b_op));

  static bool attr_set = false;
  static int dev_sms = 148;
  static bool db = true;
  const int b = prog.passes[0].b;
  if (!attr_set) {
    const int maxs = int(2 * (size_t(1) << kMaxB) * sizeof(double2));
    CUDA_CHECK(cudaFuncSetAttribute(k_fused<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs));
    CUDA_CHECK(cudaFuncSetAttribute(k_fused<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs));
    CUDA_CHECK(cudaFuncSetAttribute(k_fused<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs / 2));
    CUDA_CHECK(cudaFuncSetAttribute(k_fused<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs / 2));
    CUDA_CHECK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, h->device));
    const char* mode = getenv("SVB200_FUSED_MODE");   // "sb": single-buffer 2 CTAs/SM (experiments)
    db = !(mode && std::string(mode) == "sb");
    attr_set = true;
  }
  const size_t smem = (db ? 2 : 1) * (size_t(1) << b) * sizeof(double2);
  size_t pi = 0;
  for (auto& pp : plan) {
    if (!pp.fused) {
      launch_prim(h, state, prims[pp.single]);
      continue;
    }
    const FPassArgs& A = prog.passes[pi++];
    const int threads = 1 << (A.b - kRB);
    // persistent grid: one (DB) or two CTAs per SM
    const u64 grid = std::min<u64>(A.n_tiles, u64(dev_sms) * (db ? 1 : 2));
    const double bytes = 32.0 * double(h->n_local);
    cudaEvent_t ev[2];
    stat_begin(h, KC_FUSED, bytes, ev);
    const bool full = prog.full[pi - 1];
    if (db && full)
      k_fused<true, true><<<unsigned(grid), threads, smem, h->stream>>>(state, A, d_ph, d_op, d_cf);
    else if (db)
      k_fused<false, true><<<unsigned(grid), threads, smem, h->stream>>>(state, A, d_ph, d_op, d_cf);
    else if (full)
      k_fused<true, false><<<unsigned(grid), threads, smem, h->stream>>>(state, A, d_ph, d_op, d_cf);
    else
      k_fused<false, false><<<unsigned(grid), threads, smem, h->stream>>>(state, A, d_ph, d_op, d_cf);
    stat_end(h, KC_FUSED, bytes, ev);
    CUDA_CHECK(cudaGetLastError());
  }
}

PlanStats plan_stats(int nl, const std::vector<Prim>& prims) {
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
