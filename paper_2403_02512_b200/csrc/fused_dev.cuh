// K7 device-side building blocks, shared by the prebuilt op-interpreting tile kernel (fused.cu)
// and the per-pass specialised kernels the runtime pass compiler generates (fused_jit.cpp hands
// this file, verbatim, to NVRTC in front of every generated kernel).  Self-contained: no host
// headers, nothing but CUDA built-ins.
//
// Register model (see fused.cu): a thread holds 16 amplitudes a[r] of its tile, r = the 4
// "register bits".  Every update below is in place (a[] never moves between registers).
#pragma once

typedef unsigned long long u64;

namespace fdev {

constexpr int kMaxB = 12;        // tile bits (2^12 amplitudes = 64 KiB)
constexpr int kRB = 4;           // register bits per thread
constexpr int kRegs = 1 << kRB;  // amplitudes per thread
constexpr int kTB = kMaxB - kRB; // max thread-index bits
constexpr int kMaxGens = 64;     // generator slots per pass (per-warp shared accumulators)
constexpr int kGenSub = 4;       // accumulators per warp and slot in run_pass: one per 8-lane group
constexpr int kMtGeneral = 0, kMtReal = 1, kMtRxLike = 2;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// XOR swizzle of a tile index: linear over GF(2), so swz(a ^ b) == swz(a) ^ swz(b)
__device__ __forceinline__ int swz(int s) { return s ^ (((s >> 3) ^ (s >> 6) ^ (s >> 9)) & 7); }

// In-place 2x2 update of (x0, x1): products needing OLD values first, then overwriting FMAs.
template <int MT>
__device__ __forceinline__ void pair_upd(double2& x0, double2& x1, const double2 m0, const double2 m1, const double2 m2,
                                         const double2 m3) {
  if (MT == kMtReal) {
    const double px = m1.x * x1.x, py = m1.x * x1.y, qx = m2.x * x0.x, qy = m2.x * x0.y;
    x0.x = fma(m0.x, x0.x, px);
    x0.y = fma(m0.x, x0.y, py);
    x1.x = fma(m3.x, x1.x, qx);
    x1.y = fma(m3.x, x1.y, qy);
  } else if (MT == kMtRxLike) {   // m0, m3 real; m1, m2 imaginary: (i b)(x + i y) = -b y + i b x
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

// every (r, r | 1<<K) pair, no register-side predicate
template <int K, int MT>
__device__ __forceinline__ void pair1(double2 (&a)[kRegs], const double2 m0, const double2 m1, const double2 m2,
                                      const double2 m3) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r)
    if (!((r >> K) & 1)) pair_upd<MT>(a[r], a[r | (1 << K)], m0, m1, m2, m3);
}

// general pair: xmask XR in register space, runtime register pattern (cm, cv)
template <int XR, int MT>
__device__ __forceinline__ void pairg(double2 (&a)[kRegs], const double2 m0, const double2 m1, const double2 m2,
                                      const double2 m3, int cm, int cv) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r)
    if ((r & cm) == cv) pair_upd<MT>(a[r], a[r ^ XR], m0, m1, m2, m3);
}

// register-controlled X (CNOT-type) on register xmask XR: a[r] <-> a[r ^ XR] for the registers
// whose control bits CC equal CV.  Control bits without a per-thread flip in this phase resolve at
// compile time -- the swap is a register renaming, no instructions at all; bits that may carry a
// flip (MD, runtime value fthr) select at run time (SEL on the integer pipe, no FP64).
// XP = i0's pattern on XR (a multi-bit XR, e.g. SWAP, exchanges only the pairs through XP).
template <int XR, int CC, int CV, int MD, int XP>
__device__ __forceinline__ void swap_x(double2 (&a)[kRegs], const int fthr) {
  constexpr int LOW = XR & -XR;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if (r & LOW) continue;   // one representative per pair {r, r ^ XR}
    if ((r & XR) != XP && ((r ^ XR) & XR) != XP) continue;
    if ((r & CC & ~MD) != (CV & CC & ~MD)) continue;
    if (MD & CC) {
      const bool c = (r & MD) == ((CV ^ fthr) & MD);
      const double2 x0 = a[r], x1 = a[r ^ XR];
      a[r] = c ? x1 : x0;
      a[r ^ XR] = c ? x0 : x1;
    } else {
      const double2 t = a[r];
      a[r] = a[r ^ XR];
      a[r ^ XR] = t;
    }
  }
}

// rotation R(phi) of every (x0, x1) pair on register bit K as shears u += t v; v += s u; u += t v
// (RY type: on (re0, re1) and (im0, im1); RX type: R(-phi) on (re0, im1), R(phi) on (im0, re1))
template <int K, bool RX>
__device__ __forceinline__ void pair_shear(double2 (&a)[kRegs], const double t, const double s) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r >> K) & 1) continue;
    double2& x0 = a[r];
    double2& x1 = a[r | (1 << K)];
    if (RX) {
      x0.x = fma(-t, x1.y, x0.x);
      x0.y = fma(t, x1.x, x0.y);
      x1.y = fma(-s, x0.x, x1.y);
      x1.x = fma(s, x0.y, x1.x);
      x0.x = fma(-t, x1.y, x0.x);
      x0.y = fma(t, x1.x, x0.y);
    } else {
      x0.x = fma(t, x1.x, x0.x);
      x0.y = fma(t, x1.y, x0.y);
      x1.x = fma(s, x0.x, x1.x);
      x1.y = fma(s, x0.y, x1.y);
      x0.x = fma(t, x1.x, x0.x);
      x0.y = fma(t, x1.y, x0.y);
    }
  }
}

// rotation R(phi) of every (x0, x1) pair on register bit K, scaled: R/cos(phi) (TAN, t = tan phi)
// or R/sin(phi) (COT, t = cot phi) -- 2 FMAs per real pair instead of the shears' 3; the pass owes
// the state the dropped factor, absorbed once per pass by the planner (fused_plan.cpp).
//   RY type R = [[c, -s], [s, c]]:     TAN x0 - t x1, x1 + t x0          COT t x0 - x1, t x1 + x0
//   RX type R = [[c, -is], [-is, c]]:  TAN x0 - i t x1, x1 - i t x0      COT t x0 - i x1, t x1 - i x0
// NEG: the flipped roles of a per-thread flip, R(-phi) (RY type; TAN negates t, COT the +-1 terms)
template <int K, bool RX, bool COT, bool NEG = false>
__device__ __forceinline__ void pair_tan(double2 (&a)[kRegs], double t) {
  if (NEG && !COT) t = -t;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r >> K) & 1) continue;
    double2& x0 = a[r];
    double2& x1 = a[r | (1 << K)];
    const double2 y0 = x0, y1 = x1;
    if (RX) {   // -i t x = t x.y - i t x.x
      if (COT) {
        x0.x = fma(t, y0.x, y1.y);
        x0.y = fma(t, y0.y, -y1.x);
        x1.x = fma(t, y1.x, y0.y);
        x1.y = fma(t, y1.y, -y0.x);
      } else {
        x0.x = fma(t, y1.y, y0.x);
        x0.y = fma(-t, y1.x, y0.y);
        x1.x = fma(t, y0.y, y1.x);
        x1.y = fma(-t, y0.x, y1.y);
      }
    } else {
      if (COT && NEG) {
        x0.x = fma(t, y0.x, y1.x);
        x0.y = fma(t, y0.y, y1.y);
        x1.x = fma(t, y1.x, -y0.x);
        x1.y = fma(t, y1.y, -y0.y);
      } else if (COT) {
        x0.x = fma(t, y0.x, -y1.x);
        x0.y = fma(t, y0.y, -y1.y);
        x1.x = fma(t, y1.x, y0.x);
        x1.y = fma(t, y1.y, y0.y);
      } else {
        x0.x = fma(-t, y1.x, y0.x);
        x0.y = fma(-t, y1.y, y0.y);
        x1.x = fma(t, y0.x, y1.x);
        x1.y = fma(t, y0.y, y1.y);
      }
    }
  }
}

// a[r] *= d for registers r with parity(r & M) == 1 ^ tp (tp: the thread's parity part)
template <int M>
__device__ __forceinline__ void parity_phase(double2 (&a)[kRegs], const double2 d, const int tp) {
  if (tp) {
#pragma unroll
    for (int r = 0; r < kRegs; ++r)
      if (!(__popc(r & M) & 1)) cmul_ip(a[r], d);
  } else {
#pragma unroll
    for (int r = 0; r < kRegs; ++r)
      if (__popc(r & M) & 1) cmul_ip(a[r], d);
  }
}

template <int K, int V>
__device__ __forceinline__ void phase1(double2 (&a)[kRegs], const double2 d) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r)
    if (((r >> K) & 1) == V) cmul_ip(a[r], d);
}

template <int K0, int K1>
__device__ __forceinline__ void dense2(double2 (&a)[kRegs], const double2* __restrict__ M, int cm, int cv, int f) {
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
      for (int cc = 0; cc < 4; ++cc) acc = cfma(M[(q ^ f) * 4 + (cc ^ f)], v[cc], acc);
      a[idx[q]] = acc;
    }
  }
}

// diagonal table: a[r] *= tab[tconst ^ W(r)], W(r) = the table bits register r carries (compile-time
// when the planner's table layout is known, i.e. in generated pass kernels)
template <int W0, int W1, int W2, int W3>
__device__ __forceinline__ void diag_tab(double2 (&a)[kRegs], const double2* __restrict__ tab, int tconst, int cm,
                                         int cv) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r & cm) != cv) continue;
    const int t = tconst ^ (((r & 1) ? W0 : 0) | ((r & 2) ? W1 : 0) | ((r & 4) ? W2 : 0) | ((r & 8) ? W3 : 0));
    cmul_ip(a[r], tab[t]);
  }
}

// ---- adjoint bra-kets: psi and lambda share the tile (register bit T selects lambda) --------
__device__ __forceinline__ void cacc_conj(double& re, double& im, const double2 l, const double2 t) {
  re = fma(l.x, t.x, fma(l.y, t.y, re));   // conj(l) * t
  im = fma(l.x, t.y, fma(-l.y, t.x, im));
}

template <int K, int T>
__device__ __forceinline__ void gen1(const double2 (&a)[kRegs], const double2 g0, const double2 g1, const double2 g2,
                                     const double2 g3, int cm, int cv, double& re, double& im) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if (((r >> K) & 1) || ((r >> T) & 1)) continue;
    if ((r & cm) != cv) continue;
    const double2 p0 = a[r], p1 = a[r | (1 << K)];
    const double2 l0 = a[r | (1 << T)], l1 = a[r | (1 << K) | (1 << T)];
    cacc_conj(re, im, l0, cfma(g0, p0, cmul(g1, p1)));
    cacc_conj(re, im, l1, cfma(g2, p0, cmul(g3, p1)));
  }
}

template <int K0, int K1, int T>
__device__ __forceinline__ void gen2(const double2 (&a)[kRegs], const double2* __restrict__ M, int cm, int cv, int f,
                                     double& re, double& im) {
  constexpr int B0 = 1 << K0, B1 = 1 << K1, BT = 1 << T;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if (r & (B0 | B1 | BT)) continue;
    if ((r & cm) != cv) continue;
    const int idx[4] = {r, r | B0, r | B1, r | B0 | B1};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < 4; ++c) acc = cfma(M[(q ^ f) * 4 + (c ^ f)], a[idx[c]], acc);
      cacc_conj(re, im, a[idx[q] | BT], acc);
    }
  }
}

// diagonal generator over a table (like diag_tab): sum_r conj(lambda_r) g[t(r)] psi_r
template <int T, int W0, int W1, int W2, int W3>
__device__ __forceinline__ void gen_diag_tab(const double2 (&a)[kRegs], const double2* __restrict__ tab, int tconst,
                                             int cm, int cv, double& re, double& im) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r >> T) & 1) continue;
    if ((r & cm) != cv) continue;
    const int t = tconst ^ (((r & 1) ? W0 : 0) | ((r & 2) ? W1 : 0) | ((r & 4) ? W2 : 0) | ((r & 8) ? W3 : 0));
    cacc_conj(re, im, a[r | (1 << T)], cmul(tab[t], a[r]));
  }
}

// diagonal generator whose table is a parity table (1 on even-parity indices, d on odd: Z, Z..Z):
// sum_r conj(lambda_r) g psi_r = S_even + d S_odd -- no table loads, no complex product per amplitude.
// M = register bits carrying table bits, tp = parity of the table's off-register bits and flips.
template <int T, int M>
__device__ __forceinline__ void gen_parity(const double2 (&a)[kRegs], const double2 d, int tp, int cm, int cv,
                                           double& re, double& im) {
  double er = 0.0, ei = 0.0, orr = 0.0, oi = 0.0;   // register parity 0 / 1 sums
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r >> T) & 1) continue;
    if ((r & cm) != cv) continue;
    if (__popc(r & M) & 1) cacc_conj(orr, oi, a[r | (1 << T)], a[r]);
    else cacc_conj(er, ei, a[r | (1 << T)], a[r]);
  }
  if (tp) {   // the thread's off-register parity swaps the roles
    double t0 = er, t1 = ei;
    er = orr;
    ei = oi;
    orr = t0;
    oi = t1;
  }
  re += er + (d.x * orr - d.y * oi);
  im += ei + (d.x * oi + d.y * orr);
}

// reduce one bra-ket over groups of 32 / SUB lanes and add each group's sum to its own accumulator
// of this warp's slot (every lane calls).  SUB = 4: 3 shuffle rounds instead of 5 per bra-ket, the
// four 8-lane sums land in adjacent accumulators (conflict-free); the end of the kernel adds them in
// fixed order with the warps' (deterministic).
template <int SUB>
__device__ __forceinline__ void gen_commit(double re, double im, double2* __restrict__ acc_warp, int slot) {
  for (int s = 16 / SUB; s > 0; s >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, s);
    im += __shfl_xor_sync(0xffffffffu, im, s);
  }
  if ((threadIdx.x & (32 / SUB - 1)) == 0) {
    double2& c = acc_warp[slot * SUB + (threadIdx.x & 31) / (32 / SUB)];
    c.x += re;
    c.y += im;
  }
}

// Launch-time records derived from the planned program (computed once on the host): see fused.cu.
// The thread-index -> (swizzled shared offset, physical bits) maps of a phase are GF(2)-linear in
// the thread index (<= 8 bits), so each is two 16-entry nibble tables: s0 = s_lo[tid & 15] ^
// s_hi[tid >> 4].
struct __align__(16) DPhase {
  int W[kRB];        // swz(1 << reg[k]): offset of register bit k
  int s_lo[16], s_hi[16];   // swizzled shared offset of the thread's slot, per tid nibble
  u64 g_lo[16], g_hi[16];   // physical bits of the thread's slot, per tid nibble
  int op_begin, op_end;     // pass-local op range
  int flip, pad;
};
static_assert(sizeof(DPhase) == 416, "DPhase layout");
static_assert(kTB <= 8, "two tid nibbles");

struct DPass {
  u64 n_tiles;
  u64 outer;           // physical bits NOT in the tile (the tile index deposits into these)
  u64 grid_step;       // deposit(gridDim.x): tile t -> t + grid is a masked add
  u64 grid_step2;      // deposit(2 gridDim.x), deposit(3 gridDim.x) (ping-pong tile loop)
  u64 grid_step3;
  u64 hi;              // two-array state: indices with this bit live in state_hi
  u64 ld_off[kRegs];   // load slot i: physical offset of its register-slot bits (without hi)
  u64 st_off[kRegs];   // store slot i: the same after the pass's in-tile relabeling
  u64 ld_tb[kTB];      // physical bit of thread-index bit j at load (may be hi)
  u64 st_tb[kTB];      // ... at store
  int ld_sm[kRegs];    // swizzled shared offset of load slot i
  int st_sm[kRegs];    // swizzled shared offset of store slot i
  int st_tsm[kTB];     // swizzled shared offset of thread-index bit j at store
  unsigned ld_hsel, st_hsel;   // slots whose index carries the hi bit
  int b, nthr, n_phases, n_ops, n_gen, gen_base, n_gen_total, pad;
  u64 gbits;           // sharded rank-uniform programs: this rank's global bits (positions >= nl),
                       // ORed into every predicate base (never into addresses)
};

// The tile loop of one pass for the generated (per-pass specialised) kernels: persistent CTAs;
// stage -> body(tile, phase records, tile base, warp accumulators) -> store with the pass's in-tile
// relabeling -> next tile.  Same data movement as k_fused<*, DB, TWO>:
//   DB = false: 2 CTAs per SM, one tile buffer each (the two CTAs overlap each other);
//   DB = true : 1 CTA per SM, two tile buffers: tile t + grid streams in while tile t is computed.
// Dynamic shared memory: [tile buffer(s)] [phase records] [generator accumulators].
//   DIRECT (single buffer, one array): the body's last phase stores its registers straight to HBM
//   and calls next_load() once it has read the tile, so the next tile streams into the buffer while
//   the last phase computes; the loop itself then has no store.
//   SPLIT (with DIRECT): the tile lives in two half buffers (index bit b-1 selects the half) and a
//   third half buffer rotates with the low one: the next tile's low half streams in during the
//   whole of this tile's phases, its high half during the last phase (3 half tiles = 96 KiB per
//   CTA, two CTAs per SM).
//   DFL (with DIRECT): no staged load at all -- the first phase reads its registers straight from
//   global memory (L2 hits: every tile's 128-byte lines were prefetched into L2 with
//   cp.async.bulk.prefetch while the CTA's previous tile was computed), saving the tile's
//   shared-memory write and first read; next_load() then issues the following tile's L2 prefetch.
template <bool TWO, bool DB, bool DIRECT, class Body, bool SPLIT = false, bool DFL = false>
__device__ __forceinline__ void run_pass(double2* __restrict__ state, double2* __restrict__ state_hi, const DPass& P,
                                         const DPhase* __restrict__ phases, double2* __restrict__ gen_partials,
                                         Body body) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* tile = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;
  const int T = 1 << P.b;
  DPhase* s_ph = reinterpret_cast<DPhase*>(smem_raw + size_t(DB ? 4 : (SPLIT ? 3 : 2)) * (T >> 1) * sizeof(double2));
  double2* s_gen = reinterpret_cast<double2*>(s_ph + P.n_phases);
  {
    const int4* src = reinterpret_cast<const int4*>(phases);
    int4* dst = reinterpret_cast<int4*>(s_ph);
    const int n16p = P.n_phases * int(sizeof(DPhase) / 16);
    for (int i = tid; i < n16p; i += nthreads) dst[i] = src[i];
    if (P.n_gen)
      for (int i = tid; i < (nthreads >> 5) * kMaxGens * kGenSub; i += nthreads) s_gen[i] = make_double2(0.0, 0.0);
  }
  u64 ld_tid = 0, st_tid = 0;
  int st_sw = 0;
#pragma unroll
  for (int j = 0; j < kTB; ++j)
    if (j < P.nthr && ((tid >> j) & 1)) {
      ld_tid |= P.ld_tb[j];
      st_tid |= P.st_tb[j];
      st_sw ^= P.st_tsm[j];
    }
  const int ld_sw = swz(tid);
  auto slot_ptrs = [&](u64 g, double2*& p_lo, double2*& p_hi) {
    if (!TWO) {
      p_lo = p_hi = state + g;
      return;
    }
    const u64 gl = g & ~P.hi;
    p_hi = state_hi + gl;
    p_lo = (g & P.hi) ? p_hi : state + gl;
  };
  u64 base = 0;
  {
    u64 m = P.outer;
    for (u64 v = blockIdx.x; m && v; m &= m - 1, v >>= 1)
      if (v & 1) base |= m & (~m + 1);
  }
  double2* acc_warp = s_gen + (tid >> 5) * kMaxGens * kGenSub;
  auto issue_load = [&](u64 b0, double2* buf) {
    double2 *p_lo, *p_hi;
    slot_ptrs(b0 | ld_tid, p_lo, p_hi);
    const unsigned sb = (unsigned)__cvta_generic_to_shared(buf);
#pragma unroll
    for (int i = 0; i < kRegs; ++i) {
      const double2* src = (TWO && ((P.ld_hsel >> i) & 1) ? p_hi : p_lo) + P.ld_off[i];
      const unsigned dst = sb + unsigned(ld_sw ^ P.ld_sm[i]) * 16u;
#ifndef FDEV_EXP_NOMEM
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
#else
      (void)dst;
      (void)src;
#endif
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  int cur = 0;
  if (DFL) {
    // L2 prefetch of a tile: its 2^(b-3) 128-byte lines, two per thread (thread group tid >> 3
    // covers the lines of load slots tid & 7 and (tid & 7) + 8, as issue_load would read them)
    auto prefetch_tile = [&](u64 b0) {
      double2 *p_lo, *p_hi;
      slot_ptrs(b0 | (ld_tid & ~7ull), p_lo, p_hi);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = (tid & 7) + 8 * h;
        const double2* src = (TWO && ((P.ld_hsel >> i) & 1) ? p_hi : p_lo) + P.ld_off[i];
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;\n" ::"l"(src) : "memory");
      }
    };
    for (u64 t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
      const u64 nbase = ((base | ~P.outer) + P.grid_step) & P.outer;
      if (t == blockIdx.x) {
        __syncthreads();   // phase records and generator accumulators staged
        prefetch_tile(base);
      }
      const bool more = t + gridDim.x < P.n_tiles;
      body(tile, tile + (T >> 1), s_ph, base, acc_warp, [&]() {
        if (more) prefetch_tile(nbase);
      });
      base = nbase;
    }
  } else if (SPLIT) {
    const int HB = T >> 1;
    auto issue_half = [&](u64 b0, double2* buf, int h) {
      double2 *p_lo, *p_hi;
      slot_ptrs(b0 | ld_tid, p_lo, p_hi);
      const unsigned sb = (unsigned)__cvta_generic_to_shared(buf);
#pragma unroll
      for (int i = 8 * h; i < 8 * h + 8; ++i) {   // slot bit 3 is tile index bit b-1
        const double2* src = (TWO && ((P.ld_hsel >> i) & 1) ? p_hi : p_lo) + P.ld_off[i];
        const unsigned dst = sb + unsigned((ld_sw ^ P.ld_sm[i]) & (HB - 1)) * 16u;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    double2* lo_cur = tile;
    double2* lo_spare = tile + HB;
    double2* hi_buf = tile + 2 * HB;
    for (u64 t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
      const u64 nbase = ((base | ~P.outer) + P.grid_step) & P.outer;
      if (t == blockIdx.x) {
        __syncthreads();   // phase records staged
        issue_half(base, lo_cur, 0);
        issue_half(base, hi_buf, 1);
      }
      asm volatile("cp.async.wait_all;\n" ::);
      __syncthreads();
      const bool more = t + gridDim.x < P.n_tiles;
      if (more) issue_half(nbase, lo_spare, 0);   // its last readers passed the barrier above
      body(lo_cur, hi_buf, s_ph, base, acc_warp, [&]() {
        if (more) issue_half(nbase, hi_buf, 1);
      });
      double2* tmp = lo_cur;
      lo_cur = lo_spare;
      lo_spare = tmp;
      base = nbase;
    }
  } else if (DIRECT) {
#ifdef FDEV_STAGGER_NS
    // the two CTAs sharing an SM would otherwise run in lockstep (load together, compute together)
    if (FDEV_STAGGER_SEL) __nanosleep(FDEV_STAGGER_NS);
#endif
    for (u64 t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
      const u64 nbase = ((base | ~P.outer) + P.grid_step) & P.outer;
      if (t == blockIdx.x) {
        __syncthreads();   // phase records staged
        issue_load(base, tile);
      }
      asm volatile("cp.async.wait_all;\n" ::);
      __syncthreads();
      const bool more = t + gridDim.x < P.n_tiles;
      body(tile, tile + (T >> 1), s_ph, base, acc_warp, [&]() {
        if (more) issue_load(nbase, tile);
      });
      base = nbase;
    }
  } else {
  if (DB && blockIdx.x < P.n_tiles) {
    __syncthreads();   // phase records staged
    issue_load(base, tile);
  }
  for (u64 t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
    const u64 nbase = ((base | ~P.outer) + P.grid_step) & P.outer;
    double2* tl = tile + (DB ? cur * T : 0);
    if (!DB) {
      __syncthreads();   // previous tile stored (and phase records staged) before the buffer is refilled
      issue_load(base, tile);
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    // DB: the other buffer's previous tile was fully read by the store loop before this barrier
    if (DB && t + gridDim.x < P.n_tiles) issue_load(nbase, tile + (cur ^ 1) * T);
    body(tl, tl + (T >> 1), s_ph, base, acc_warp, []() {});   // every phase, each ending with __syncthreads()
    {
      double2 *p_lo, *p_hi;
      slot_ptrs(base | st_tid, p_lo, p_hi);
#pragma unroll
      for (int i = 0; i < kRegs; ++i)
        (TWO && ((P.st_hsel >> i) & 1) ? p_hi : p_lo)[P.st_off[i]] = tl[st_sw ^ P.st_sm[i]];
    }
    base = nbase;
    cur ^= 1;
  }
  }
  if (P.n_gen) {
    __syncthreads();
    const int nw = nthreads >> 5;
    for (int g = tid; g < P.n_gen; g += nthreads) {
      double2 s = make_double2(0.0, 0.0);
      for (int w = 0; w < nw; ++w)
        for (int q = 0; q < kGenSub; ++q) {
          s.x += s_gen[(w * kMaxGens + g) * kGenSub + q].x;
          s.y += s_gen[(w * kMaxGens + g) * kGenSub + q].y;
        }
      gen_partials[size_t(blockIdx.x) * P.n_gen_total + P.gen_base + g] = s;
    }
  }
}

// ---- ping-pong tile loop (generated kernels, PP): two consumer groups, three tile buffers ------
//
// One 512-thread CTA per SM = two groups of 8 warps (A = threads 0..255, B = 256..511), each working
// on its own tile (A: the CTA's even local tiles, B: odd), in three rotating 64 KiB buffers.  A tile
// is 2P "segments": T_k (phase k's smem round trip: store phase k-1's registers, group barrier, load
// phase k's registers) and C_k (phase k's gate arithmetic).  Every segment ends with a CTA-wide step
// barrier, and group B runs an odd number of segments behind A, so the two groups are always in
// opposite segment kinds: one group's FP64 arithmetic runs while the other group's shared-memory
// round trip runs (two free-running CTAs per SM instead drift into lockstep -- they contend for the
// same pipe at the same time -- and the FP64 and shared-memory work of a pass then add up).
// Loads: a group's last phase, once its registers hold the tile, refills the buffer with the CTA's
// local tile j+3 by cp.async (16 B per amplitude, through the swizzle) whose completion arrives on
// the buffer's mbarrier (cp.async.mbarrier.arrive.noinc, 256 arrivals per fill); the consumer --
// the other group -- waits on the mbarrier's phase parity before its first phase.  The prefetch
// distance is ~P segments, i.e. the load overlaps both groups' work.
__device__ __forceinline__ void step_barrier() { asm volatile("barrier.sync 0;\n" ::: "memory"); }
__device__ __forceinline__ void group_barrier() {
  asm volatile("barrier.sync %0, 256;\n" ::"r"(1 + (int(threadIdx.x) >> 8)) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned addr, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(unsigned addr) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned addr, unsigned parity) {
  asm volatile(
      "{\n"
      "  .reg .pred p;\n"
      "SVB200_WAIT_%=:\n"
      "  mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "  @!p bra SVB200_WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ u64 masked_add(u64 base, u64 outer, u64 step) { return ((base | ~outer) + step) & outer; }

constexpr int kPPThreads = 512;
// dynamic shared memory of the PP loop: [3 tile buffers][3 mbarriers + pad][generator accumulators]
__host__ __device__ constexpr unsigned pp_smem_bytes(int b, bool gens) {
  return 3u * (1u << b) * 16u + 32u + (gens ? unsigned(kPPThreads / 32) * kMaxGens * 16u : 0u);
}

#ifdef FDEV_SEGPROF
__shared__ long long fdev_prof[2][64][2];
__shared__ long long fdev_tl[2];
#define fdev_t fdev::fdev_tl[threadIdx.x >> 8]
#endif
template <bool TWO, class Body>
__device__ __forceinline__ void run_pass_pp(double2* __restrict__ state, double2* __restrict__ state_hi, const DPass& P,
                                            double2* __restrict__ gen_partials, Body body) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = 1 << P.b;   // 4096 amplitudes: 256 threads x 16 registers per group
  double2* bufs = reinterpret_cast<double2*>(smem_raw);
  const unsigned mbar0 = unsigned(__cvta_generic_to_shared(smem_raw + size_t(3) * T * sizeof(double2)));
  double2* s_gen = reinterpret_cast<double2*>(smem_raw + size_t(3) * T * sizeof(double2) + 32);
  const int tid = threadIdx.x;
  const int grp = tid >> 8, gtid = tid & 255;
  if (P.n_gen)
    for (int i = tid; i < (kPPThreads >> 5) * kMaxGens; i += kPPThreads) s_gen[i] = make_double2(0.0, 0.0);
#ifdef FDEV_SEGPROF
  for (int i = tid; i < 2 * 64 * 2; i += kPPThreads) (&fdev_prof[0][0][0])[i] = 0;
#endif
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(mbar0 + 8u * i, 256u);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  u64 ld_tid = 0;
#pragma unroll
  for (int j = 0; j < kTB; ++j)
    if (j < P.nthr && ((gtid >> j) & 1)) ld_tid |= P.ld_tb[j];
  const int ld_sw = swz(gtid);
  // 16 cp.async per thread (one tile slot per register index), completion -> the buffer's mbarrier
  auto issue_load = [&](u64 b0, int buf) {
    u64 g = b0 | ld_tid;
    const double2* p_lo;
    const double2* p_hi;
    if (TWO) {
      const u64 gl = g & ~P.hi;
      p_hi = state_hi + gl;
      p_lo = (g & P.hi) ? p_hi : state + gl;
    } else {
      p_lo = p_hi = state + g;
    }
    const unsigned sb = unsigned(__cvta_generic_to_shared(bufs + size_t(buf) * T));
#pragma unroll
    for (int i = 0; i < kRegs; ++i) {
      const double2* src = (TWO && ((P.ld_hsel >> i) & 1) ? p_hi : p_lo) + P.ld_off[i];
      const unsigned dst = sb + unsigned(ld_sw ^ P.ld_sm[i]) * 16u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
    }
    mbar_arrive_cp_async(mbar0 + 8u * buf);
  };
  const u64 nt = P.n_tiles;
  const u64 ncta = nt > blockIdx.x ? (nt - 1 - blockIdx.x) / gridDim.x + 1 : 0;   // this CTA's tiles
  u64 base0 = 0;
  {
    u64 m = P.outer;
    for (u64 v = blockIdx.x; m && v; m &= m - 1, v >>= 1)
      if (v & 1) base0 |= m & (~m + 1);
  }
  if (grp == 0) {
    if (ncta > 0) issue_load(base0, 0);
    if (ncta > 2) issue_load(masked_add(base0, P.outer, P.grid_step2), 2);
  } else if (ncta > 1) {
    issue_load(masked_add(base0, P.outer, P.grid_step), 1);
  }
  u64 base = grp ? masked_add(base0, P.outer, P.grid_step) : base0;
  const int segs = 2 * P.n_phases;
  const int offset = P.n_phases | 1;   // odd: B's smem segments line up with A's arithmetic
  double2* acc_warp = s_gen + (tid >> 5) * kMaxGens;
#ifdef FDEV_PP_FREE
  // free-running groups (no step barriers): each group is an independent consumer of the shared
  // three-buffer ring; only the mbarriers order loads and uses
  (void)offset;
  (void)segs;
#else
  if (grp == 1)
    for (int i = 0; i < offset; ++i) step_barrier();
#endif
  int buf = grp;              // local tile j lives in buffer j % 3; its fill number is j / 3
  unsigned fill = 0;
  const u64 periods = (ncta + 1) >> 1;
  for (u64 k = 0; k < periods; ++k) {
    const u64 j = 2 * k + grp;
    if (j < ncta) {
      mbar_wait_parity(mbar0 + 8u * buf, fill & 1u);
      const int cb = buf;
#ifdef FDEV_SEGPROF
      if (gtid == 0) fdev_t = clock64();
#endif
      body(cb << P.b, base, acc_warp, [&]() {
#ifdef FDEV_PP_FREE
        group_barrier();   // every thread of the group has read the buffer (no step barrier did it)
#endif
        if (j + 3 < ncta) issue_load(masked_add(base, P.outer, P.grid_step3), cb);
      });
      base = masked_add(base, P.outer, P.grid_step2);
    } else {
#ifndef FDEV_PP_FREE
      for (int i = 0; i < segs; ++i) step_barrier();
#endif
    }
    // next local tile of this group: j + 2
    buf += 2;
    if (buf >= 3) {
      buf -= 3;
      ++fill;
    }
  }
#ifndef FDEV_PP_FREE
  if (grp == 0)
    for (int i = 0; i < offset; ++i) step_barrier();
#endif
#ifdef FDEV_SEGPROF
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {
    for (int g = 0; g < 2; ++g)
      for (int k = 0; k < segs; ++k)
        printf("SEGPROF n_phases=%d grp=%d seg=%d kind=%c work=%lld wait=%lld\n", P.n_phases, g, k, (k & 1) ? 'C' : 'T',
               fdev_prof[g][k][0], fdev_prof[g][k][1]);
  }
#endif
  if (P.n_gen) {
    __syncthreads();
    for (int g = tid; g < P.n_gen; g += kPPThreads) {
      double2 s = make_double2(0.0, 0.0);
      for (int w = 0; w < (kPPThreads >> 5); ++w) {
        s.x += s_gen[w * kMaxGens + g].x;
        s.y += s_gen[w * kMaxGens + g].y;
      }
      gen_partials[size_t(blockIdx.x) * P.n_gen_total + P.gen_base + g] = s;
    }
  }
}

// phase entry / exit for generated kernels: registers <- tile (offsets s0 ^ W(r)), and the store
// honouring the phase's uniform flip and the thread's dynamic flips
// tile element i (swizzled index): one buffer, or two half buffers selected by index bit b-1
// PP (ping-pong loop): a phase's smem round trip syncs only its group; FDEV_STEP ends a segment
#ifdef FDEV_PP
#define FDEV_PHASE_SYNC() fdev::group_barrier()
#ifdef FDEV_SEGPROF
// diagnostic (SVB200_JIT_SEGPROF=1): thread 0 of each group accumulates, per segment of the tile,
// the cycles it spent working and the cycles it then waited at the step barrier; CTA 0 prints them
#define FDEV_STEP_I(K)                                                  \
  {                                                                     \
    const long long t1_ = clock64();                                    \
    if ((threadIdx.x & 255) == 0) fdev::fdev_prof[threadIdx.x >> 8][K][0] += t1_ - fdev_t;  \
    fdev::step_barrier();                                               \
    const long long t2_ = clock64();                                    \
    if ((threadIdx.x & 255) == 0) fdev::fdev_prof[threadIdx.x >> 8][K][1] += t2_ - t1_;     \
    if ((threadIdx.x & 255) == 0) fdev_t = t2_;                         \
  }
#elif defined(FDEV_PP_FREE)
#define FDEV_STEP_I(K)
#else
#define FDEV_STEP_I(K) fdev::step_barrier()
#endif
#else
// (non-aligned: versioned phases store from different switch cases in different warps)
#define FDEV_PHASE_SYNC() asm volatile("barrier.sync 0;\n" ::: "memory")
#define FDEV_STEP_I(K)
#endif
#ifdef FDEV_SPLIT
#define FDEV_TILE(i) ((((i) & FDEV_HB) ? tile_hi : tile)[(i) & (FDEV_HB - 1)])
#else
#define FDEV_TILE(i) tile[i]
#endif
#define FDEV_PHASE_LOAD(F, W0, W1, W2, W3)                                                                       \
  const int s0 = (F).s_lo[threadIdx.x & 15] ^ (F).s_hi[threadIdx.x >> 4];                                      \
  const u64 pb = base | (F).g_lo[threadIdx.x & 15] | (F).g_hi[threadIdx.x >> 4] | P.gbits;                                \
  double2 a[fdev::kRegs];                                                                                       \
  _Pragma("unroll") for (int r = 0; r < fdev::kRegs; ++r) a[r] =                                                \
      FDEV_TILE(s0 ^ ((r & 1) ? (W0) : 0) ^ ((r & 2) ? (W1) : 0) ^ ((r & 4) ? (W2) : 0) ^ ((r & 8) ? (W3) : 0)); \
  int fthr = 0;                                                                                                 \
  (void)pb;                                                                                                     \
  (void)fthr;
// ... with the thread's slot offset and physical bits given as expressions (generated kernels
// compute them from threadIdx.x with literal masks instead of loading the phase's nibble tables)
#ifdef FDEV_PP
#define FDEV_TILE_OFF tile_off   // PP: the tile buffer enters the slot index (bits 12-13), base fixed
#else
#define FDEV_TILE_OFF 0
#endif
#define FDEV_PHASE_LOAD_X(S0, PB, W0, W1, W2, W3)                                                                \
  const int s0 = (S0) ^ FDEV_TILE_OFF;                                                                         \
  const u64 pb = base | (PB) | P.gbits;                                                                                   \
  double2 a[fdev::kRegs];                                                                                       \
  _Pragma("unroll") for (int r = 0; r < fdev::kRegs; ++r) a[r] =                                                \
      FDEV_TILE(s0 ^ ((r & 1) ? (W0) : 0) ^ ((r & 2) ? (W1) : 0) ^ ((r & 4) ? (W2) : 0) ^ ((r & 8) ? (W3) : 0)); \
  int fthr = 0;                                                                                                 \
  (void)pb;                                                                                                     \
  (void)fthr;
#define FDEV_PHASE_STORE(FLIP, W0, W1, W2, W3)                                                                   \
  {                                                                                                             \
    const int fl = (FLIP) ^ fthr;                                                                               \
    const int sf = s0 ^ ((fl & 1) ? (W0) : 0) ^ ((fl & 2) ? (W1) : 0) ^ ((fl & 4) ? (W2) : 0) ^ ((fl & 8) ? (W3) : 0); \
    _Pragma("unroll") for (int r = 0; r < fdev::kRegs; ++r)                                                     \
      FDEV_TILE(sf ^ ((r & 1) ? (W0) : 0) ^ ((r & 2) ? (W1) : 0) ^ ((r & 4) ? (W2) : 0) ^ ((r & 8) ? (W3) : 0)) = a[r]; \
  }                                                                                                             \
  FDEV_PHASE_SYNC();
// ... when the next phase keeps this phase's warp-bit positions: the exchange stays inside each
// warp (fused_plan.cpp choose_warp_bits), so only the warp synchronises
#define FDEV_PHASE_STORE_WARP(FLIP, W0, W1, W2, W3)                                                                   \
  {                                                                                                             \
    const int fl = (FLIP) ^ fthr;                                                                               \
    const int sf = s0 ^ ((fl & 1) ? (W0) : 0) ^ ((fl & 2) ? (W1) : 0) ^ ((fl & 4) ? (W2) : 0) ^ ((fl & 8) ? (W3) : 0); \
    _Pragma("unroll") for (int r = 0; r < fdev::kRegs; ++r)                                                     \
      FDEV_TILE(sf ^ ((r & 1) ? (W0) : 0) ^ ((r & 2) ? (W1) : 0) ^ ((r & 4) ? (W2) : 0) ^ ((r & 8) ? (W3) : 0)) = a[r]; \
  }                                                                                                             \
  __syncwarp();

// ... when the next phase keeps the top one / two thread bits: each 128-thread half / 64-thread
// quarter of the CTA holds the same amplitudes in both phases, so only that group synchronises
// (named barriers 1-2 for halves, 3-6 for quarters; fused_plan.cpp build_program `fixed`)
#define FDEV_PHASE_STORE_GROUP(FLIP, W0, W1, W2, W3, BAR_ID, BAR_N)                                                   \
  {                                                                                                             \
    const int fl = (FLIP) ^ fthr;                                                                               \
    const int sf = s0 ^ ((fl & 1) ? (W0) : 0) ^ ((fl & 2) ? (W1) : 0) ^ ((fl & 4) ? (W2) : 0) ^ ((fl & 8) ? (W3) : 0); \
    _Pragma("unroll") for (int r = 0; r < fdev::kRegs; ++r)                                                     \
      FDEV_TILE(sf ^ ((r & 1) ? (W0) : 0) ^ ((r & 2) ? (W1) : 0) ^ ((r & 4) ? (W2) : 0) ^ ((r & 8) ? (W3) : 0)) = a[r]; \
  }                                                                                                             \
  asm volatile("barrier.sync %0, %1;\n" ::"r"(BAR_ID), "r"(BAR_N) : "memory");

#ifdef FDEV_PLAIN_STORE
#define FDEV_STG(p, v) (*(p) = (v))
#elif defined(FDEV_EXP_NOMEM)
// timing experiment only (wrong results): no HBM traffic -- the store is kept alive behind a
// condition that is never true at run time
#define FDEV_STG(p, v) \
  if (P.n_tiles == 0) *(p) = (v)
#else
#define FDEV_STG(p, v) __stcs((p), (v))   // streaming: the state is not re-read before eviction
#endif
// last phase of a DIRECT pass: after reading the tile into registers (barrier: every warp has
// read it), start the next tile's load, compute, then store each register to HBM at
// gb | WOFF(r ^ fl) (gb = tile base | the thread's store bits, WOFF(r) = register r's store bits)
#define FDEV_PHASE_STORE_GLOBAL(FLIP, O0, O1, O2, O3)                                                            \
  {                                                                                                             \
    const int fl = (FLIP) ^ fthr;                                                                               \
    const u64 wf = ((fl & 1) ? (O0) : 0ull) | ((fl & 2) ? (O1) : 0ull) | ((fl & 4) ? (O2) : 0ull) |             \
                   ((fl & 8) ? (O3) : 0ull);                                                                    \
    double2* __restrict__ gp = state + (base | st_thr);                                                         \
    _Pragma("unroll") for (int r = 0; r < fdev::kRegs; ++r)                                                     \
      FDEV_STG(gp + ((((r & 1) ? (O0) : 0ull) | ((r & 2) ? (O1) : 0ull) | ((r & 4) ? (O2) : 0ull) |              \
                     ((r & 8) ? (O3) : 0ull)) ^ wf), a[r]);                                                     \
  }

// first phase of a DFL pass: registers straight from global memory (L2-resident after the
// prefetch), a[r] = state[pb | OFF(r)]; s0 is still the thread's shared-memory slot for the store
#define FDEV_PHASE_LOAD_G(S0, PB, O0, O1, O2, O3)                                                                \
  const int s0 = (S0);                                                                                         \
  const u64 pb = base | (PB) | P.gbits;                                                                                   \
  double2 a[fdev::kRegs];                                                                                       \
  _Pragma("unroll") for (int r = 0; r < fdev::kRegs; ++r) {                                                     \
    const u64 g_ = pb | (((r & 1) ? (O0) : 0ull) | ((r & 2) ? (O1) : 0ull) | ((r & 4) ? (O2) : 0ull) |         \
                         ((r & 8) ? (O3) : 0ull));                                                              \
    a[r] = __ldcg(((g_ & P.hi) ? state_hi : state) + (g_ & ~P.hi));                                             \
  }                                                                                                             \
  int fthr = 0;                                                                                                 \
  (void)fthr;

// ... two-array state (adjoint sweep): indices carrying the selector bit P.hi live in state_hi
#define FDEV_PHASE_STORE_GLOBAL2(FLIP, O0, O1, O2, O3)                                                           \
  {                                                                                                             \
    const int fl = (FLIP) ^ fthr;                                                                               \
    const u64 wf = ((fl & 1) ? (O0) : 0ull) | ((fl & 2) ? (O1) : 0ull) | ((fl & 4) ? (O2) : 0ull) |             \
                   ((fl & 8) ? (O3) : 0ull);                                                                    \
    const u64 gb = base | st_thr;                                                                               \
    _Pragma("unroll") for (int r = 0; r < fdev::kRegs; ++r) {                                                   \
      const u64 g = gb | ((((r & 1) ? (O0) : 0ull) | ((r & 2) ? (O1) : 0ull) | ((r & 4) ? (O2) : 0ull) |          \
                          ((r & 8) ? (O3) : 0ull)) ^ wf);                                                        \
      FDEV_STG(((g & P.hi) ? state_hi : state) + (g & ~P.hi), a[r]);                                           \
    }                                                                                                           \
  }

}  // namespace fdev
