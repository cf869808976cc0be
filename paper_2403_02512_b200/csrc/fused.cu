// K7: gate-fusion tile engine (device side + launch).
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
// No op ever moves amplitudes between registers: X gates are register relabelings (a uniform
// flip mask applied by the host planner, plus a per-thread flip mask `fthr` toggled by
// thread-predicated X), honoured by the *D cases and by the phase store.  Every update is
// written in an in-place form.  Both rules keep a[] in fixed registers across the op dispatch;
// violating either costs ~4 register moves per amplitude per op.  Planner: fused_plan.cpp.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "fused.h"
#include "fused_dev.cuh"

namespace fused {
static_assert(fdev::kGenSub == 4, "fused_jit.cpp fdev_gen_sub must match fdev::kGenSub");
namespace {

using fdev::cacc_conj;
using fdev::cfma;
using fdev::cmul;
using fdev::cmul_ip;
using fdev::dense2;
using fdev::DPass;
using fdev::DPhase;
using fdev::gen2;
using fdev::pair1;
using fdev::pair_shear;
using fdev::pairg;
using fdev::parity_phase;
using fdev::phase1;
using fdev::swz;
using fdev::kTB;

__device__ __forceinline__ void diagg(double2 (&a)[kRegs], const FOp& op, const double2* __restrict__ coef,
                                      u64 phys_base, int fthr) {
  // table index = (tconst | sum_k bit_k(r) * w_k) ^ tflip (w_k built without dynamic register indexing)
  int tconst = 0, w0 = 0, w1 = 0, w2 = 0, w3 = 0, tflip = 0;
  const int nt = op.nt;
  for (int j = 0; j < nt; ++j) {
    const int rg = op.treg[j];
    const int bit = 1 << j;
    if (rg == 0xFF)
      tconst |= int((phys_base >> op.tphys[j]) & 1ull) << j;
    else if ((fthr >> rg) & 1)
      tflip |= bit;
    w0 |= (rg == 0) ? bit : 0;
    w1 |= (rg == 1) ? bit : 0;
    w2 |= (rg == 2) ? bit : 0;
    w3 |= (rg == 3) ? bit : 0;
  }
  tconst ^= tflip;
  const int cm = op.cm, cv = op.cv ^ (fthr & op.cm), tab = op.tab;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r & cm) != cv) continue;
    const int t = tconst ^ (((r & 1) ? w0 : 0) | ((r & 2) ? w1 : 0) | ((r & 4) ? w2 : 0) | ((r & 8) ? w3 : 0));
    cmul_ip(a[r], coef[tab + t]);
  }
}

#define PAIR1_CASE(K)                                                                           \
  case CS_PAIR1 + K * 4 + MT_GENERAL: pair1<K, MT_GENERAL>(a, op.c[0], op.c[1], op.c[2], op.c[3]); break; \
  case CS_PAIR1 + K * 4 + MT_REAL: pair1<K, MT_REAL>(a, op.c[0], op.c[1], op.c[2], op.c[3]); break;       \
  case CS_PAIR1 + K * 4 + MT_RXLIKE: pair1<K, MT_RXLIKE>(a, op.c[0], op.c[1], op.c[2], op.c[3]); break;
// PAIR1 on a bit whose per-thread flip is set: logical i0 sits in the bit-1 register -> swap roles
#define PAIR1D_CASE(K)                                                                          \
  case CS_PAIR1D + K * 4 + MT_GENERAL:                                                          \
  case CS_PAIR1D + K * 4 + MT_REAL:                                                             \
  case CS_PAIR1D + K * 4 + MT_RXLIKE: {                                                         \
    const bool sw = (fthr >> K) & 1;                                                            \
    const double2 m0 = sw ? op.c[3] : op.c[0], m1 = sw ? op.c[2] : op.c[1];                     \
    const double2 m2 = sw ? op.c[1] : op.c[2], m3 = sw ? op.c[0] : op.c[3];                     \
    if (op.mtype == MT_REAL) pair1<K, MT_REAL>(a, m0, m1, m2, m3);                              \
    else if (op.mtype == MT_RXLIKE) pair1<K, MT_RXLIKE>(a, m0, m1, m2, m3);                     \
    else pair1<K, MT_GENERAL>(a, m0, m1, m2, m3);                                               \
    break;                                                                                      \
  }
#define PHASE1_CASE(K)                                                 \
  case CS_PHASE1 + K * 2 + 0: phase1<K, 0>(a, op.c[0]); break;         \
  case CS_PHASE1 + K * 2 + 1: phase1<K, 1>(a, op.c[0]); break;         \
  case CS_PHASE1D + K * 2 + 0:                                         \
  case CS_PHASE1D + K * 2 + 1:                                         \
    if (((fthr >> K) & 1) ^ op.v) phase1<K, 1>(a, op.c[0]);            \
    else phase1<K, 0>(a, op.c[0]);                                     \
    break;
#define SHEAR_CASE(K)                                                                       \
  case CS_SHEAR + K * 4 + SH_RY: pair_shear<K, false>(a, op.c[0].x, op.c[0].y); break;         \
  case CS_SHEAR + K * 4 + SH_RX: pair_shear<K, true>(a, op.c[0].x, op.c[0].y); break;          \
  case CS_SHEAR + K * 4 + SH_RYD: {   /* flipped roles: R(-phi) */                            \
    const bool sw = (fthr >> K) & 1;                                                          \
    pair_shear<K, false>(a, sw ? -op.c[0].x : op.c[0].x, sw ? -op.c[0].y : op.c[0].y);       \
    break;                                                                                    \
  }
#define TAN_CASE(K)                                                                   \
  case CS_TAN + K * 4 + 0: fdev::pair_tan<K, false, false>(a, op.c[0].x); break;      \
  case CS_TAN + K * 4 + 1: fdev::pair_tan<K, true, false>(a, op.c[0].x); break;       \
  case CS_TAN + K * 4 + 2: fdev::pair_tan<K, false, true>(a, op.c[0].x); break;       \
  case CS_TAN + K * 4 + 3: fdev::pair_tan<K, true, true>(a, op.c[0].x); break;       \
  case CS_TAND + K * 2 + 0:                                                            \
    if ((fthr >> K) & 1) fdev::pair_tan<K, false, false, true>(a, op.c[0].x);          \
    else fdev::pair_tan<K, false, false>(a, op.c[0].x);                                \
    break;                                                                             \
  case CS_TAND + K * 2 + 1:                                                            \
    if ((fthr >> K) & 1) fdev::pair_tan<K, false, true, true>(a, op.c[0].x);           \
    else fdev::pair_tan<K, false, true>(a, op.c[0].x);                                 \
    break;
#define DENSE2_CASE(PI, K0, K1)                                                         \
  case CS_DENSE2 + PI:                                                                        \
    if (FULL) {                                                                               \
      const int f = ((fthr >> K0) & 1) | (((fthr >> K1) & 1) << 1);                          \
      dense2<K0, K1>(a, coef + op.tab, op.cm, op.cv ^ (fthr & op.cm), f);                     \
    }                                                                                         \
    break;
#define PARITY_CASE(M)                                                                          \
  case CS_PARITY + M:                                                                           \
    parity_phase<M>(a, op.c[0], (__popcll(phys_base & op.xm) + __popc(fthr & M) + op.v) & 1);   \
    break;
#define PAIRG_CASE(XR)                                                                     \
  case CS_PAIRGR + XR - 1: pairg<XR, MT_REAL>(a, op.c[0], op.c[1], op.c[2], op.c[3], op.cm, op.cv ^ (fthr & op.cm)); break; \
  case CS_PAIRG + XR - 1: if (FULL) pairg<XR, MT_GENERAL>(a, op.c[0], op.c[1], op.c[2], op.c[3], op.cm, op.cv ^ (fthr & op.cm)); break;

#define GEN1_CASE(K, T) \
  case CS_GEN1 + K * 4 + T: {                                                                  \
    const bool sw = ((fthr >> K) & 1) != 0;                                                      \
    fdev::gen1<K, T>(a, sw ? op.c[3] : op.c[0], sw ? op.c[2] : op.c[1], sw ? op.c[1] : op.c[2],  \
                     sw ? op.c[0] : op.c[3], op.cm, cv, re, im);                                  \
    break;                                                                                       \
  }
#define GEN2_CASES(PI, K0, K1, TA, TB)                                              \
  case CS_GEN2 + PI * 4 + TA: if (FULL) gen2<K0, K1, TA>(a, M, op.cm, cv, f, re, im); break; \
  case CS_GEN2 + PI * 4 + TB: if (FULL) gen2<K0, K1, TB>(a, M, op.cm, cv, f, re, im); break;

// diagonal generator: sum_r conj(lambda_r) g(bits of r) psi_r, table bits anywhere (like diagg)
template <int T>
__device__ __forceinline__ void gen_diag(const double2 (&a)[kRegs], const FOp& op, int cv, int fthr, u64 phys_base,
                                         const double2* __restrict__ coef, double& re, double& im) {
  int tconst = 0, w0 = 0, w1 = 0, w2 = 0, w3 = 0;
  for (int j = 0; j < op.nt; ++j) {
    const int rg = op.treg[j];
    const int bit = 1 << j;
    if (rg == 0xFF)
      tconst |= int((phys_base >> op.tphys[j]) & 1ull) << j;
    else if ((fthr >> rg) & 1)
      tconst ^= bit;
    w0 |= (rg == 0) ? bit : 0;
    w1 |= (rg == 1) ? bit : 0;
    w2 |= (rg == 2) ? bit : 0;
    w3 |= (rg == 3) ? bit : 0;
  }
  const int cm = op.cm, tab = op.tab;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if ((r >> T) & 1) continue;
    if ((r & cm) != cv) continue;
    const int t = tconst ^ (((r & 1) ? w0 : 0) | ((r & 2) ? w1 : 0) | ((r & 4) ? w2 : 0) | ((r & 8) ? w3 : 0));
    cacc_conj(re, im, a[r | (1 << T)], cmul(coef[tab + t], a[r]));
  }
}

// One generator bra-ket, reduced over the warp into this warp's shared accumulator.  Every lane
// must call it (uniform op; predicate-false lanes contribute zero).
template <bool FULL>
__device__ __forceinline__ void gen_op(const double2 (&a)[kRegs], const int cs, const FOp& op, bool pred, int fthr,
                                       u64 phys_base, const double2* __restrict__ coef,
                                       double2* __restrict__ acc_warp) {
  double re = 0.0, im = 0.0;
  if (pred) {
    const int cv = op.cv ^ (fthr & op.cm);
    const int k0 = op.xr & 15, k1 = op.xr >> 4;
    const int f = ((fthr >> k0) & 1) | (((fthr >> k1) & 1) << 1);
    const double2* M = coef + op.tab;
    switch (cs) {
      GEN1_CASE(0, 1) GEN1_CASE(0, 2) GEN1_CASE(0, 3) GEN1_CASE(1, 0) GEN1_CASE(1, 2) GEN1_CASE(1, 3)
      GEN1_CASE(2, 0) GEN1_CASE(2, 1) GEN1_CASE(2, 3) GEN1_CASE(3, 0) GEN1_CASE(3, 1) GEN1_CASE(3, 2)
      GEN2_CASES(0, 0, 1, 2, 3) GEN2_CASES(1, 0, 2, 1, 3) GEN2_CASES(2, 0, 3, 1, 2)
      GEN2_CASES(3, 1, 2, 0, 3) GEN2_CASES(4, 1, 3, 0, 2) GEN2_CASES(5, 2, 3, 0, 1)
      case CS_GEND + 0: gen_diag<0>(a, op, cv, fthr, phys_base, coef, re, im); break;
      case CS_GEND + 1: gen_diag<1>(a, op, cv, fthr, phys_base, coef, re, im); break;
      case CS_GEND + 2: gen_diag<2>(a, op, cv, fthr, phys_base, coef, re, im); break;
      case CS_GEND + 3: gen_diag<3>(a, op, cv, fthr, phys_base, coef, re, im); break;
      default: break;
    }
  }
  for (int s = 16; s > 0; s >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, s);
    im += __shfl_xor_sync(0xffffffffu, im, s);
  }
  if ((threadIdx.x & 31) == 0) {
    acc_warp[op.slot].x += re;
    acc_warp[op.slot].y += im;
  }
}

// One flat switch on the dense case index.  FULL = false compiles only the common kinds;
// passes that need DIAGG / DENSE2 / complex PAIRG use the FULL kernel.  `op` is in shared memory.
template <bool FULL>
__device__ __forceinline__ void apply_op(double2 (&a)[kRegs], const int cs, const FOp& op,
                                         const double2* __restrict__ coef, u64 phys_base, int& fthr) {
  // every index 0 .. CS_GEN1-1 is an explicit label and the default is unreachable, so the
  // compiler emits one jump table (a compare tree here costs ~5 dependent branches per op)
  switch (cs) {
    PAIR1_CASE(0) PAIR1_CASE(1) PAIR1_CASE(2) PAIR1_CASE(3)
    case CS_PAIR1 + 3: case CS_PAIR1 + 7: case CS_PAIR1 + 11: case CS_PAIR1 + 15: break;
    PAIR1D_CASE(0) PAIR1D_CASE(1) PAIR1D_CASE(2) PAIR1D_CASE(3)
    case CS_PAIR1D + 3: case CS_PAIR1D + 7: case CS_PAIR1D + 11: case CS_PAIR1D + 15: break;
    PHASE1_CASE(0) PHASE1_CASE(1) PHASE1_CASE(2) PHASE1_CASE(3)
    SHEAR_CASE(0) SHEAR_CASE(1) SHEAR_CASE(2) SHEAR_CASE(3)
    case CS_SHEAR + 3: case CS_SHEAR + 7: case CS_SHEAR + 11: case CS_SHEAR + 15: break;
    TAN_CASE(0) TAN_CASE(1) TAN_CASE(2) TAN_CASE(3)
    PARITY_CASE(0) PARITY_CASE(1) PARITY_CASE(2) PARITY_CASE(3) PARITY_CASE(4) PARITY_CASE(5)
    PARITY_CASE(6) PARITY_CASE(7) PARITY_CASE(8) PARITY_CASE(9) PARITY_CASE(10) PARITY_CASE(11)
    PARITY_CASE(12) PARITY_CASE(13) PARITY_CASE(14) PARITY_CASE(15)
    case CS_SCALAR: {
      const double2 d = op.c[0];
#pragma unroll
      for (int r = 0; r < kRegs; ++r) cmul_ip(a[r], d);
      break;
    }
    case CS_XFLIP + 0: fthr ^= 1; break;
    case CS_XFLIP + 1: fthr ^= 2; break;
    case CS_XFLIP + 2: fthr ^= 4; break;
    case CS_XFLIP + 3: fthr ^= 8; break;
    case CS_RDIAG: {
      const unsigned aff = unsigned(op.xm);
#pragma unroll
      for (int r = 0; r < kRegs; ++r)
        if ((aff >> r) & 1) cmul_ip(a[r], coef[op.tab + r]);
      break;
    }
    case CS_RDIAG + 1: break;
    PAIRG_CASE(1) PAIRG_CASE(2) PAIRG_CASE(3) PAIRG_CASE(4) PAIRG_CASE(5) PAIRG_CASE(6) PAIRG_CASE(7)
    PAIRG_CASE(8) PAIRG_CASE(9) PAIRG_CASE(10) PAIRG_CASE(11) PAIRG_CASE(12) PAIRG_CASE(13)
    PAIRG_CASE(14) PAIRG_CASE(15)
    case CS_DIAGG:
      if (FULL) diagg(a, op, coef, phys_base, fthr);
      break;
    DENSE2_CASE(0, 0, 1) DENSE2_CASE(1, 0, 2) DENSE2_CASE(2, 0, 3)
    DENSE2_CASE(3, 1, 2) DENSE2_CASE(4, 1, 3) DENSE2_CASE(5, 2, 3)
    default: __builtin_unreachable();
  }
}

// Launch-time records (DPass / DPhase, fused_dev.cuh): every per-pass / per-phase quantity the
// kernel would otherwise recompute per tile or per phase (swizzled shared-memory offsets, spread
// physical bit masks) is computed once on the host.  Shared-memory offsets compose by XOR because
// swz is GF(2)-linear.

// DB = true : one persistent CTA per SM, two tile buffers, tile t+grid prefetched during tile t.
// DB = false: two CTAs per SM (128 registers), one buffer each; CTAs overlap each other instead.
// TWO = the adjoint sweep's two-array state (psi | lambda selected by bit P.hi).
// Dynamic shared memory: [tile buffer(s)] [phase records] [op records] [generator accumulators].
template <bool FULL, bool DB, bool TWO>
__global__ void __launch_bounds__(256, DB ? 1 : 2) k_fused(double2* __restrict__ state, const DPass P,
                                                            const DPhase* __restrict__ phases,
                                                            const FOp* __restrict__ ops,
                                                            const double2* __restrict__ coef,
                                                            double2* __restrict__ gen_partials,
                                                            double2* __restrict__ state_hi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* tile_mem = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;            // 2^(b-4)
  const int T = 1 << P.b;
  DPhase* s_ph = reinterpret_cast<DPhase*>(smem_raw + size_t(DB ? 2 : 1) * T * sizeof(double2));
  FOp* s_ops = reinterpret_cast<FOp*>(s_ph + P.n_phases);
  double2* s_gen = reinterpret_cast<double2*>(s_ops + P.n_ops);   // per-warp accumulators [warp][kMaxGens]
  {
    // stage the pass's phase and op records (uniform broadcast reads in the phase / op loops)
    const int4* src = reinterpret_cast<const int4*>(phases);
    int4* dst = reinterpret_cast<int4*>(s_ph);
    const int n16p = P.n_phases * int(sizeof(DPhase) / 16);
    for (int i = tid; i < n16p; i += nthreads) dst[i] = src[i];
    src = reinterpret_cast<const int4*>(ops);
    dst = reinterpret_cast<int4*>(s_ops);
    const int n16 = P.n_ops * int(sizeof(FOp) / 16);
    for (int i = tid; i < n16; i += nthreads) dst[i] = src[i];
    if (P.n_gen)
      for (int i = tid; i < (nthreads >> 5) * kMaxGens; i += nthreads) s_gen[i] = make_double2(0.0, 0.0);
    __syncthreads();
  }
  // per-thread constants of the pass
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
  // slot i of a thread whose index bits are g lives at (g | off_i); the bits are disjoint, so the
  // address is a pointer computed once per tile plus a per-slot constant.  Two-array states pick
  // the array by the hi bit (off_i never carries it; hsel says which slots do).
  auto slot_ptrs = [&](u64 g, double2*& p_lo, double2*& p_hi) {
    if (!TWO) {
      p_lo = p_hi = state + g;
      return;
    }
    const u64 gl = g & ~P.hi;
    p_hi = state_hi + gl;
    p_lo = (g & P.hi) ? p_hi : state + gl;
  };
  // global -> shared (cp.async 16 B per amplitude, conflict-free through the swizzle), one group
  auto issue_load = [&](u64 base, double2* dst_buf) {
    double2 *p_lo, *p_hi;
    slot_ptrs(base | ld_tid, p_lo, p_hi);
    const unsigned sb = (unsigned)__cvta_generic_to_shared(dst_buf);
#pragma unroll
    for (int i = 0; i < kRegs; ++i) {
      const double2* src = (TWO && ((P.ld_hsel >> i) & 1) ? p_hi : p_lo) + P.ld_off[i];
      const unsigned dst = sb + unsigned(ld_sw ^ P.ld_sm[i]) * 16u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // first tile's base: deposit blockIdx.x into the outer bits; later tiles: masked add
  u64 base = 0;
  {
    u64 m = P.outer;
    for (u64 v = blockIdx.x; m && v; m &= m - 1, v >>= 1)
      if (v & 1) base |= m & (~m + 1);
  }
  int cur = 0;
  if (DB && blockIdx.x < P.n_tiles) issue_load(base, tile_mem);
  for (u64 t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
    double2* tile = tile_mem + (DB ? cur * T : 0);
    const u64 nbase = ((base | ~P.outer) + P.grid_step) & P.outer;
    if (!DB) {
      __syncthreads();   // previous tile fully stored before the buffer is refilled
      issue_load(base, tile_mem);
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    if (DB && t + gridDim.x < P.n_tiles) issue_load(nbase, tile_mem + (cur ^ 1) * T);
    for (int ph = 0; ph < P.n_phases; ++ph) {
      const DPhase& F = s_ph[ph];
      const int s0 = F.s_lo[tid & 15] ^ F.s_hi[tid >> 4];
      const u64 phys_base = base | F.g_lo[tid & 15] | F.g_hi[tid >> 4] | P.gbits;
      const int W0 = F.W[0], W1 = F.W[1], W2 = F.W[2], W3 = F.W[3];
      double2 a[kRegs];
#pragma unroll
      for (int r = 0; r < kRegs; ++r)
        a[r] = tile[s0 ^ ((r & 1) ? W0 : 0) ^ ((r & 2) ? W1 : 0) ^ ((r & 4) ? W2 : 0) ^ ((r & 8) ? W3 : 0)];
      int fthr = 0;   // per-thread register relabeling from thread-predicated X gates
      const int oe = F.op_end;
      // the next op's header (case, pattern) is loaded one iteration ahead, so the dispatch
      // branches do not wait on shared memory
      int oi = F.op_begin;
      int cs_n = 0;
      u64 pm_n = 0, pv_n = 0;
      if (oi < oe) {
        cs_n = s_ops[oi].cs;
        pm_n = s_ops[oi].pm;
        pv_n = s_ops[oi].pv;
      }
      for (; oi < oe; ++oi) {
        const FOp& op = s_ops[oi];
        const int cs = cs_n & 0xFFFF;
        if (cs_n >> 16) {   // attached thread-predicated X (host: FOp.fk)
          if ((phys_base & op.fpm) == op.fpv) fthr ^= cs_n >> 16;
        }
        const bool pred = (phys_base & pm_n) == pv_n;
        if (oi + 1 < oe) {
          cs_n = s_ops[oi + 1].cs;
          pm_n = s_ops[oi + 1].pm;
          pv_n = s_ops[oi + 1].pv;
        }
        if (cs >= CS_GEN1)
          gen_op<FULL>(a, cs, op, pred, fthr, phys_base, coef, s_gen + (tid >> 5) * kMaxGens);
        else if (pred)
          apply_op<FULL>(a, cs, op, coef, phys_base, fthr);
      }
      {
        // register r holds logical index r ^ flip: store offset = s0 ^ W(r ^ flip) (W linear)
        const int fl = F.flip ^ fthr;
        const int sf = s0 ^ ((fl & 1) ? W0 : 0) ^ ((fl & 2) ? W1 : 0) ^ ((fl & 4) ? W2 : 0) ^ ((fl & 8) ? W3 : 0);
#pragma unroll
        for (int r = 0; r < kRegs; ++r)
          tile[sf ^ ((r & 1) ? W0 : 0) ^ ((r & 2) ? W1 : 0) ^ ((r & 4) ? W2 : 0) ^ ((r & 8) ? W3 : 0)] = a[r];
      }
      __syncthreads();
    }
    // shared -> global with the pass's in-tile relabeling (store slot offsets precomputed; the
    // three lowest tile bits still land on physical bits 0..2, so 8 lanes write 128 contiguous
    // bytes).  Same address set as the load: in-place safe.  (The buffer is refilled only after
    // the next iteration's barrier.)
    {
      double2 *p_lo, *p_hi;
      slot_ptrs(base | st_tid, p_lo, p_hi);
#pragma unroll
      for (int i = 0; i < kRegs; ++i)
        (TWO && ((P.st_hsel >> i) & 1) ? p_hi : p_lo)[P.st_off[i]] = tile[st_sw ^ P.st_sm[i]];
    }
    base = nbase;
    cur ^= 1;
  }
  // generator partials of this CTA: fixed-order sum over warps -> gen_partials[block][slot]
  if (P.n_gen) {
    __syncthreads();
    const int nw = nthreads >> 5;
    for (int g = tid; g < P.n_gen; g += nthreads) {
      double2 s = make_double2(0.0, 0.0);
      for (int w = 0; w < nw; ++w) {
        s.x += s_gen[w * kMaxGens + g].x;
        s.y += s_gen[w * kMaxGens + g].y;
      }
      gen_partials[size_t(blockIdx.x) * P.n_gen_total + P.gen_base + g] = s;
    }
  }
}

inline int swz_host(int s) { return s ^ (((s >> 3) ^ (s >> 6) ^ (s >> 9)) & 7); }

inline u64 deposit_host(u64 v, u64 m) {
  u64 r = 0;
  for (; m && v; m &= m - 1, v >>= 1)
    if (v & 1) r |= m & (~m + 1);
  return r;
}

DPass make_dpass(const FPassArgs& A, int nl, u64 grid) {
  DPass D;
  std::memset(&D, 0, sizeof(D));
  D.n_tiles = A.n_tiles;
  u64 tilemask = 0;
  for (int j = 0; j < A.b; ++j) tilemask |= 1ull << A.tpos[j];
  D.outer = ((nl >= 64) ? ~0ull : ((1ull << nl) - 1)) & ~tilemask;
  D.grid_step = deposit_host(grid, D.outer);
  D.grid_step2 = deposit_host(2 * grid, D.outer);
  D.grid_step3 = deposit_host(3 * grid, D.outer);
  D.hi = A.hi_mask;
  const int nthr = A.nthr, nthreads = 1 << nthr;
  for (int j = 0; j < nthr; ++j) {
    D.ld_tb[j] = 1ull << A.tpos[j];
    D.st_tb[j] = 1ull << A.tpos_st[A.q[j]];
    D.st_tsm[j] = swz_host(1 << A.q[j]);
  }
  for (int i = 0; i < kRegs; ++i) {
    u64 lo = 0, so = 0;
    int ss = 0;
    for (int k = 0; k < kRB; ++k)
      if ((i >> k) & 1) {
        lo |= 1ull << A.tpos[nthr + k];
        so |= 1ull << A.tpos_st[A.q[nthr + k]];
        ss |= 1 << A.q[nthr + k];
      }
    D.ld_off[i] = lo & ~D.hi;
    D.st_off[i] = so & ~D.hi;
    if (lo & D.hi) D.ld_hsel |= 1u << i;
    if (so & D.hi) D.st_hsel |= 1u << i;
    D.ld_sm[i] = swz_host(nthreads * i);
    D.st_sm[i] = swz_host(ss);
  }
  D.b = A.b;
  D.nthr = nthr;
  D.n_phases = A.n_phases;
  D.n_ops = A.op_end - A.op_begin;
  D.n_gen = A.n_gen;
  D.gen_base = A.gen_base;
  D.n_gen_total = A.n_gen_total;
  return D;
}

DPhase make_dphase(const FPhase& F, const FPassArgs& A) {
  DPhase D;
  std::memset(&D, 0, sizeof(D));
  for (int k = 0; k < kRB; ++k) D.W[k] = swz_host(1 << F.reg[k]);
  for (int v = 0; v < 16; ++v)
    for (int j = 0; j < 4; ++j) {
      if ((v >> j) & 1) {
        if (j < A.nthr) {
          D.s_lo[v] ^= swz_host(1 << F.thr[j]);
          D.g_lo[v] |= 1ull << A.tpos[F.thr[j]];
        }
        if (j + 4 < A.nthr) {
          D.s_hi[v] ^= swz_host(1 << F.thr[j + 4]);
          D.g_hi[v] |= 1ull << A.tpos[F.thr[j + 4]];
        }
      }
    }
  D.op_begin = F.op_begin - A.op_begin;
  D.op_end = F.op_end - A.op_begin;
  D.flip = F.flip;
  return D;
}

struct DevProgram {
  void* buf = nullptr;
  size_t cap = 0;
};
std::mutex g_prog_mu;
std::vector<std::pair<sv_handle*, DevProgram>> g_progs;

// Plan cache: the same primitive list on the same layout plans to the same program (repeated
// circuits, and every observable row of a multi-observable adjoint sweep), so the host planner
// runs once.  A few entries per handle, exact comparison of the inputs.
struct PlanKey {
  int nl;
  bool remap, pin;
  std::vector<Prim> prims;
};
bool same_prim(const Prim& a, const Prim& b) {
  if (a.type != b.type || a.fmask != b.fmask || a.fval != b.fval || a.xmask != b.xmask || a.nb != b.nb ||
      a.skip != b.skip || a.slot != b.slot || a.m != b.m)
    return false;
  for (int j = 0; j < a.nb; ++j)
    if (a.pos[j] != b.pos[j]) return false;
  return true;
}
std::mutex g_plan_mu;
std::vector<std::pair<sv_handle*, std::vector<std::pair<PlanKey, std::shared_ptr<Program>>>>> g_plans;

std::shared_ptr<Program> cached_program(sv_handle* h, const std::vector<Prim>& prims, bool remap, bool pin) {
  static const bool off = getenv("SVB200_PLAN_CACHE") && std::string(getenv("SVB200_PLAN_CACHE")) == "0";
  if (off) return std::make_shared<Program>(build_program(h->nl, prims, remap, pin));
  std::lock_guard<std::mutex> lk(g_plan_mu);
  std::vector<std::pair<PlanKey, std::shared_ptr<Program>>>* lst = nullptr;
  for (auto& e : g_plans)
    if (e.first == h) lst = &e.second;
  if (!lst) {
    g_plans.push_back({h, {}});
    lst = &g_plans.back().second;
  }
  for (size_t i = 0; i < lst->size(); ++i) {
    const PlanKey& k = (*lst)[i].first;
    if (k.nl != h->nl || k.remap != remap || k.pin != pin || k.prims.size() != prims.size()) continue;
    bool eq = true;
    for (size_t j = 0; j < prims.size() && eq; ++j) eq = same_prim(k.prims[j], prims[j]);
    if (eq) {
      auto hit = (*lst)[i];
      lst->erase(lst->begin() + i);
      lst->insert(lst->begin(), hit);   // most recent first
      return hit.second;
    }
  }
  auto prog = std::make_shared<Program>(build_program(h->nl, prims, remap, pin));
  lst->insert(lst->begin(), {PlanKey{h->nl, remap, pin, prims}, prog});
  if (lst->size() > 16) lst->pop_back();   // a sharded circuit runs one program per exchange-free batch
  return prog;
}

void* program_buffer(sv_handle* h, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_prog_mu);
  for (auto& e : g_progs)
    if (e.first == h) {
      if (e.second.cap < bytes) {
        stream_sync(h);
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

template <bool FULL, bool DB, bool TWO>
void set_smem_attr(int bytes) {
  CUDA_CHECK(cudaFuncSetAttribute(k_fused<FULL, DB, TWO>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

template <bool FULL, bool DB, bool TWO>
void launch_fused(unsigned grid, int threads, size_t smem, cudaStream_t st, double2* state, const DPass& D,
                  const DPhase* ph, const FOp* op, const double2* cf, double2* gen, double2* state_hi) {
  k_fused<FULL, DB, TWO><<<grid, threads, smem, st>>>(state, D, ph, op, cf, gen, state_hi);
}

}  // namespace
}  // namespace fused

void release_fused(sv_handle* h) {
  using namespace fused;
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    for (size_t i = 0; i < g_plans.size(); ++i)
      if (g_plans[i].first == h) {
        g_plans.erase(g_plans.begin() + i);
        break;
      }
  }
  std::lock_guard<std::mutex> lk(g_prog_mu);
  for (size_t i = 0; i < g_progs.size(); ++i)
    if (g_progs[i].first == h) {
      cudaFree(g_progs[i].second.buf);
      g_progs.erase(g_progs.begin() + i);
      return;
    }
}

std::vector<int> apply_prims_fused(sv_handle* h, const std::vector<double2*>& states, const std::vector<Prim>& prims,
                                   std::vector<std::pair<int, cplx>>* gen_out, double2* state_hi, bool allow_remap,
                                   bool rank_uniform) {
  using namespace fused;
  std::vector<int> identity(h->nl);
  for (int p = 0; p < h->nl; ++p) identity[p] = p;
  // two-array state (state_hi): the top bit selects the array; singles run on each half
  auto run_single = [&](double2* st, const Prim& p0) {
    Prim p = p0;
    if (rank_uniform) {   // the per-primitive kernels see only local bits: resolve for this rank
      resolve_global(p, h->nl, h->rank);
      if (p.skip) return;
    }
    if (!state_hi) {
      launch_prim(h, st, p);
      return;
    }
    h->nl -= 1;
    h->n_local /= 2;
    launch_prim(h, st, p);
    launch_prim(h, state_hi, p);
    h->nl += 1;
    h->n_local *= 2;
  };
  if (h->nl < 5) {
    for (double2* st : states)
      for (const Prim& p : prims) run_single(st, p);
    return identity;
  }
  static const bool remap_env = !(getenv("SVB200_REMAP") && std::string(getenv("SVB200_REMAP")) == "0");
  // Sharded handles: globally-controlled primitives resolve differently per rank (skipped on one,
  // unconditional on another), so each rank plans a different program; an in-tile relabeling
  // would then leave the ranks with different layouts and the next swap would exchange
  // mismatched halves.  Every rank must keep the same layout: no relabeling when world > 1.
  // (rank_uniform programs are identical on every rank, so they may relabel)
  const bool remap = remap_env && (h->world == 1 || rank_uniform) && allow_remap;
  const u64 gbits = rank_uniform ? (u64(h->rank) << h->nl) : 0ull;
  host_prof_mark("fused: enter");
  const std::shared_ptr<Program> prog_ptr = cached_program(h, prims, remap, state_hi != nullptr);
  host_prof_mark("fused: program ready");
  Program& prog = *prog_ptr;
  if (state_hi)
    for (auto& A : prog.passes) A.hi_mask = 1ull << (h->nl - 1);
  if (prog.passes.empty()) {
    for (double2* st : states)
      for (const Prim& p : prog.singles) run_single(st, p);
    return identity;
  }
  // kernel attributes are per device: one-time setup for each device this process uses
  static std::once_flag once_dev[64];
  static int sms_dev[64];
  static bool db = false;
  if (h->device < 0 || h->device >= 64) sv_fail(SV_ERR_DEVICE, "device ordinal out of range");
  std::call_once(once_dev[h->device], [&]() {
    // the attribute is an upper bound; a launch's real footprint sets its occupancy
    const int tile = int((size_t(1) << kMaxB) * sizeof(double2));
    const int recs = 200 * 1024 - 2 * tile;
    set_smem_attr<true, true, false>(2 * tile + recs);
    set_smem_attr<false, true, false>(2 * tile + recs);
    set_smem_attr<true, false, false>(tile + recs);
    set_smem_attr<false, false, false>(tile + recs);
    set_smem_attr<true, true, true>(2 * tile + recs);
    set_smem_attr<false, true, true>(2 * tile + recs);
    set_smem_attr<true, false, true>(tile + recs);
    set_smem_attr<false, false, true>(tile + recs);
    CUDA_CHECK(cudaDeviceGetAttribute(&sms_dev[h->device], cudaDevAttrMultiProcessorCount, h->device));
    // default: single buffer, 2 CTAs/SM (measured faster: 16 warps hide the op-loop latency
    // better than 8 warps with a prefetched tile); "db" selects the double-buffered variant
    const char* mode = getenv("SVB200_FUSED_MODE");
    db = mode && std::string(mode) == "db";
  });
  const int b = prog.passes[0].b;
  const bool jdb = !db && jit_db();   // generated kernels in their double-buffered 1-CTA/SM form
  const u64 grid = std::min<u64>(prog.passes[0].n_tiles, u64(sms_dev[h->device]) * ((db || jdb) ? 1 : (jit_enabled() ? jit_ctas_per_sm() : 2)) *
                                                    (u64(1) << (kMaxB - std::min(kMaxB, prog.passes[0].b))));   // persistent grid

  // generated ping-pong passes: one CTA per SM (their generator partials use the same [CTA][slot]
  // layout, so the partial buffer is sized for the larger of the two grids)
  const u64 pp_grid = std::min<u64>(grid, u64(sms_dev[h->device]));
  // launch records + upload phases | ops | coef in one copy (the buffer is only reused after a sync)
  std::vector<DPhase> dph(prog.phases.size());
  for (const FPassArgs& A : prog.passes)
    for (int ph = 0; ph < A.n_phases; ++ph) dph[A.phase_begin + ph] = make_dphase(prog.phases[A.phase_begin + ph], A);
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t b_ph = dph.size() * sizeof(DPhase);
  const size_t b_op = prog.ops.size() * sizeof(FOp);
  const size_t b_cf = prog.coef.size() * sizeof(double2);
  const bool two = state_hi != nullptr;
  if (!db) jit_prepare(prog, two);   // per-pass compiled kernels (cached by structure)
  const size_t b_jt = prog.jit_tabs.size() * sizeof(double2);
  const size_t total = align(b_ph) + align(b_op) + align(b_cf) + align(b_jt);
  std::vector<char> host(total);
  std::memcpy(host.data(), dph.data(), b_ph);
  std::memcpy(host.data() + align(b_ph), prog.ops.data(), b_op);
  {
    FOp* dev_ops = reinterpret_cast<FOp*>(host.data() + align(b_ph));
    for (size_t i = 0; i < prog.ops.size(); ++i) dev_ops[i].cs |= dev_ops[i].fk << 16;   // one prefetched word
  }
  std::memcpy(host.data() + align(b_ph) + align(b_op), prog.coef.data(), b_cf);
  if (b_jt) std::memcpy(host.data() + align(b_ph) + align(b_op) + align(b_cf), prog.jit_tabs.data(), b_jt);
  host_prof_mark("fused: records built");
  stream_sync(h);   // previous program may still be in use
  host_prof_mark("fused: prev program synced");
  char* dbuf = (char*)program_buffer(h, total);
  CUDA_CHECK(cudaMemcpyAsync(dbuf, host.data(), total, cudaMemcpyHostToDevice, h->stream));
  const DPhase* d_ph = (const DPhase*)dbuf;
  const FOp* d_op = (const FOp*)(dbuf + align(b_ph));
  const double2* d_cf = (const double2*)(dbuf + align(b_ph) + align(b_op));
  const double2* d_jt = (const double2*)(dbuf + align(b_ph) + align(b_op) + align(b_cf));

  const int n_gen = int(prog.gen_slot_of.size());
  double2* d_gen = nullptr;
  if (n_gen) {
    if (!gen_out || states.size() != 1) sv_fail(SV_ERR_DEVICE, "internal: generator ops need one combined state");
    CUDA_CHECK(cudaMallocAsync(&d_gen, grid * n_gen * sizeof(double2), h->stream));
    CUDA_CHECK(cudaMemsetAsync(d_gen, 0, grid * n_gen * sizeof(double2), h->stream));
  }
  for (double2* state : states) {
    for (const Step& s : prog.steps) {
      if (!s.fused) {
        if (prog.singles[s.index].type >= PRIM_GEN) sv_fail(SV_ERR_DEVICE, "internal: unfusable generator");
        run_single(state, prog.singles[s.index]);
        continue;
      }
      const FPassArgs& A = prog.passes[s.index];
      DPass D = make_dpass(A, h->nl, grid);
      D.gbits = gbits;
      const bool full = prog.full[s.index];
      const int threads = 1 << (A.b - kRB);
      const size_t smem = (db ? 2 : 1) * (size_t(1) << b) * sizeof(double2) + size_t(D.n_phases) * sizeof(DPhase) +
                          size_t(D.n_ops) * sizeof(FOp) + (A.n_gen ? size_t(threads / 32) * kMaxGens * sizeof(double2) : 0);
      const DPhase* ph = d_ph + A.phase_begin;
      const FOp* op = d_op + A.op_begin;
      const double bytes = 32.0 * double(h->n_local);
      cudaEvent_t ev[2];
      stat_begin(h, KC_FUSED, bytes, ev);
      const unsigned g = unsigned(grid);
      cudaStream_t st = h->stream;
      const JitPass* jp = (!db && s.index < int(prog.jit.size()) && prog.jit[s.index].kernel) ? &prog.jit[s.index] : nullptr;
      if (jp && jp->pp) {
        // ping-pong loop: one 512-thread CTA per SM, three tile buffers (fused_dev.cuh run_pass_pp)
        DPass Dp = make_dpass(A, h->nl, pp_grid);
        Dp.gbits = gbits;
        const size_t psmem = fdev::pp_smem_bytes(A.b, A.n_gen > 0);
        jit_launch(*jp, h->device, unsigned(pp_grid), fdev::kPPThreads, psmem, st, state, state_hi, &Dp, ph, d_jt, d_gen);
      } else if (jp) {
        // generated kernel of this pass: [tile] [phase records] [generator accumulators]
        const size_t jsmem = (jdb ? 4 : (jp->split ? 3 : 2)) * (size_t(1) << (b - 1)) * sizeof(double2) + size_t(D.n_phases) * sizeof(DPhase) +
                             (A.n_gen ? size_t(threads / 32) * kMaxGens * fdev::kGenSub * sizeof(double2) : 0);
        jit_launch(*jp, h->device, g, threads, jsmem, st, state, state_hi, &D, ph, d_jt, d_gen);
      } else if (two) {
        if (db && full) launch_fused<true, true, true>(g, threads, smem, st, state, D, ph, op, d_cf, d_gen, state_hi);
        else if (db) launch_fused<false, true, true>(g, threads, smem, st, state, D, ph, op, d_cf, d_gen, state_hi);
        else if (full) launch_fused<true, false, true>(g, threads, smem, st, state, D, ph, op, d_cf, d_gen, state_hi);
        else launch_fused<false, false, true>(g, threads, smem, st, state, D, ph, op, d_cf, d_gen, state_hi);
      } else {
        if (db && full) launch_fused<true, true, false>(g, threads, smem, st, state, D, ph, op, d_cf, d_gen, state_hi);
        else if (db) launch_fused<false, true, false>(g, threads, smem, st, state, D, ph, op, d_cf, d_gen, state_hi);
        else if (full) launch_fused<true, false, false>(g, threads, smem, st, state, D, ph, op, d_cf, d_gen, state_hi);
        else launch_fused<false, false, false>(g, threads, smem, st, state, D, ph, op, d_cf, d_gen, state_hi);
      }
      stat_end(h, KC_FUSED, bytes, ev);
      CUDA_CHECK(cudaGetLastError());
    }
  }
  host_prof_mark("fused: launched");
  if (n_gen) {
    // fixed-order reduction over the persistent CTAs -> one complex per program slot
    ensure_results(h, size_t(2) * n_gen);
    sum_partials(h, reinterpret_cast<const double*>(d_gen), int(grid), 2 * n_gen, h->d_results);
    std::vector<double> z(size_t(2) * n_gen);
    CUDA_CHECK(cudaFreeAsync(d_gen, h->stream));
    d2h(h, z.data(), h->d_results, z.size() * sizeof(double));
    gen_out->clear();
    for (int s = 0; s < n_gen; ++s)   // gen_scale: scaled rotations ahead of the bra-ket in its pass
      gen_out->push_back({prog.gen_slot_of[s], prog.gen_scale[s] * cplx(z[2 * s], z[2 * s + 1])});
  }
  return prog.perm;
}
