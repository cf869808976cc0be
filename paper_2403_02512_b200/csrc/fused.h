// K7 fusion engine: program format shared by the host planner (fused_plan.cpp) and the
// sm_100a tile kernel (fused.cu).
#pragma once

#include <vector>

#include "fused_jit.h"
#include "sv_internal.h"

namespace fused {

constexpr int kMaxB = 12;        // tile bits (2^12 amplitudes = 64 KiB)
constexpr int kRB = 4;           // register bits per thread (16 amplitudes)
constexpr int kRegs = 1 << kRB;
constexpr int kMaxSmemOps = 320; // op records staged in shared memory per pass

// op kinds; the *1 kinds are fast paths whose register predicate is compile-time
enum FKind : uint8_t {
  FK_PAIR1 = 0,   // 2x2 on register bit k, no register-side control
  FK_PAIRG = 1,   // 2x2 on register xmask xr with register pattern (cm, cv)
  FK_PHASE1 = 2,  // a *= d where register bit k == v (no other register-side pattern)
  FK_SCALAR = 3,  // a *= d on all 16 amplitudes (pattern only on thread / outer bits)
  FK_DIAGG = 4,   // table lookup diagonal, general
  FK_DENSE2 = 5,  // 4x4 on register bits (k0 < k1) = xr & 15, xr >> 4
  FK_PARITY = 6,  // diagonal phase on the parity of its bits (IsingZZ, Z-string phases)
};
enum MType : uint8_t { MT_GENERAL = 0, MT_REAL = 1, MT_RXLIKE = 2, MT_X = 3 };

struct __align__(16) FOp {
  u64 pm, pv;            // fixed pattern on non-register bits (tested on the thread's physical base)
  u64 xm;                // PARITY: non-register bits whose parity (on the physical base) enters the phase
  u64 fpm, fpv;          // attached thread-predicated X (applied before the op): pattern ...
  uint8_t kind, mtype;
  uint8_t xr;            // PAIRG: register-space xmask; DENSE2: k0 | (k1 << 4)
  uint8_t cm, cv;        // register-space pattern (PAIRG includes i0's pattern on xr)
  uint8_t nt;            // DIAGG: table bits
  uint8_t k, v;          // PAIR1 / PHASE1: register bit and value
  uint8_t treg[6];       // DIAGG: register bit of table bit j, or 0xFF
  uint8_t tphys[6];      // DIAGG: physical position of table bit j when not a register bit
  int tab;               // offset into the coefficient array (DIAGG / DENSE2)
  int cs;                // dense dispatch case (CS_* below)
  int slot;              // GEN: accumulator slot within the pass
  int fk;                // ... and register-flip mask (0: none).  The device copy carries fk in cs >> 16
  double2 c[4];          // inline coefficients (PAIR1 / PAIRG: m00 m01 m10 m11; PHASE1 / SCALAR: d)
};
// Dense dispatch cases.  No case moves amplitudes between registers (data-moving swaps
// poison register allocation for the whole op loop): X gates become register relabelings --
// uniform ones are applied by the host (FPhase.flip), thread-predicated ones toggle a
// per-thread flip mask (CS_XFLIP) that the *D cases and the phase store honour.
constexpr int CS_PAIR1 = 0;      // + k*4 + mtype (mtype != MT_X)            (0..15)
constexpr int CS_PHASE1 = 16;    // + k*2 + v                                (16..23)
constexpr int CS_SCALAR = 24;
constexpr int CS_PAIRGR = 25;    // + xr - 1: real-matrix PAIRG (controlled X) (25..39)
constexpr int CS_PAIRG = 40;     // + xr - 1: complex PAIRG                  (40..54)
constexpr int CS_DIAGG = 55;
constexpr int CS_DENSE2 = 56;    // + pair index 0..5                        (56..61)
constexpr int CS_XFLIP = 62;     // + k: thread-predicated X on register bit k (62..65)
constexpr int CS_PAIR1D = 66;    // + k*4 + mtype: PAIR1 on a dynamically flipped bit (66..81)
constexpr int CS_PHASE1D = 82;   // + k*2 + v: PHASE1 on a dynamically flipped bit   (82..89)
// unconditioned rotations as three in-place shears per real pair (6 FMAs instead of 4 DMUL +
// 4 DFMA); c[0] = (t, s) = (-tan(phi/2), sin(phi)), |phi| <= pi/2
constexpr int CS_SHEAR = 90;     // + k*4 + {0: RY-type, 1: RX-type, 2: RY-type on a flipped bit} (90..105)
constexpr int SH_RY = 0, SH_RX = 1, SH_RYD = 2;
// parity phase (IsingZZ / ZZ..Z-string phases): a *= d where parity(register bits M of r) ^
// parity(physical base & xm) ^ parity(fthr & M) ^ v == 1
constexpr int CS_PARITY = 106;   // + M (register mask, 0..15)                        (106..121)
// unconditioned rotations in scaled form, 2 FMAs per real pair (runtime pass compiler only): the op
// applies R(phi)/c (TAN: tau = tan(phi), |phi| <= pi/4) or R(phi)/s (COT: kappa = cot(phi)); the
// pass's product of the dropped factors is absorbed once per pass (fused_plan.cpp absorb_pass_scale).
// c[0] = (tau or kappa, dropped factor), c[1].x = cos(phi), c[2] = (sin(phi), RX-type ? 1 : 0)
constexpr double kTanBand = 2.5;  // hysteresis: a remembered form is kept while |tau| or |kappa| <= 2.5
constexpr int CS_TAN = 122;      // + k*4 + {0: RY-type TAN, 1: RX-type TAN, 2: RY-type COT, 3: RX-type COT} (122..137)
// ... RY type on a register bit that may carry a per-thread flip (the flipped threads apply R(-phi))
constexpr int CS_TAND = 138;     // + k*2 + {0: TAN, 1: COT}                                 (138..145)
// register diagonal: a[r] *= coef[tab + r] for the registers r in the 16-bit mask xm -- a group of
// PHASE1 ops of one phase multiplied together (fused_plan.cpp group_phase_diagonals)
constexpr int CS_RDIAG = 146;    // (147 unused)
// adjoint bra-kets (psi and lambda share the tile; t = register bit selecting lambda)
constexpr int CS_GEN1 = 148;     // + k*4 + t: 2x2 generator on register bit k        (148..163)
constexpr int CS_GEN2 = 164;     // + pair*4 + t: 4x4 generator on register bits pair (164..187)
constexpr int CS_GEND = 188;     // + t: diagonal generator (table on any bits; only t in registers) (188..191)
constexpr int kMaxGens = 64;     // generator slots per pass (per-warp shared-memory accumulators)
static_assert(sizeof(FOp) == 144, "FOp layout");

struct FPhase {
  uint8_t reg[kRB];      // tile positions held in registers
  uint8_t flip;          // absorbed X gates: logical register index j is stored in register j ^ flip
  uint8_t thr[kMaxB];    // tile positions of thread-index bits (b - 4 of them; lanes 0..2 first)
  int op_begin, op_end;
};

struct FPassArgs {
  int b;                 // tile bits
  int nthr;              // b - kRB
  unsigned char tpos[kMaxB];     // physical positions of tile bits at load (ascending)
  unsigned char tpos_st[kMaxB];  // physical position of tile bit j at store (a permutation of tpos:
                                 // the pass relabels qubits inside its tile for free)
  unsigned char q[kMaxB];        // store-loop order of tile bits (q[0..2] land on physical bits 0..2)
  u64 n_tiles;
  int phase_begin, n_phases;
  int op_begin, op_end;  // op records of the whole pass (contiguous)
  u64 hi_mask;           // two-array state: indices with this bit live in the second array
  int n_gen;             // GEN slots used by this pass
  int gen_base;          // first global result slot of this pass
  int n_gen_total;       // result slots of the whole program (row length of the partials)
  int direct = 0;        // last phase's lane bits = the tile bits stored to physical 0..2
};

// One step of a planned program: a fused pass (index into Program::passes) or a single
// unfusable primitive (index into Program::singles), in execution order.
struct Step {
  bool fused = false;
  int index = -1;
};

struct Program {
  std::vector<Step> steps;
  std::vector<FPassArgs> passes;
  std::vector<char> full;          // pass needs the FULL kernel variant
  std::vector<Prim> singles;       // unfusable prims, already in the layout at their step
  std::vector<FPhase> phases;
  std::vector<FOp> ops;
  std::vector<double2> coef;
  std::vector<int> perm;           // final layout: physical position p now holds what was at p before...
                                   // ... i.e. the qubit at p moved to perm[p]
  std::vector<int> gen_slot_of;    // program result slot -> Prim::slot (the caller's Jacobian slot)
  std::vector<double> gen_scale;   // ... and the factor its bra-ket is multiplied by (scaled rotations
                                   // before it in its pass leave psi and lambda scaled: 1 / f^2)
  int64_t n_prims_in = 0, n_prims_merged = 0;
  int owed_neg = 0;                // global -1 owed by rotations emitted as -R(phi') (planner only)
  std::vector<uint8_t> tan_forms;  // planner only: COT (1) / TAN (0) of each scaled rotation, in order
  std::vector<uint8_t> tan_hint;   // ... as the previous plan of the same structure chose them
  // runtime pass compiler (fused_jit.cpp): per-pass kernels and their parameter blocks
  bool jit_ready = false, jit_two = false;
  std::vector<JitPass> jit;
  std::vector<double2> jit_tabs;   // coefficient tables of the generated kernels, all passes
};

// remap = let passes relabel qubits inside their tile (moves upcoming qubits onto the low bits)
// pin_top = never relabel bit nl-1 (the psi/lambda selector of the adjoint sweep's two arrays)
int tile_bits();   // tile bits of a fused pass (default kMaxB)
Program build_program(int nl, const std::vector<Prim>& prims, bool remap, bool pin_top = false);
// flat int64/double serialisation of a program (tests/fused_emulator.py re-executes it on the CPU)
void serialize_program(const Program& prog, int nl, std::vector<int64_t>& ints, std::vector<double>& dbls);

}  // namespace fused
