// Internal types shared by the host runtime and the sm_100a kernels of libsvb200.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <complex>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/svb200.h"

// SVB200_HOST_PROF=1: host-side timeline of the adjoint / fused-program paths on stderr
// (diagnostics: wall time since the previous mark, and whether the stream was idle)
void host_prof_mark(const char* what);

typedef unsigned long long u64;
using cplx = std::complex<double>;

// ---------------------------------------------------------------------------
// errors: thrown inside the library, converted to status codes at the C-ABI
// ---------------------------------------------------------------------------
struct SvError {
  int status;
  std::string msg;
};
[[noreturn]] void sv_fail(int status, const std::string& msg);
void sv_cuda_check(cudaError_t e, const char* what);
void sv_nccl_check(ncclResult_t r, const char* what);
#define CUDA_CHECK(x) sv_cuda_check((x), #x)
#define NCCL_CHECK(x) sv_nccl_check((x), #x)

// ---------------------------------------------------------------------------
// Primitive ops: what every gate lowers to, in PHYSICAL local bit positions.
//   PAIR : 2x2 update of (a[i0], a[i0 ^ xmask]) for every i0 with (i0 & fmask) == fval.
//          fmask contains the controls and the xmask bits (i0's pattern on them).
//          Covers Alg. 1 / Alg. 2 (state.py:154-226), SWAP, IsingXY, Single/DoubleExcitation.
//   DIAG : a[i] *= table[bits of i at pos[0..nb)] for every i with (i & fmask) == fval.
//   DENSE: 2^k x 2^k matvec on target bits pos[0..k) (ascending; matrix index bit j <-> pos[j])
//          for every group base with (base & fmask) == fval (fmask includes the targets).
// ---------------------------------------------------------------------------
//   GEN  : adjoint bra-ket <lambda| G |psi> (does not modify the state).  psi and lambda live in
//          one array: lambda is the half whose bit `xmask` (one bit) is set.  G is a 2^nb x 2^nb
//          matrix on pos[] (targets, fmask includes them with value 0 plus the controls);
//          the result accumulates into Jacobian slot `slot`.
//   GEND : GEN with a diagonal G given as a table over pos[] (like DIAG; pos need not be local to
//          a register), restricted by fmask/fval.
enum PrimType { PRIM_PAIR = 0, PRIM_DIAG = 1, PRIM_DENSE = 2, PRIM_GEN = 3, PRIM_GEND = 4 };

struct Prim {
  int type = PRIM_PAIR;
  u64 fmask = 0, fval = 0;
  u64 xmask = 0;          // PAIR: partner mask; GEN: the psi/lambda bit
  int nb = 0;             // DIAG / DENSE / GEN: number of bits in pos
  int pos[16] = {0};      // ascending physical positions
  std::vector<cplx> m;    // PAIR: 4 (row-major), DIAG: 2^nb, DENSE / GEN: 4^nb (row-major)
  bool skip = false;      // resolved to identity on this shard
  int slot = -1;          // GEN: result slot
};

// Generator record of a single-parameter piece for the adjoint sweep:
// <lambda| G |psi> with G a DENSE-style small matrix on pos[] restricted by fmask/fval.
struct GenPrim {
  Prim g;                 // type PRIM_DENSE (k = nb) with m = generator matrix
  double prefactor = 0;   // gate(theta) = exp(i prefactor theta G)
  int column = -1;        // Jacobian column
};

// A lowered op: one or more prims (Rot -> 3 pieces) plus adjoint bookkeeping.
struct Piece {
  Prim fwd;               // the unitary U as a prim
  Prim inv;               // U^dagger
  bool has_gen = false;
  GenPrim gen;
};

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------
enum KernelClass {
  KC_PAIR = 0, KC_DIAG, KC_DENSE, KC_FUSED, KC_REDUCE, KC_APPLY_OBS, KC_BRAKET,
  KC_PROBS, KC_INIT, KC_SWAP, KC_COUNT
};
extern const char* kKernelClassNames[KC_COUNT];

// Recording mode (host-only planning of a sharded run, used by sv_plan_sharded): instead of
// launching, the executors append what they would do.
enum RecKind { REC_PRIM = 0, REC_GSWAP = 1, REC_XSWAP = 2 };
struct RecStep {
  int kind;
  Prim p;      // REC_PRIM
  int G = -1;  // REC_GSWAP: global physical position exchanged with the top local bit
  std::vector<int> Gs, ps;   // REC_XSWAP: global positions Gs[i] exchanged with local positions ps[i]
};

struct PendingTiming {
  int cls;
  double bytes;
  cudaEvent_t start, stop;
};

struct sv_handle {
  int n = 0;          // total qubits
  int nl = 0;         // local qubits
  int rank = 0, world = 1, g = 0;
  int device = 0;
  int prec = 64;                // 64: complex128 (double2); 32: complex64 (float2, state.py:20 "f32")
  cudaStream_t stream = nullptr;
  double2* state = nullptr;     // 2^nl amplitudes (float2 storage when prec == 32)
  u64 n_local = 0;
  // logical bit offset o = n-1-q  ->  physical position (>= nl: global/rank bit)
  std::vector<int> phys;
  ncclComm_t comm = nullptr;
  double2* staging = nullptr;
  u64 staging_amps = 0;
  cudaStream_t copy_stream = nullptr;          // swap pipeline: staging -> state copies
  cudaEvent_t ev_recv[2] = {nullptr, nullptr};
  cudaEvent_t ev_copy[2] = {nullptr, nullptr};
  // peer-memory swaps (dist.cpp): each swapped buffer's partner copies mapped through CUDA
  // IPC, per global bit j (partner rank ^ 2^j); registered collectively on first swap
  struct PeerMap {
    double2* local;
    double2* by_rank[8];   // every other rank's copy (world <= 8), nullptr for this rank
  };
  bool p2p = false;
  std::vector<PeerMap> peers;
  int* d_barrier = nullptr;
  // reduction scratch
  double* d_partials = nullptr;
  size_t partials_cap = 0;      // doubles
  double* d_results = nullptr;  // small result vector
  size_t results_cap = 0;
  double* h_pinned = nullptr;
  size_t h_pinned_cap = 0;
  // ring of upload buffers for small per-launch tables (kernels.cu scratch_upload); owned by the
  // handle, so concurrent handles on other threads never touch it
  struct ScratchBuf {
    void* ptr = nullptr;
    size_t cap = 0;
  };
  ScratchBuf scratch[64];
  int scratch_slot = 0;
  std::vector<double2*> aux;    // lambda states for the adjoint sweep
  double2* adj_lam = nullptr;   // fused adjoint: lambda, kept across calls
  double2* adj_saved = nullptr; // fused adjoint: saved final psi (several observables)
  std::mutex mu;
  bool recording = false;       // host-only planning handle (no device memory)
  bool zero_state = false;      // the state is exactly |0...0> in the canonical layout (create / reset)
  std::vector<RecStep> rec;
  // stats
  int64_t launches = 0;
  bool profiling = false;
  std::vector<PendingTiming> pending;
  std::vector<cudaEvent_t> event_pool;
  double kc_launches[KC_COUNT] = {0};
  double kc_ms[KC_COUNT] = {0};
  double kc_bytes[KC_COUNT] = {0};
};

// ---------------------------------------------------------------------------
// host-side modules
// ---------------------------------------------------------------------------
// gates.cpp
void validate_op(const sv_op& op, int n);
// phys: logical offset (n-1-q) -> physical position (>= nl: shard-index bit); nullptr = identity
std::vector<Piece> lower_op(const sv_op& op, int n, int& next_column, bool need_gen, const int* phys);
Prim make_dense_prim(const std::vector<int>& wires, const std::vector<cplx>& m, int n,
                     const std::vector<int>& ctrls, const std::vector<int>& cvals, const int* phys);
void resolve_global(Prim& p, int nl, int rank);
void fold_diag_phases(std::vector<Prim>& prims);
std::vector<cplx> gate_matrix(int kind, const double* params, int n_wires, const double* matrix);
void classify_prim(Prim& p);   // DENSE -> DIAG / PAIR specialisations when exact
Prim adjoint_prim(const Prim& p);


// api.cpp: wait for the handle's stream (sharded handles: NCCL watchdog + ncclCommAbort)
void stream_sync(sv_handle* h);
// small device->host copy (pinned bounce buffer, then stream_sync)
void d2h(sv_handle* h, void* host, const void* dev, size_t bytes);
// dist.cpp: abort the communicator after a failure (peers then fail their own waits, not hang)
void dist_abort(sv_handle* h);

// kernels.cu
double prim_bytes(const sv_handle* h, const Prim& p);
void release_scratch(sv_handle* h);
void launch_prim(sv_handle* h, double2* state, const Prim& p);
void launch_init_zero(sv_handle* h, double2* state, u64 basis_local, bool set_one);
void launch_copy(sv_handle* h, double2* dst, const double2* src, u64 n);
// element-wise exchange a[i] <-> b[i], i < n (b may be a peer GPU's memory mapped over NVLink)
void launch_exchange(sv_handle* h, double2* a, double2* b, u64 n);
// multi-bit exchange over peer memory (dist.cpp exchange_bits): for every partner c < nc with
// peer_by_c[c] != nullptr, swap a[base | own[c] | vdep[c]] with peer_by_c[c][base | own[c] | gdep];
// base = deposit(t, zero bits at split_fmask) for t < count
void launch_exchange_multi(sv_handle* h, double2* a, double2* const* peer_by_c, const u64* vdep, const u64* own, u64 gdep,
                           int nc, u64 split_fmask, u64 count);
// buf[t] = a[deposit(t_begin + t, zeros at victim_mask) | vdep] for t < n (unpack: the reverse)
void launch_pack_sel(sv_handle* h, double2* a, double2* buf, u64 victim_mask, u64 vdep, u64 t_begin, u64 n, bool unpack);
double reduce_norm2(sv_handle* h, const double2* state);
// per-term Pauli expectation: terms sharing an x-mask; returns sum_t Re(cc_t * <P_t>) (local part)
struct PauliTerm {
  u64 zmask;
  cplx cc;   // coefficient * i^{nY} * global-sign
};
// K14: state = scale * exp(i f), f(i) = sum_t Re(cc_t) (-1)^{pc(i & zmask_t)} (one write-only pass)
void init_uniform_phase(sv_handle* h, double2* state, const std::vector<PauliTerm>& terms, double scale);
int pauli_groups_expval_batched(sv_handle* h, const double2* psi,
                                std::vector<std::pair<u64, std::vector<PauliTerm>>> groups, double* d_out);
void pauli_group_expval_async(sv_handle* h, const double2* state, u64 xmask, const std::vector<PauliTerm>& terms,
                              double* d_out);
void pauli_group_apply(sv_handle* h, const double2* psi, double2* lam, u64 xmask,
                       const std::vector<PauliTerm>& terms, bool accumulate);
// lam = sum over x-groups (batched: psi read once per group, lam written once per batch of 16)
void pauli_groups_apply(sv_handle* h, const double2* psi, double2* lam,
                        const std::vector<std::pair<u64, std::vector<PauliTerm>>>& groups);
double reduce_dot_re(sv_handle* h, const double2* a, const double2* b);   // Re <a|b> (local part)
// CSR observable on a single-GPU state: <psi|A|psi> (lam == nullptr) or lam = A psi
double csr_apply_or_expval(sv_handle* h, const sv_obs& o, const double2* psi, double2* lam);
// <bra| P_f (G) |ket> complex, written to d_out[0..1]
void braket_prim_async(sv_handle* h, const double2* bra, const double2* ket, const Prim& g, double* d_out);
void probs_async(sv_handle* h, const double2* state, const std::vector<int>& pos_msb_first, double* d_out);
void sum_partials(sv_handle* h, const double* partials, int nblocks, int ncomp, double* d_out);

// stats
void stat_begin(sv_handle* h, int cls, double bytes, cudaEvent_t* ev_pair);
void stat_end(sv_handle* h, int cls, double bytes, cudaEvent_t* ev_pair);
void ensure_partials(sv_handle* h, size_t doubles);
void ensure_results(sv_handle* h, size_t doubles);

// fused tile engine (fused.cu / planner.cpp)
// runs the fused program on every state; returns the layout change (qubit at local p -> perm[p])
// gen_out (adjoint sweep, PRIM_GEN prims present): receives (Prim::slot, <lambda|G|psi>) pairs
// state_hi: two-array state (indices with the top local bit live in state_hi; that bit is pinned)
// allow_remap = false: no in-tile relabeling (the program leaves every qubit where it found it)
// rank_uniform (sharded): prims still carry their controls / diagonal bits on global positions
// (>= nl), identical on every rank; the kernels evaluate them against this rank's global bits
// (DPass::gbits), so every rank runs the same program and in-tile relabeling is allowed
std::vector<int> apply_prims_fused(sv_handle* h, const std::vector<double2*>& states, const std::vector<Prim>& prims,
                                   std::vector<std::pair<int, cplx>>* gen_out = nullptr, double2* state_hi = nullptr,
                                   bool allow_remap = true, bool rank_uniform = false);
// flat serialisation of the fused program for an op list (host only; tests re-execute it on CPU)
void plan_program_serialized(int n_qubits, const std::vector<Prim>& prims, std::vector<int64_t>& ints,
                             std::vector<double>& dbls);
void release_fused(sv_handle* h);
struct PlanStats {
  int64_t passes = 0, ops = 0, tile_bits = 0, phases = 0;
  double fp64_flops_per_amp = 0.0;
};
PlanStats plan_stats(int nl, const std::vector<Prim>& prims);
void plan_compile(int nl, const std::vector<Prim>& prims, bool two, int64_t* out4);

// bytes per amplitude in the handle's precision
inline size_t amp_bytes(const sv_handle* h) { return h->prec == 32 ? sizeof(float2) : sizeof(double2); }

inline int popcount64(u64 x) { return __builtin_popcountll(x); }
