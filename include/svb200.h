/*
 * svb200.h -- C-ABI of the B200-native complex128 state-vector hot path.
 *
 * This is the drop-in boundary for the reference's device API (py-bindings,
 * bind_device / apply / expval / probs / adjoint_jacobian /
 * get_state / set_state).  Plain C types only: opaque handle, int status,
 * caller-owned host buffers copied synchronously (copy-out marshalling,
 * SPEC.md:663).  Amplitudes are interleaved (re, im) doubles == numpy
 * complex128, qubit 0 = most significant index bit (state.py:1-5).
 *
 * Status codes map 1:1 onto the reference exception classes (errors.py:4-17,
 * SPEC.md:652); sv_last_error() returns the thread-local message.
 *
 * Reference interface each entry point replaces (file:line under
 * /root/reference):
 *   sv_create / sv_reset           StateVector.__init__ / zero_state   pkg/src/svkit/state.py:34-47, 90-92
 *   sv_set_state / sv_get_state    StateVector.from_amplitudes / .amplitudes  state.py:49-66
 *   sv_norm                        StateVector.norm                    state.py:76-78
 *   sv_apply_single_qubit          apply_single_qubit (Alg. 1)         state.py:154-171
 *   sv_apply_controlled_single_qubit apply_controlled_single_qubit (Alg. 2) state.py:192-226
 *   sv_apply_matrix                apply_matrix                        state.py:278-303
 *   sv_apply_ops                   Device.apply (op list)              SPEC.md:649 (circuit op SPEC.md:494)
 *   sv_expval / sv_probs           measurements.expval / probabilities SPEC.md:283-301
 *   sv_var                         measurements.variance
 *   sv_sample                      measurements.sample / sample_root
 *   sv_adjoint_jacobian            adjoint_jacobian
 *   sv_create_sharded              ShardedState / shard
 *   sv_create_ex (precision 32)    StateVector(n, precision="f32")     state.py:20, 34-47
 *   sv_set_state_c64 / sv_get_state_c64  from_amplitudes(complex64) / .amplitudes  state.py:49-66
 */
#ifndef SVB200_H
#define SVB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-17) ---- */
#define SV_OK 0
#define SV_ERR_VALIDATION 1   /* ValidationError */
#define SV_ERR_CAPACITY 2     /* CapacityError (incl. cudaErrorMemoryAllocation) */
#define SV_ERR_UNSUPPORTED 3  /* UnsupportedOperationError */
#define SV_ERR_DEVICE 4       /* CUDA / NCCL failure */

/* ---- gate kinds, SPEC.md:129 order ---- */
enum sv_gate_kind {
  SV_GATE_I = 0, SV_GATE_X, SV_GATE_Y, SV_GATE_Z, SV_GATE_H, SV_GATE_S, SV_GATE_T,
  SV_GATE_PHASE, SV_GATE_RX, SV_GATE_RY, SV_GATE_RZ, SV_GATE_ROT, SV_GATE_CNOT,
  SV_GATE_CZ, SV_GATE_SWAP, SV_GATE_ISINGXX, SV_GATE_ISINGXY, SV_GATE_ISINGYY,
  SV_GATE_ISINGZZ, SV_GATE_SINGLE_EXCITATION, SV_GATE_DOUBLE_EXCITATION,
  SV_GATE_CONTROLLED_MATRIX, SV_GATE_MATRIX, SV_GATE_COUNT
};

/* One circuit operation.  wires = target wires (CNOT: control,
 * target).  ctrl_values may be NULL (all ones, state.py:175-176) and align
 * with ctrls as given (state.py:214-215).  trainable_mask bit p marks
 * params[p] trainable.  matrix: row-major interleaved complex 2^w x 2^w
 * (MATRIX / CONTROLLED_MATRIX only), wires[0] = MSB of the matrix index. */
typedef struct sv_op {
  int32_t kind;
  int32_t n_wires;
  const int32_t* wires;
  int32_t n_ctrls;
  const int32_t* ctrls;
  const int32_t* ctrl_values;
  double params[3];
  int32_t inverse;
  int32_t trainable_mask;
  const double* matrix;
} sv_op;

/* Observables. */
#define SV_OBS_PAULI 0        /* one Pauli word, coefficient 1 */
#define SV_OBS_HAMILTONIAN 1  /* sum_t coeffs[t] * P_t */
#define SV_OBS_DENSE 2        /* dense Hermitian on wires */
#define SV_OBS_SPARSE 3       /* CSR Hermitian on the whole register (single-GPU states) */
typedef struct sv_obs {
  int32_t type;
  int32_t n_terms;             /* PAULI: 1 */
  const double* coeffs;        /* HAMILTONIAN: n_terms (NULL for PAULI) */
  const int32_t* term_len;     /* per term: number of (wire, pauli) factors */
  const int32_t* term_wires;   /* concatenated factor wires */
  const char* term_paulis;     /* concatenated 'I'/'X'/'Y'/'Z' */
  int32_t n_wires;             /* DENSE */
  const int32_t* wires;        /* DENSE */
  const double* matrix;        /* DENSE: interleaved complex 2^w x 2^w */
  /* SPARSE: CSR over logical basis indices, dim = 2^n_qubits */
  int64_t csr_dim;
  int64_t csr_nnz;
  const int64_t* csr_indptr;   /* dim + 1, monotone, [0] = 0, [dim] = nnz */
  const int64_t* csr_indices;  /* nnz columns in [0, dim) */
  const double* csr_data;      /* nnz interleaved complex values */
} sv_obs;

typedef struct sv_handle sv_handle;

/* ---- lifecycle ---- */
int sv_device_count(int* out);
int sv_create(int n_qubits, int device, sv_handle** out);
/* Sharded state over `world` processes (one per GPU, world a power of two);
 * global qubits are the top log2(world).  nccl_id = the 128-byte
 * ncclUniqueId produced by sv_nccl_unique_id on rank 0 and broadcast. */
int sv_nccl_unique_id(void* out128);
int sv_create_sharded(int n_qubits, int rank, int world, int device, const void* nccl_id, sv_handle** out);
int sv_destroy(sv_handle* h);
int sv_info(const sv_handle* h, int64_t* out6); /* n, n_local, rank, world, device, precision bits */
/* Single-GPU state in either precision of the reference's StateVector (state.py:20):
 * precision_bits 64 = complex128 (as sv_create), 32 = complex64.  A complex64 state runs the
 * one-kernel-per-op gate kernels in FP32 arithmetic (the reference casts gate matrices to the
 * state dtype, state.py:264, 273) -- the tile-fusion engine and the fused adjoint sweep are
 * complex128-only, so `fuse` is ignored -- while expval / var / probs / sample / adjoint
 * bra-kets accumulate in FP64.  State I/O goes through the _c64 entry points (interleaved
 * floats == numpy complex64); the double-buffer ones return a validation error. */
int sv_create_ex(int n_qubits, int device, int precision_bits, sv_handle** out);

/* ---- state I/O (bit-exact round trip) ---- */
int sv_reset(sv_handle* h);                                  /* |0...0> */
int sv_set_basis_state(sv_handle* h, uint64_t index);
int sv_set_state(sv_handle* h, const double* amps, uint64_t n_amps);   /* full 2^n vector */
int sv_get_state(sv_handle* h, double* out, uint64_t n_amps);         /* full 2^n vector */
int sv_norm(sv_handle* h, double* out);
int sv_set_state_c64(sv_handle* h, const float* amps, uint64_t n_amps);  /* complex64 handles */
int sv_get_state_c64(sv_handle* h, float* out, uint64_t n_amps);

/* ---- gate application ---- */
int sv_apply_single_qubit(sv_handle* h, int q, const double* m2x2);
int sv_apply_controlled_single_qubit(sv_handle* h, const int32_t* ctrls, int n_ctrls, int q,
                                     const double* m2x2, const int32_t* ctrl_values);
int sv_apply_matrix(sv_handle* h, const int32_t* wires, int n_wires, const double* matrix);
/* fuse: 0 = one kernel per op, 1 = shared-memory tile fusion (default in Device). */
int sv_apply_ops(sv_handle* h, const sv_op* ops, int n_ops, int fuse);

/* ---- measurements ---- */
/* Dense observables: <= 4 wires as one in-register bra-ket pass; 5..12 wires need one extra
 * state buffer (lambda = O psi, then Re<psi|lambda>), SV_ERR_CAPACITY when it does not fit. */
int sv_expval(sv_handle* h, const sv_obs* obs, double* out);
int sv_probs(sv_handle* h, const int32_t* wires, int n_wires, double* out); /* n_wires=0: all */
/* <O^2> - <O>^2 (Pauli word: 1 - <P>^2; otherwise |O psi|^2 - <psi|O psi>^2). */
int sv_var(sv_handle* h, const sv_obs* obs, double* out);
/* shots i.i.d. outcomes over `wires` (n_wires=0: all; wires[0] = MSB of the outcome index),
 * deterministic per seed and identical for sharded and single-GPU states: with p = the
 * marginal probabilities (sv_probs) and C their sequential inclusive prefix sums, shot i draws
 * x = splitmix64(seed + (i + 1) * 0x9E3779B97F4A7C15), u = (x >> 11) * 2^-53, and returns the
 * first b with C[b] > u * C[last].  out: shots int64 outcome indices.  shots == 0 -> validation
 * error; more than 30 wires -> capacity error. */
int sv_sample(sv_handle* h, const int32_t* wires, int n_wires, uint64_t shots, uint64_t seed, int64_t* out);

/* ---- adjoint Jacobian ----
 * Runs ops forward from the handle's current state, then the reverse sweep.
 * jac: row-major n_obs x n_trainable (trainable = set bits of trainable_mask
 * in op order, Rot params in (phi, theta, omega) order).  expvals (may be
 * NULL): <O_k> of the final state.  On return the handle holds the forward
 * state swept back to the input (to fp64 round-off). */
int sv_adjoint_jacobian(sv_handle* h, const sv_op* ops, int n_ops, const sv_obs* obs, int n_obs,
                        int fuse, double* jac, double* expvals);

/* ---- diagnostics / measurement support ---- */
const char* sv_last_error(void);
int sv_synchronize(sv_handle* h);
void* sv_stream(sv_handle* h);                 /* cudaStream_t the kernels run on */
int64_t sv_launch_count(const sv_handle* h);   /* kernels launched by this handle */
/* Per-kernel-class device time (CUDA events around each launch when enabled). */
int sv_set_profiling(sv_handle* h, int enabled);
/* out[3*k+0]=launches, out[3*k+1]=total ms, out[3*k+2]=algorithmic bytes, for k < n_classes. */
int sv_kernel_stats(sv_handle* h, double* out, int max_classes, int* n_classes, char* names, int names_len);
int sv_reset_stats(sv_handle* h);
/* Fusion plan summary for an op list (host-only; no GPU needed):
 * out[0]=passes, out[1]=ops, out[2]=tile bits, out[3]=phases. */
int sv_plan_summary(int n_qubits, const sv_op* ops, int n_ops, int64_t* out4);
/* The fused program itself, flattened (format: fused_plan.cpp serialize_program); host-only.
 * sizes2 receives the needed int64 / double counts; buffers are filled when large enough. */
int sv_plan_program(int n_qubits, const sv_op* ops, int n_ops, int64_t* ints, int64_t ints_cap, double* dbls,
                    int64_t dbls_cap, int64_t* sizes2);
/* FP64 floating-point operations per state amplitude that the fused program of an op list performs
 * (DFMA = 2), counted from its planned op cases; host-only (bench.py's FP64 roofline). */
int sv_plan_fp64(int n_qubits, const sv_op* ops, int n_ops, double* flops_per_amp);
/* Runtime pass compiler (host-only, no GPU needed): plan the op list and compile every fused pass
 * into its own sm_100a kernel with NVRTC (the kernels the device path launches; cached
 * process-wide by pass structure).  two_array = plan for the adjoint sweep's psi|lambda state.
 * out[0]=passes, out[1]=passes with a generated kernel, out[2]=kernels compiled so far in this
 * process, out[3]=their total compile time in microseconds. */
int sv_plan_compile(int n_qubits, const sv_op* ops, int n_ops, int two_array, int64_t* out4);
/* Process-wide pass-compiler counters: out3[0] = kernels compiled (NVRTC runs, disk-cache hits
 * excluded), out3[1] = microseconds spent compiling, out3[2] = distinct kernels held. */
int sv_jit_stats(int64_t* out3);
/* The sharded driver's decisions for one rank (local primitives, global-qubit swaps, final
 * canonicalisation), recorded without a GPU; same sizing convention. */
int sv_plan_sharded(int n_qubits, int rank, int world, const sv_op* ops, int n_ops, int64_t* ints, int64_t ints_cap,
                    double* dbls, int64_t dbls_cap, int64_t* sizes2);

#ifdef __cplusplus
}
#endif
#endif /* SVB200_H */
