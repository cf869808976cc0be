// sm_100a kernels of libsvb200: one-op-per-pass gate kernels (K1-K6 of SURVEY.md §2.3),
// observable reductions (K8/K9/K12/K13), observable application (K10) and the generator
// bra-ket used by the adjoint sweep (K11).  All complex128 (double2), in place, 64-bit
// indices; every kernel is an HBM streaming pass (~0.44 flop/B).
//
// Index arithmetic: a PAIR / DIAG / DENSE primitive enumerates a compact counter k over the
// non-fixed bits and spreads it around the fixed bit positions ("insert a zero bit at each
// fixed position, ascending"), then ORs the fixed pattern -- the get_masks / MaskSet.expand
// construction of the reference (state.py:112-151, 212-225) done with shifts, no division.
#include <algorithm>
#include <cstring>

#include "sv_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kRedBlocks = 148 * 4;   // fixed reduction grid: deterministic partial order

struct Ins {
  int n;
  unsigned char p[63];   // ascending fixed bit positions
};

__device__ __forceinline__ u64 deposit(u64 k, const Ins& s) {
  for (int i = 0; i < s.n; ++i) {
    const int p = s.p[i];
    const u64 lo = k & ((1ull << p) - 1ull);
    k = ((k ^ lo) << 1) | lo;
  }
  return k;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 conjmul(double2 a, double2 b) {        // conj(a)*b
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}

// ---------------------------------------------------------------------------
// K1/K2/K4: PAIR  (Alg. 1 / Alg. 2 generalised; 2x2 on (i0, i0^xmask))
// ---------------------------------------------------------------------------
struct PairParams {
  double2 m[4];
  u64 fval, xmask, count;
  Ins ins;
};

template <int ITEMS>
__global__ void __launch_bounds__(kThreads) k_pair(double2* __restrict__ a, const PairParams P) {
  const u64 base = u64(blockIdx.x) * (ITEMS * kThreads) + threadIdx.x;
  u64 i0[ITEMS];
  double2 v0[ITEMS], v1[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const u64 k = base + u64(j) * kThreads;
    i0[j] = (k < P.count) ? (deposit(k, P.ins) | P.fval) : ~0ull;
    if (i0[j] != ~0ull) {
      v0[j] = a[i0[j]];
      v1[j] = a[i0[j] ^ P.xmask];
    }
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (i0[j] == ~0ull) continue;
    const double2 o0 = cfma(P.m[0], v0[j], cmul(P.m[1], v1[j]));
    const double2 o1 = cfma(P.m[2], v0[j], cmul(P.m[3], v1[j]));
    a[i0[j]] = o0;
    a[i0[j] ^ P.xmask] = o1;
  }
}

// ---------------------------------------------------------------------------
// K3: DIAG  (a[i] *= table[bits]; restricted to (i & fmask) == fval)
// ---------------------------------------------------------------------------
struct DiagParams {
  double2 t[64];
  u64 fval, count;
  int nb;
  unsigned char pos[6];
  Ins ins;
};

template <int ITEMS>
__global__ void __launch_bounds__(kThreads) k_diag(double2* __restrict__ a, const DiagParams P) {
  const u64 base = u64(blockIdx.x) * (ITEMS * kThreads) + threadIdx.x;
  u64 idx[ITEMS];
  double2 v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const u64 k = base + u64(j) * kThreads;
    idx[j] = (k < P.count) ? (deposit(k, P.ins) | P.fval) : ~0ull;
    if (idx[j] != ~0ull) v[j] = a[idx[j]];
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (idx[j] == ~0ull) continue;
    int t = 0;
    for (int b = 0; b < P.nb; ++b) t |= int((idx[j] >> P.pos[b]) & 1ull) << b;
    a[idx[j]] = cmul(P.t[t], v[j]);
  }
}

// ---------------------------------------------------------------------------
// K5/K6: DENSE k-qubit (matrix in shared memory; amplitudes in registers for k <= 4)
// ---------------------------------------------------------------------------
struct DenseParams {
  const double2* mat;    // 4^k entries, row-major, index bit j <-> pos[j]
  u64 fval, count;
  int k;
  unsigned char pos[16];
  Ins ins;
};

template <int K>
__global__ void __launch_bounds__(kThreads) k_dense(double2* __restrict__ a, const DenseParams P) {
  constexpr int D = 1 << K;
  __shared__ double2 M[D * D];
  for (int i = threadIdx.x; i < D * D; i += kThreads) M[i] = P.mat[i];
  __syncthreads();
  const u64 k = u64(blockIdx.x) * kThreads + threadIdx.x;
  if (k >= P.count) return;
  const u64 base = deposit(k, P.ins) | P.fval;
  u64 off[D];
  double2 v[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    u64 o = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if ((r >> j) & 1) o |= 1ull << P.pos[j];
    off[r] = base | o;
    v[r] = a[off[r]];
  }
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < D; ++c) acc = cfma(M[r * D + c], v[c], acc);
    a[off[r]] = acc;
  }
}

// k >= 5: one block per group, amplitudes staged in shared memory, one warp per output row.
__global__ void __launch_bounds__(kThreads) k_dense_big(double2* __restrict__ a, const DenseParams P) {
  extern __shared__ double2 sm[];
  const int D = 1 << P.k;
  double2* in = sm;
  double2* out = sm + D;
  for (u64 g = blockIdx.x; g < P.count; g += gridDim.x) {
    const u64 base = deposit(g, P.ins) | P.fval;
    for (int r = threadIdx.x; r < D; r += kThreads) {
      u64 o = 0;
      for (int j = 0; j < P.k; ++j)
        if ((r >> j) & 1) o |= 1ull << P.pos[j];
      in[r] = a[base | o];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = warp; r < D; r += kThreads / 32) {
      double2 acc = make_double2(0.0, 0.0);
      const double2* row = P.mat + size_t(r) * D;
      for (int c = lane; c < D; c += 32) acc = cfma(row[c], in[c], acc);
      for (int s = 16; s > 0; s >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, s);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, s);
      }
      if (lane == 0) out[r] = acc;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < D; r += kThreads) {
      u64 o = 0;
      for (int j = 0; j < P.k; ++j)
        if ((r >> j) & 1) o |= 1ull << P.pos[j];
      a[base | o] = out[r];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// block reduction helpers (deterministic: fixed grid, fixed tree)
// ---------------------------------------------------------------------------
template <int NC>
__device__ __forceinline__ void block_reduce_store(double (&v)[NC], double* __restrict__ out) {
  __shared__ double red[NC][kThreads / 32];
#pragma unroll
  for (int c = 0; c < NC; ++c)
    for (int s = 16; s > 0; s >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], s);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < NC; ++c) red[c][warp] = v[c];
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double x = (lane < kThreads / 32) ? red[c][lane] : 0.0;
      for (int s = 16; s > 0; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
      if (lane == 0) out[size_t(blockIdx.x) * NC + c] = x;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_sum_partials(const double* __restrict__ in, int nblocks, int ncomp,
                                                           double* __restrict__ out) {
  const int c = blockIdx.x;
  double v[1] = {0.0};
  for (int b = threadIdx.x; b < nblocks; b += kThreads) v[0] += in[size_t(b) * ncomp + c];
  __shared__ double red[kThreads / 32];
  for (int s = 16; s > 0; s >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v[0];
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = (threadIdx.x < kThreads / 32) ? red[threadIdx.x] : 0.0;
    for (int s = 16; s > 0; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
    if (threadIdx.x == 0) out[c] = x;
  }
}

// Pauli-sum term for K10 (observable application): coefficient * i^{nY} and the z-mask
struct PauliApplyTermDev {
  u64 z;
  double2 cc;
};

__global__ void __launch_bounds__(kThreads) k_norm2(const double2* __restrict__ a, u64 n, double* __restrict__ partials) {
  double v[1] = {0.0};
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    const double2 x = a[i];
    v[0] = fma(x.x, x.x, fma(x.y, x.y, v[0]));
  }
  block_reduce_store<1>(v, partials);
}

// Re <a|b> partials (K12)
__global__ void __launch_bounds__(kThreads) k_dot_re(const double2* __restrict__ a, const double2* __restrict__ b, u64 n,
                                                     double* __restrict__ partials) {
  double v[1] = {0.0};
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    const double2 x = a[i], y = b[i];
    v[0] = fma(x.x, y.x, fma(x.y, y.y, v[0]));
  }
  block_reduce_store<1>(v, partials);
}

// ---- sparse (CSR) observables ---------------------------------------
// Row i / column j are LOGICAL basis indices; the state is addressed through the layout
// permutation (logical bit o -> physical bit phys[o]) as five byte-wise lookup tables.
struct CsrArgs {
  const int64_t* indptr;
  const int64_t* indices;
  const double2* data;
  const u64* perm_tab;   // [5][256]: physical bits of logical byte b with value v (nullptr: identity)
  u64 rows;
};

__device__ __forceinline__ u64 to_phys(u64 i, const u64* __restrict__ t) {
  if (!t) return i;
  return t[i & 255] | t[256 + ((i >> 8) & 255)] | t[512 + ((i >> 16) & 255)] | t[768 + ((i >> 24) & 255)] |
         t[1024 + ((i >> 32) & 255)];
}

// one warp per row: acc = sum_k A[i, j_k] psi_j; expval partial += Re(conj(psi_i) acc), or lam_i = acc
template <bool APPLY>
__global__ void __launch_bounds__(kThreads) k_csr(const double2* __restrict__ psi, const CsrArgs A,
                                                  double2* __restrict__ lam, double* __restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (kThreads / 32);
  double v[1] = {0.0};
  for (u64 row = u64(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5); row < A.rows; row += warps) {
    double ax = 0.0, ay = 0.0;
    for (int64_t k = A.indptr[row] + lane; k < A.indptr[row + 1]; k += 32) {
      const double2 m = A.data[k];
      const double2 x = psi[to_phys(u64(A.indices[k]), A.perm_tab)];
      ax = fma(m.x, x.x, fma(-m.y, x.y, ax));
      ay = fma(m.x, x.y, fma(m.y, x.x, ay));
    }
    for (int s = 16; s > 0; s >>= 1) {
      ax += __shfl_xor_sync(0xffffffffu, ax, s);
      ay += __shfl_xor_sync(0xffffffffu, ay, s);
    }
    if (lane == 0) {
      const u64 pr = to_phys(row, A.perm_tab);
      if (APPLY) {
        lam[pr] = make_double2(ax, ay);
      } else {
        const double2 p = psi[pr];
        v[0] += p.x * ax + p.y * ay;   // Re(conj(p) * acc)
      }
    }
  }
  if (!APPLY) block_reduce_store<1>(v, partials);
}

// K10 batched: lam = sum over up to kMaxXG x-groups of sum_t cc_t (-1)^{pc((i^x_g) & z_t)} psi_{i^x_g};
// psi is read once per group, lam written once (instead of a read-modify-write per group).
constexpr int kMaxXG = 16;
struct PauliGroupsArgs {
  u64 x[kMaxXG];
  int t_begin[kMaxXG + 1];   // term ranges per group in the shared term array
  int ng;
};

__global__ void __launch_bounds__(kThreads) k_pauli_apply_multi(const double2* __restrict__ psi, double2* __restrict__ lam,
                                                                u64 n, const PauliGroupsArgs G,
                                                                const PauliApplyTermDev* __restrict__ terms, int nterms,
                                                                int accumulate) {
  extern __shared__ PauliApplyTermDev sat2[];
  for (int t = threadIdx.x; t < nterms; t += kThreads) sat2[t] = terms[t];
  __syncthreads();
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    double2 o = accumulate ? lam[i] : make_double2(0.0, 0.0);
    for (int g = 0; g < G.ng; ++g) {
      const u64 j = i ^ G.x[g];
      const double2 b = psi[j];
      double2 s = make_double2(0.0, 0.0);
      for (int t = G.t_begin[g]; t < G.t_begin[g + 1]; ++t) {
        const double sg = (__popcll(j & sat2[t].z) & 1) ? -1.0 : 1.0;
        s.x = fma(sg, sat2[t].cc.x, s.x);
        s.y = fma(sg, sat2[t].cc.y, s.y);
      }
      o = cfma(s, b, o);
    }
    lam[i] = o;
  }
}

// ---------------------------------------------------------------------------
// K8/K9: Pauli-group expectation  sum_t Re(cc_t <psi| P_t |psi>)  for terms sharing xmask.
//   x != 0: pairs (i, j = i^x) with bit `pivot` of i = 0; w = conj(psi_j) psi_i;
//           term contribution s_i(t) * r_t * (e_t ? Re w : Im w) with r_t precomputed.
//   x == 0: |psi_i|^2 * sum_t s_i(t) Re(cc_t).
// ---------------------------------------------------------------------------
struct PauliTermDev {
  u64 z;
  double r;       // real weight
  int use_im;     // 0: Re(w), 1: Im(w)
};

__global__ void __launch_bounds__(kThreads) k_pauli_expval(const double2* __restrict__ a, u64 xmask, int pivot, u64 count,
                                                           const PauliTermDev* __restrict__ terms, int nterms,
                                                           double* __restrict__ partials) {
  extern __shared__ PauliTermDev st[];
  for (int t = threadIdx.x; t < nterms; t += kThreads) st[t] = terms[t];
  __syncthreads();
  double v[1] = {0.0};
  for (u64 k = u64(blockIdx.x) * kThreads + threadIdx.x; k < count; k += u64(gridDim.x) * kThreads) {
    if (xmask == 0) {
      const double2 x = a[k];
      const double p = fma(x.x, x.x, x.y * x.y);
      double s = 0.0;
      for (int t = 0; t < nterms; ++t) s += (__popcll(k & st[t].z) & 1) ? -st[t].r : st[t].r;
      v[0] = fma(p, s, v[0]);
    } else {
      const u64 lo = k & ((1ull << pivot) - 1ull);
      const u64 i = ((k ^ lo) << 1) | lo;
      const double2 ai = a[i], aj = a[i ^ xmask];
      const double2 w = conjmul(aj, ai);
      double s = 0.0;
      for (int t = 0; t < nterms; ++t) {
        const double c = st[t].use_im ? w.y : w.x;
        s += (__popcll(i & st[t].z) & 1) ? -st[t].r * c : st[t].r * c;
      }
      v[0] += s;
    }
  }
  block_reduce_store<1>(v, partials);
}

// K10: lambda (+)= sum_t cc_t (-1)^{pc((i^x) & z_t)} psi_{i^x}   (PauliApplyTermDev: see above)

__global__ void __launch_bounds__(kThreads) k_pauli_apply(const double2* __restrict__ psi, double2* __restrict__ lam, u64 xmask,
                                                          u64 n, const PauliApplyTermDev* __restrict__ terms, int nterms,
                                                          int accumulate) {
  extern __shared__ PauliApplyTermDev sat[];
  for (int t = threadIdx.x; t < nterms; t += kThreads) sat[t] = terms[t];
  __syncthreads();
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    const u64 j = i ^ xmask;
    const double2 b = psi[j];
    double2 s = make_double2(0.0, 0.0);
    for (int t = 0; t < nterms; ++t) {
      const double sg = (__popcll(j & sat[t].z) & 1) ? -1.0 : 1.0;
      s.x = fma(sg, sat[t].cc.x, s.x);
      s.y = fma(sg, sat[t].cc.y, s.y);
    }
    double2 o = cmul(s, b);
    if (accumulate) {
      const double2 l = lam[i];
      o.x += l.x;
      o.y += l.y;
    }
    lam[i] = o;
  }
}

// K11 helper: <bra| P (G (x) I) |ket> over groups (complex partial), G dense 2^K x 2^K in smem.
template <int K>
__global__ void __launch_bounds__(kThreads) k_braket(const double2* __restrict__ bra, const double2* __restrict__ ket,
                                                     const DenseParams P, double* __restrict__ partials) {
  constexpr int D = 1 << K;
  __shared__ double2 M[D * D];
  for (int i = threadIdx.x; i < D * D; i += kThreads) M[i] = P.mat[i];
  __syncthreads();
  double v[2] = {0.0, 0.0};
  for (u64 k = u64(blockIdx.x) * kThreads + threadIdx.x; k < P.count; k += u64(gridDim.x) * kThreads) {
    const u64 base = deposit(k, P.ins) | P.fval;
    double2 x[D];
    u64 off[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      u64 o = 0;
#pragma unroll
      for (int j = 0; j < K; ++j)
        if ((r >> j) & 1) o |= 1ull << P.pos[j];
      off[r] = base | o;
      x[r] = ket[off[r]];
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < D; ++c) acc = cfma(M[r * D + c], x[c], acc);
      const double2 b = bra[off[r]];
      const double2 t = conjmul(b, acc);
      v[0] += t.x;
      v[1] += t.y;
    }
  }
  block_reduce_store<2>(v, partials);
}

// K13: marginal probabilities.  bins = 2^w, bin bit (w-1-j) <- position pos[j] (wires[0] = MSB).
struct ProbParams {
  u64 members;     // 2^(nl - w) per bin
  int w;
  unsigned char pos[63];
  Ins ins;         // ascending wire positions (to enumerate members)
};

__device__ __forceinline__ u64 bin_pattern(u64 b, const ProbParams& P) {
  u64 o = 0;
  for (int j = 0; j < P.w; ++j)
    if ((b >> (P.w - 1 - j)) & 1) o |= 1ull << P.pos[j];
  return o;
}

// one block per (chunk, bin): partials[chunk * bins + bin]
__global__ void __launch_bounds__(kThreads) k_probs_chunked(const double2* __restrict__ a, const ProbParams P, int chunks,
                                                            double* __restrict__ partials) {
  const u64 bins = 1ull << P.w;
  const u64 bin = blockIdx.x % bins;
  const int chunk = int(blockIdx.x / bins);
  const u64 pat = bin_pattern(bin, P);
  double v[1] = {0.0};
  for (u64 k = u64(chunk) * kThreads + threadIdx.x; k < P.members; k += u64(chunks) * kThreads) {
    const double2 x = a[deposit(k, P.ins) | pat];
    v[0] = fma(x.x, x.x, fma(x.y, x.y, v[0]));
  }
  block_reduce_store<1>(v, partials);
}

// one thread per bin (few members per bin)
__global__ void __launch_bounds__(kThreads) k_probs_perbin(const double2* __restrict__ a, const ProbParams P, u64 bins,
                                                           double* __restrict__ out) {
  const u64 bin = u64(blockIdx.x) * kThreads + threadIdx.x;
  if (bin >= bins) return;
  const u64 pat = bin_pattern(bin, P);
  double s = 0.0;
  for (u64 k = 0; k < P.members; ++k) {
    const double2 x = a[deposit(k, P.ins) | pat];
    s = fma(x.x, x.x, fma(x.y, x.y, s));
  }
  out[bin] = s;
}

Ins make_ins(u64 fmask) {
  Ins s;
  s.n = 0;
  for (int b = 0; b < 64; ++b)
    if ((fmask >> b) & 1) s.p[s.n++] = (unsigned char)b;
  return s;
}

inline unsigned grid_for(u64 work, u64 per_block) {
  u64 g = (work + per_block - 1) / per_block;
  return unsigned(std::max<u64>(g, 1));
}

inline unsigned red_grid(u64 work) {
  u64 g = (work + kThreads * 4 - 1) / (kThreads * 4);
  return unsigned(std::min<u64>(std::max<u64>(g, 1), kRedBlocks));
}

double2 d2(cplx c) { return make_double2(c.real(), c.imag()); }

// device buffer for small per-launch tables (matrices, term lists); grows, never shrinks
void* scratch_upload(sv_handle* h, const void* src, size_t bytes);

}  // namespace

// ===========================================================================
// host launchers
// ===========================================================================
const char* kKernelClassNames[KC_COUNT] = {"pair", "diag", "dense", "fused_tile", "reduce", "apply_obs",
                                           "braket", "probs", "init", "swap"};

namespace {
struct ScratchBuf {
  void* ptr = nullptr;
  size_t cap = 0;
};
// per-handle upload scratch lives in a side table keyed by handle
std::mutex g_scratch_mu;
std::vector<std::pair<sv_handle*, std::vector<ScratchBuf>>> g_scratch;
thread_local int g_scratch_slot = 0;

void* scratch_upload(sv_handle* h, const void* src, size_t bytes) {
  // ring of 64 buffers so back-to-back async uploads do not overwrite in-flight tables
  std::vector<ScratchBuf>* bufs = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    for (auto& e : g_scratch)
      if (e.first == h) bufs = &e.second;
    if (!bufs) {
      g_scratch.push_back({h, std::vector<ScratchBuf>(64)});
      bufs = &g_scratch.back().second;
    }
  }
  ScratchBuf& b = (*bufs)[g_scratch_slot];
  g_scratch_slot = (g_scratch_slot + 1) % 64;
  if (b.cap < bytes) {
    if (b.ptr) {
      CUDA_CHECK(cudaStreamSynchronize(h->stream));
      CUDA_CHECK(cudaFree(b.ptr));
    }
    size_t cap = std::max<size_t>(bytes, 4096);
    CUDA_CHECK(cudaMalloc(&b.ptr, cap));
    b.cap = cap;
  }
  CUDA_CHECK(cudaMemcpyAsync(b.ptr, src, bytes, cudaMemcpyHostToDevice, h->stream));
  return b.ptr;
}
}  // namespace

void release_scratch(sv_handle* h) {
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  for (size_t i = 0; i < g_scratch.size(); ++i)
    if (g_scratch[i].first == h) {
      for (auto& b : g_scratch[i].second)
        if (b.ptr) cudaFree(b.ptr);
      g_scratch.erase(g_scratch.begin() + i);
      return;
    }
}

// Algorithmic bytes of one unfused primitive: 32 B (16 read + 16 written) per touched amplitude.
double prim_bytes(const sv_handle* h, const Prim& p) {
  if (p.skip) return 0.0;
  if (p.type == PRIM_PAIR) return 32.0 * 2.0 * double(h->n_local >> popcount64(p.fmask));
  if (p.type == PRIM_DIAG) return 32.0 * double(h->n_local >> popcount64(p.fmask));
  return 32.0 * double(h->n_local >> (popcount64(p.fmask) - p.nb));
}

void launch_prim(sv_handle* h, double2* a, const Prim& p) {
  if (p.skip) return;
  if (h->recording) {   // host-only planning (sv_plan_sharded)
    h->rec.push_back({REC_PRIM, p, -1});
    return;
  }
  const int nf = popcount64(p.fmask);
  if (nf > h->nl) sv_fail(SV_ERR_DEVICE, "internal: primitive fixes more bits than the shard has");
  const u64 count = h->n_local >> nf;
  cudaEvent_t ev[2];
  if (p.type == PRIM_PAIR) {
    PairParams P;
    for (int i = 0; i < 4; ++i) P.m[i] = d2(p.m[i]);
    P.fval = p.fval;
    P.xmask = p.xmask;
    P.count = count;
    P.ins = make_ins(p.fmask);
    stat_begin(h, KC_PAIR, prim_bytes(h, p), ev);
    k_pair<4><<<grid_for(count, 4 * kThreads), kThreads, 0, h->stream>>>(a, P);
    stat_end(h, KC_PAIR, prim_bytes(h, p), ev);
  } else if (p.type == PRIM_DIAG) {
    DiagParams P;
    if (p.nb > 6) sv_fail(SV_ERR_DEVICE, "internal: diagonal table too large");
    for (size_t i = 0; i < p.m.size(); ++i) P.t[i] = d2(p.m[i]);
    P.fval = p.fval;
    P.count = count;
    P.nb = p.nb;
    for (int j = 0; j < p.nb; ++j) P.pos[j] = (unsigned char)p.pos[j];
    P.ins = make_ins(p.fmask);
    stat_begin(h, KC_DIAG, prim_bytes(h, p), ev);
    k_diag<4><<<grid_for(count, 4 * kThreads), kThreads, 0, h->stream>>>(a, P);
    stat_end(h, KC_DIAG, prim_bytes(h, p), ev);
  } else {
    DenseParams P;
    std::vector<double2> mat(p.m.size());
    for (size_t i = 0; i < p.m.size(); ++i) mat[i] = d2(p.m[i]);
    P.mat = (const double2*)scratch_upload(h, mat.data(), mat.size() * sizeof(double2));
    P.fval = p.fval;
    P.count = count;
    P.k = p.nb;
    for (int j = 0; j < p.nb; ++j) P.pos[j] = (unsigned char)p.pos[j];
    P.ins = make_ins(p.fmask);
    stat_begin(h, KC_DENSE, prim_bytes(h, p), ev);
    const unsigned g = grid_for(count, kThreads);
    switch (p.nb) {
      case 1: k_dense<1><<<g, kThreads, 0, h->stream>>>(a, P); break;
      case 2: k_dense<2><<<g, kThreads, 0, h->stream>>>(a, P); break;
      case 3: k_dense<3><<<g, kThreads, 0, h->stream>>>(a, P); break;
      case 4: k_dense<4><<<g, kThreads, 0, h->stream>>>(a, P); break;
      default: {
        if (p.nb > 12) sv_fail(SV_ERR_UNSUPPORTED, "dense matrices on more than 12 wires are not supported on the GPU path");
        const size_t smem = (size_t(2) << p.nb) * sizeof(double2);   // in + out, 2^k each
        if (smem > 48 * 1024) CUDA_CHECK(cudaFuncSetAttribute(k_dense_big, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        unsigned gb = unsigned(std::min<u64>(count, 148ull * 16));
        k_dense_big<<<gb, kThreads, smem, h->stream>>>(a, P);
      }
    }
    stat_end(h, KC_DENSE, prim_bytes(h, p), ev);
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_init_zero(sv_handle* h, double2* a, u64 basis_local, bool set_one) {
  cudaEvent_t ev[2];
  stat_begin(h, KC_INIT, 16.0 * double(h->n_local), ev);
  CUDA_CHECK(cudaMemsetAsync(a, 0, h->n_local * sizeof(double2), h->stream));
  if (set_one) {
    static const double2 one = {1.0, 0.0};
    CUDA_CHECK(cudaMemcpyAsync(a + basis_local, &one, sizeof(double2), cudaMemcpyHostToDevice, h->stream));
  }
  stat_end(h, KC_INIT, 16.0 * double(h->n_local), ev);
}

void launch_copy(sv_handle* h, double2* dst, const double2* src, u64 n) {
  cudaEvent_t ev[2];
  stat_begin(h, KC_INIT, 32.0 * double(n), ev);
  CUDA_CHECK(cudaMemcpyAsync(dst, src, n * sizeof(double2), cudaMemcpyDeviceToDevice, h->stream));
  stat_end(h, KC_INIT, 32.0 * double(n), ev);
}

void sum_partials(sv_handle* h, const double* partials, int nblocks, int ncomp, double* d_out) {
  k_sum_partials<<<ncomp, kThreads, 0, h->stream>>>(partials, nblocks, ncomp, d_out);
  h->launches++;
  CUDA_CHECK(cudaGetLastError());
}

double reduce_norm2(sv_handle* h, const double2* a) {
  const unsigned g = red_grid(h->n_local);
  ensure_partials(h, g);
  ensure_results(h, 1);
  cudaEvent_t ev[2];
  stat_begin(h, KC_REDUCE, 16.0 * double(h->n_local), ev);
  k_norm2<<<g, kThreads, 0, h->stream>>>(a, h->n_local, h->d_partials);
  stat_end(h, KC_REDUCE, 16.0 * double(h->n_local), ev);
  CUDA_CHECK(cudaGetLastError());
  sum_partials(h, h->d_partials, g, 1, h->d_results);
  double out = 0;
  CUDA_CHECK(cudaMemcpyAsync(&out, h->d_results, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->stream));
  return out;
}

void pauli_group_expval_async(sv_handle* h, const double2* a, u64 xmask, const std::vector<PauliTerm>& terms,
                              double* d_out) {
  std::vector<PauliTermDev> dt(terms.size());
  int pivot = 0;
  if (xmask) pivot = __builtin_ctzll(xmask);
  for (size_t t = 0; t < terms.size(); ++t) {
    dt[t].z = terms[t].zmask;
    if (xmask == 0) {
      dt[t].r = terms[t].cc.real();
      dt[t].use_im = 0;
    } else {
      const bool e_pos = (popcount64(xmask & terms[t].zmask) & 1) == 0;
      dt[t].r = e_pos ? 2.0 * terms[t].cc.real() : -2.0 * terms[t].cc.imag();
      dt[t].use_im = e_pos ? 0 : 1;
    }
  }
  const u64 count = xmask ? (h->n_local >> 1) : h->n_local;
  const unsigned g = red_grid(count);
  ensure_partials(h, g);
  auto* d_terms = (const PauliTermDev*)scratch_upload(h, dt.data(), dt.size() * sizeof(PauliTermDev));
  size_t smem = dt.size() * sizeof(PauliTermDev);
  if (smem > 48 * 1024) CUDA_CHECK(cudaFuncSetAttribute(k_pauli_expval, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaEvent_t ev[2];
  stat_begin(h, KC_REDUCE, 16.0 * double(h->n_local), ev);
  k_pauli_expval<<<g, kThreads, smem, h->stream>>>(a, xmask, pivot, count, d_terms, int(dt.size()), h->d_partials);
  stat_end(h, KC_REDUCE, 16.0 * double(h->n_local), ev);
  CUDA_CHECK(cudaGetLastError());
  sum_partials(h, h->d_partials, g, 1, d_out);
}

void pauli_group_apply(sv_handle* h, const double2* psi, double2* lam, u64 xmask, const std::vector<PauliTerm>& terms,
                       bool accumulate) {
  std::vector<PauliApplyTermDev> dt(terms.size());
  for (size_t t = 0; t < terms.size(); ++t) {
    dt[t].z = terms[t].zmask;
    dt[t].cc = d2(terms[t].cc);
  }
  auto* d_terms = (const PauliApplyTermDev*)scratch_upload(h, dt.data(), dt.size() * sizeof(PauliApplyTermDev));
  size_t smem = dt.size() * sizeof(PauliApplyTermDev);
  if (smem > 48 * 1024) CUDA_CHECK(cudaFuncSetAttribute(k_pauli_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const unsigned g = unsigned(std::min<u64>(grid_for(h->n_local, kThreads * 4), 148ull * 64));
  const double bytes = (accumulate ? 48.0 : 32.0) * double(h->n_local);
  cudaEvent_t ev[2];
  stat_begin(h, KC_APPLY_OBS, bytes, ev);
  k_pauli_apply<<<g, kThreads, smem, h->stream>>>(psi, lam, xmask, h->n_local, d_terms, int(dt.size()), accumulate ? 1 : 0);
  stat_end(h, KC_APPLY_OBS, bytes, ev);
  CUDA_CHECK(cudaGetLastError());
}

void pauli_groups_apply(sv_handle* h, const double2* psi, double2* lam,
                        const std::vector<std::pair<u64, std::vector<PauliTerm>>>& groups) {
  const unsigned g = unsigned(std::min<u64>(grid_for(h->n_local, kThreads * 4), 148ull * 64));
  for (size_t g0 = 0; g0 < groups.size(); g0 += kMaxXG) {
    PauliGroupsArgs G;
    std::vector<PauliApplyTermDev> dt;
    G.ng = int(std::min<size_t>(kMaxXG, groups.size() - g0));
    for (int k = 0; k < G.ng; ++k) {
      G.x[k] = groups[g0 + k].first;
      G.t_begin[k] = int(dt.size());
      for (const auto& t : groups[g0 + k].second) dt.push_back({t.zmask, d2(t.cc)});
    }
    G.t_begin[G.ng] = int(dt.size());
    auto* d_terms = (const PauliApplyTermDev*)scratch_upload(h, dt.data(), dt.size() * sizeof(PauliApplyTermDev));
    const size_t smem = dt.size() * sizeof(PauliApplyTermDev);
    if (smem > 48 * 1024)
      CUDA_CHECK(cudaFuncSetAttribute(k_pauli_apply_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int acc = g0 > 0;
    const double bytes = (16.0 * G.ng + 16.0 + (acc ? 16.0 : 0.0)) * double(h->n_local);
    cudaEvent_t ev[2];
    stat_begin(h, KC_APPLY_OBS, bytes, ev);
    k_pauli_apply_multi<<<g, kThreads, smem, h->stream>>>(psi, lam, h->n_local, G, d_terms, int(dt.size()), acc);
    stat_end(h, KC_APPLY_OBS, bytes, ev);
    CUDA_CHECK(cudaGetLastError());
  }
}

// Sparse observable on a single-GPU state: expval (lam == nullptr) or lam = A psi.  The CSR
// arrays are staged in device memory for the call (validated by the caller).
double csr_apply_or_expval(sv_handle* h, const sv_obs& o, const double2* psi, double2* lam) {
  const u64 rows = u64(o.csr_dim), nnz = u64(o.csr_nnz);
  bool ident = true;
  for (int b = 0; b < h->n; ++b) ident &= h->phys[b] == b;
  std::vector<u64> tab;
  if (!ident) {
    tab.assign(5 * 256, 0);
    for (int byte = 0; byte < 5; ++byte)
      for (int v = 0; v < 256; ++v)
        for (int j = 0; j < 8; ++j) {
          const int o_bit = byte * 8 + j;
          if (((v >> j) & 1) && o_bit < h->n) tab[byte * 256 + v] |= 1ull << h->phys[o_bit];
        }
  }
  const size_t b_ptr = (rows + 1) * sizeof(int64_t), b_idx = nnz * sizeof(int64_t), b_dat = nnz * sizeof(double2);
  const size_t b_tab = tab.size() * sizeof(u64);
  char* buf = nullptr;
  CUDA_CHECK(cudaMallocAsync(&buf, b_ptr + b_idx + b_dat + b_tab + 64, h->stream));
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  CsrArgs A;
  A.indptr = (const int64_t*)buf;
  A.indices = (const int64_t*)(buf + al(b_ptr));
  A.data = (const double2*)(buf + al(b_ptr) + al(b_idx));
  A.perm_tab = ident ? nullptr : (const u64*)(buf + al(b_ptr) + al(b_idx) + al(b_dat));
  A.rows = rows;
  CUDA_CHECK(cudaMemcpyAsync((void*)A.indptr, o.csr_indptr, b_ptr, cudaMemcpyHostToDevice, h->stream));
  if (nnz) {
    CUDA_CHECK(cudaMemcpyAsync((void*)A.indices, o.csr_indices, b_idx, cudaMemcpyHostToDevice, h->stream));
    CUDA_CHECK(cudaMemcpyAsync((void*)A.data, o.csr_data, b_dat, cudaMemcpyHostToDevice, h->stream));
  }
  if (!ident) CUDA_CHECK(cudaMemcpyAsync((void*)A.perm_tab, tab.data(), b_tab, cudaMemcpyHostToDevice, h->stream));
  const unsigned g = red_grid(rows * 32);
  double out = 0.0;
  cudaEvent_t ev[2];
  const double bytes = 16.0 * double(h->n_local) + 24.0 * double(nnz);
  if (lam) {
    CUDA_CHECK(cudaMemsetAsync(lam, 0, h->n_local * sizeof(double2), h->stream));
    stat_begin(h, KC_APPLY_OBS, bytes, ev);
    k_csr<true><<<g, kThreads, 0, h->stream>>>(psi, A, lam, nullptr);
    stat_end(h, KC_APPLY_OBS, bytes, ev);
    CUDA_CHECK(cudaGetLastError());
  } else {
    ensure_partials(h, g);
    ensure_results(h, 1);
    stat_begin(h, KC_REDUCE, bytes, ev);
    k_csr<false><<<g, kThreads, 0, h->stream>>>(psi, A, nullptr, h->d_partials);
    stat_end(h, KC_REDUCE, bytes, ev);
    CUDA_CHECK(cudaGetLastError());
    sum_partials(h, h->d_partials, g, 1, h->d_results);
    CUDA_CHECK(cudaMemcpyAsync(&out, h->d_results, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  }
  CUDA_CHECK(cudaFreeAsync(buf, h->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->stream));
  return out;
}

double reduce_dot_re(sv_handle* h, const double2* a, const double2* b) {
  const unsigned g = red_grid(h->n_local);
  ensure_partials(h, g);
  ensure_results(h, 1);
  cudaEvent_t ev[2];
  stat_begin(h, KC_REDUCE, 32.0 * double(h->n_local), ev);
  k_dot_re<<<g, kThreads, 0, h->stream>>>(a, b, h->n_local, h->d_partials);
  stat_end(h, KC_REDUCE, 32.0 * double(h->n_local), ev);
  CUDA_CHECK(cudaGetLastError());
  sum_partials(h, h->d_partials, g, 1, h->d_results);
  double out = 0;
  CUDA_CHECK(cudaMemcpyAsync(&out, h->d_results, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->stream));
  return out;
}

void braket_prim_async(sv_handle* h, const double2* bra, const double2* ket, const Prim& gp, double* d_out) {
  if (gp.nb < 1 || gp.nb > 4) sv_fail(SV_ERR_UNSUPPORTED, "generator on more than 4 wires");
  DenseParams P;
  std::vector<double2> mat(gp.m.size());
  for (size_t i = 0; i < gp.m.size(); ++i) mat[i] = d2(gp.m[i]);
  P.mat = (const double2*)scratch_upload(h, mat.data(), mat.size() * sizeof(double2));
  P.fval = gp.fval;
  const int nf = popcount64(gp.fmask);
  P.count = h->n_local >> nf;
  P.k = gp.nb;
  for (int j = 0; j < gp.nb; ++j) P.pos[j] = (unsigned char)gp.pos[j];
  P.ins = make_ins(gp.fmask);
  const unsigned g = red_grid(P.count);
  ensure_partials(h, size_t(g) * 2);
  const double bytes = 32.0 * double(P.count << gp.nb);
  cudaEvent_t ev[2];
  stat_begin(h, KC_BRAKET, bytes, ev);
  switch (gp.nb) {
    case 1: k_braket<1><<<g, kThreads, 0, h->stream>>>(bra, ket, P, h->d_partials); break;
    case 2: k_braket<2><<<g, kThreads, 0, h->stream>>>(bra, ket, P, h->d_partials); break;
    case 3: k_braket<3><<<g, kThreads, 0, h->stream>>>(bra, ket, P, h->d_partials); break;
    default: k_braket<4><<<g, kThreads, 0, h->stream>>>(bra, ket, P, h->d_partials); break;
  }
  stat_end(h, KC_BRAKET, bytes, ev);
  CUDA_CHECK(cudaGetLastError());
  sum_partials(h, h->d_partials, g, 2, d_out);
}

void probs_async(sv_handle* h, const double2* a, const std::vector<int>& pos_msb_first, double* d_out) {
  ProbParams P;
  P.w = int(pos_msb_first.size());
  u64 wmask = 0;
  for (int j = 0; j < P.w; ++j) {
    P.pos[j] = (unsigned char)pos_msb_first[j];
    wmask |= 1ull << pos_msb_first[j];
  }
  P.ins = make_ins(wmask);
  P.members = h->n_local >> P.w;
  const u64 bins = 1ull << P.w;
  cudaEvent_t ev[2];
  stat_begin(h, KC_PROBS, 16.0 * double(h->n_local), ev);
  if (P.members <= 64) {
    k_probs_perbin<<<grid_for(bins, kThreads), kThreads, 0, h->stream>>>(a, P, bins, d_out);
    stat_end(h, KC_PROBS, 16.0 * double(h->n_local), ev);
    CUDA_CHECK(cudaGetLastError());
    return;
  }
  u64 chunks = std::max<u64>(1, std::min<u64>(u64(kRedBlocks) / bins, (P.members + kThreads - 1) / kThreads));
  const u64 nblk = bins * chunks;
  ensure_partials(h, nblk);
  k_probs_chunked<<<unsigned(nblk), kThreads, 0, h->stream>>>(a, P, int(chunks), h->d_partials);
  stat_end(h, KC_PROBS, 16.0 * double(h->n_local), ev);
  CUDA_CHECK(cudaGetLastError());
  sum_partials(h, h->d_partials, int(chunks), int(bins), d_out);
}
