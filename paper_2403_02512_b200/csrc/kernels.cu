// sm_100a kernels of libsvb200: one-op-per-pass gate kernels (K1-K6 of SURVEY.md §2.3),
// observable reductions (K8/K9/K12/K13), observable application (K10) and the generator
// bra-ket used by the adjoint sweep (K11).  Each is instantiated for complex128 (double2) and
// complex64 (float2, the reference's "f32" precision, state.py:20); in place, 64-bit indices; every kernel is an HBM streaming pass (~0.44 flop/B).
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

// Complex arithmetic in the state's precision.  complex128 states compute in FP64; complex64
// states (the reference's "f32" StateVector, state.py:20) compute gate updates in FP32 -- the
// reference casts the gate matrix to the state dtype before the contraction (state.py:264, 273)
// -- while every reduction widens to FP64 before accumulating.
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 c) {
  return make_float2(fmaf(a.x, b.x, fmaf(-a.y, b.y, c.x)), fmaf(a.x, b.y, fmaf(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 conjmul(double2 a, double2 b) {        // conj(a)*b
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ double2 wide(double2 v) { return v; }
__device__ __forceinline__ double2 wide(float2 v) { return make_double2(v.x, v.y); }
template <class C> __device__ __forceinline__ C narrow(double2 v);
template <> __device__ __forceinline__ double2 narrow<double2>(double2 v) { return v; }
template <> __device__ __forceinline__ float2 narrow<float2>(double2 v) {
  return make_float2(float(v.x), float(v.y));
}
template <class C> __device__ __forceinline__ C czero();
template <> __device__ __forceinline__ double2 czero<double2>() { return make_double2(0.0, 0.0); }
template <> __device__ __forceinline__ float2 czero<float2>() { return make_float2(0.f, 0.f); }

// ---------------------------------------------------------------------------
// K1/K2/K4: PAIR  (Alg. 1 / Alg. 2 generalised; 2x2 on (i0, i0^xmask))
// ---------------------------------------------------------------------------
template <class C>
struct PairParams {
  C m[4];
  u64 fval, xmask, count;
  Ins ins;
  int stream;   // state larger than L2: streaming (evict-first) stores, the state is not re-read soon
};

// store one amplitude (vector) -- streaming when the state does not fit L2 (K1-K4
// write the state once per gate; keeping it in L2 only evicts lines the next reads need)
template <class T>
__device__ __forceinline__ void st_amp(T* p, const T v, int stream) {
  if (stream) __stcs(p, v);
  else *p = v;
}

template <int ITEMS, class C>
__global__ void __launch_bounds__(kThreads) k_pair(C* __restrict__ a, const PairParams<C> P) {
  const u64 base = u64(blockIdx.x) * (ITEMS * kThreads) + threadIdx.x;
  u64 i0[ITEMS];
  C v0[ITEMS], v1[ITEMS];
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
    const C o0 = cfma(P.m[0], v0[j], cmul(P.m[1], v1[j]));
    const C o1 = cfma(P.m[2], v0[j], cmul(P.m[3], v1[j]));
    st_amp(&a[i0[j]], o0, P.stream);
    st_amp(&a[i0[j] ^ P.xmask], o1, P.stream);
  }
}

// complex64 PAIR with bit 0 free: the two pairs at counters 2m, 2m+1 are adjacent in memory
// (i0 even), so one 16-byte float4 access moves two amplitudes -- the same access width as
// the complex128 kernel (a float2 per access only reaches ~90 % of the copy roofline).
template <int ITEMS>
__global__ void __launch_bounds__(kThreads) k_pair_v2(float2* __restrict__ a, const PairParams<float2> P) {
  const u64 base = u64(blockIdx.x) * (ITEMS * kThreads) + threadIdx.x;
  const u64 count2 = P.count >> 1;
  float4* a4 = reinterpret_cast<float4*>(a);
  u64 i0[ITEMS];
  float4 v0[ITEMS], v1[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const u64 k = base + u64(j) * kThreads;
    i0[j] = (k < count2) ? (deposit(k << 1, P.ins) | P.fval) : ~0ull;
    if (i0[j] != ~0ull) {
      v0[j] = a4[i0[j] >> 1];
      v1[j] = a4[(i0[j] ^ P.xmask) >> 1];
    }
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (i0[j] == ~0ull) continue;
    const float2 x0 = make_float2(v0[j].x, v0[j].y), y0 = make_float2(v0[j].z, v0[j].w);
    const float2 x1 = make_float2(v1[j].x, v1[j].y), y1 = make_float2(v1[j].z, v1[j].w);
    const float2 ox0 = cfma(P.m[0], x0, cmul(P.m[1], x1)), oy0 = cfma(P.m[0], y0, cmul(P.m[1], y1));
    const float2 ox1 = cfma(P.m[2], x0, cmul(P.m[3], x1)), oy1 = cfma(P.m[2], y0, cmul(P.m[3], y1));
    st_amp(&a4[i0[j] >> 1], make_float4(ox0.x, ox0.y, oy0.x, oy0.y), P.stream);
    st_amp(&a4[(i0[j] ^ P.xmask) >> 1], make_float4(ox1.x, ox1.y, oy1.x, oy1.y), P.stream);
  }
}

// ---------------------------------------------------------------------------
// K3: DIAG  (a[i] *= table[bits]; restricted to (i & fmask) == fval)
// ---------------------------------------------------------------------------
template <class C>
struct DiagParams {
  C t[64];
  u64 fval, count;
  int nb;
  int stream;
  unsigned char pos[6];
  Ins ins;
};

template <int ITEMS, class C>
__global__ void __launch_bounds__(kThreads) k_diag(C* __restrict__ a, const DiagParams<C> P) {
  const u64 base = u64(blockIdx.x) * (ITEMS * kThreads) + threadIdx.x;
  u64 idx[ITEMS];
  C v[ITEMS];
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
    st_amp(&a[idx[j]], cmul(P.t[t], v[j]), P.stream);
  }
}

// complex64 DIAG with bit 0 free: two adjacent amplitudes per float4 access (see k_pair_v2)
template <int ITEMS>
__global__ void __launch_bounds__(kThreads) k_diag_v2(float2* __restrict__ a, const DiagParams<float2> P) {
  const u64 base = u64(blockIdx.x) * (ITEMS * kThreads) + threadIdx.x;
  const u64 count2 = P.count >> 1;
  float4* a4 = reinterpret_cast<float4*>(a);
  u64 idx[ITEMS];
  float4 v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const u64 k = base + u64(j) * kThreads;
    idx[j] = (k < count2) ? (deposit(k << 1, P.ins) | P.fval) : ~0ull;
    if (idx[j] != ~0ull) v[j] = a4[idx[j] >> 1];
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (idx[j] == ~0ull) continue;
    int t = 0;
    for (int b = 0; b < P.nb; ++b) t |= int((idx[j] >> P.pos[b]) & 1ull) << b;
    int t1 = t;
    for (int b = 0; b < P.nb; ++b)
      if (P.pos[b] == 0) t1 |= 1 << b;   // the odd amplitude has bit 0 set
    const float2 o0 = cmul(P.t[t], make_float2(v[j].x, v[j].y));
    const float2 o1 = cmul(P.t[t1], make_float2(v[j].z, v[j].w));
    st_amp(&a4[idx[j] >> 1], make_float4(o0.x, o0.y, o1.x, o1.y), P.stream);
  }
}

// ---------------------------------------------------------------------------
// K5/K6: DENSE k-qubit (matrix in shared memory; amplitudes in registers for k <= 4)
// ---------------------------------------------------------------------------
struct DenseParams {
  const void* mat;       // 4^k entries (state precision; double2 for the bra-ket), row-major, bit j <-> pos[j]
  u64 fval, count;
  int k;
  unsigned char pos[16];
  Ins ins;
};

template <int K, class C>
__global__ void __launch_bounds__(kThreads) k_dense(C* __restrict__ a, const DenseParams P) {
  constexpr int D = 1 << K;
  __shared__ C M[D * D];
  const C* mat = static_cast<const C*>(P.mat);
  for (int i = threadIdx.x; i < D * D; i += kThreads) M[i] = mat[i];
  __syncthreads();
  const u64 k = u64(blockIdx.x) * kThreads + threadIdx.x;
  if (k >= P.count) return;
  const u64 base = deposit(k, P.ins) | P.fval;
  u64 off[D];
  C v[D];
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
    C acc = czero<C>();
#pragma unroll
    for (int c = 0; c < D; ++c) acc = cfma(M[r * D + c], v[c], acc);
    a[off[r]] = acc;
  }
}

// k >= 5: one block per group, amplitudes staged in shared memory, one warp per output row.
template <class C>
__global__ void __launch_bounds__(kThreads) k_dense_big(C* __restrict__ a, const DenseParams P) {
  extern __shared__ __align__(16) unsigned char dense_smem[];
  const int D = 1 << P.k;
  C* in = reinterpret_cast<C*>(dense_smem);
  C* out = in + D;
  const C* mat = static_cast<const C*>(P.mat);
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
      C acc = czero<C>();
      const C* row = mat + size_t(r) * D;
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

template <class C>
__global__ void __launch_bounds__(kThreads) k_norm2(const C* __restrict__ a, u64 n, double* __restrict__ partials) {
  double v[1] = {0.0};
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    const double2 x = wide(a[i]);
    v[0] = fma(x.x, x.x, fma(x.y, x.y, v[0]));
  }
  block_reduce_store<1>(v, partials);
}

// Re <a|b> partials (K12)
template <class C>
__global__ void __launch_bounds__(kThreads) k_dot_re(const C* __restrict__ a, const C* __restrict__ b, u64 n,
                                                     double* __restrict__ partials) {
  double v[1] = {0.0};
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    const double2 x = wide(a[i]), y = wide(b[i]);
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
template <bool APPLY, class C>
__global__ void __launch_bounds__(kThreads) k_csr(const C* __restrict__ psi, const CsrArgs A,
                                                  C* __restrict__ lam, double* __restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (kThreads / 32);
  double v[1] = {0.0};
  for (u64 row = u64(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5); row < A.rows; row += warps) {
    double ax = 0.0, ay = 0.0;
    for (int64_t k = A.indptr[row] + lane; k < A.indptr[row + 1]; k += 32) {
      const double2 m = A.data[k];
      const double2 x = wide(psi[to_phys(u64(A.indices[k]), A.perm_tab)]);
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
        lam[pr] = narrow<C>(make_double2(ax, ay));
      } else {
        const double2 p = wide(psi[pr]);
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

template <class C, int PF>
__global__ void __launch_bounds__(kThreads) k_pauli_apply_multi(const C* __restrict__ psi, C* __restrict__ lam,
                                                                u64 n, const PauliGroupsArgs G,
                                                                const PauliApplyTermDev* __restrict__ terms, int nterms,
                                                                int accumulate) {
  extern __shared__ PauliApplyTermDev sat2[];
  for (int t = threadIdx.x; t < nterms; t += kThreads) sat2[t] = terms[t];
  __syncthreads();
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    double2 o = accumulate ? wide(lam[i]) : make_double2(0.0, 0.0);
    if (PF) {
      // every group's gather issued before any arithmetic: kMaxXG loads in flight per thread
      // (the gathers are L2 hits in x-mask order; one at a time they were latency-bound)
      double2 b[kMaxXG];
#pragma unroll
      for (int g = 0; g < kMaxXG; ++g)
        if (g < G.ng) b[g] = wide(psi[i ^ G.x[g]]);
#pragma unroll
      for (int g = 0; g < kMaxXG; ++g) {
        if (g >= G.ng) break;
        const u64 j = i ^ G.x[g];
        double2 s = make_double2(0.0, 0.0);
        for (int t = G.t_begin[g]; t < G.t_begin[g + 1]; ++t) {
          const double sg = (__popcll(j & sat2[t].z) & 1) ? -1.0 : 1.0;
          s.x = fma(sg, sat2[t].cc.x, s.x);
          s.y = fma(sg, sat2[t].cc.y, s.y);
        }
        o = cfma(s, b[g], o);
      }
    } else {
      for (int g = 0; g < G.ng; ++g) {
        const u64 j = i ^ G.x[g];
        const double2 b = wide(psi[j]);
        double2 s = make_double2(0.0, 0.0);
        for (int t = G.t_begin[g]; t < G.t_begin[g + 1]; ++t) {
          const double sg = (__popcll(j & sat2[t].z) & 1) ? -1.0 : 1.0;
          s.x = fma(sg, sat2[t].cc.x, s.x);
          s.y = fma(sg, sat2[t].cc.y, s.y);
        }
        o = cfma(s, b, o);
      }
    }
    lam[i] = narrow<C>(o);
  }
}

// Batched expectation of up to kMaxXG non-diagonal x-groups: sum_i Re(conj(psi_i) (H_batch psi)_i)
// with (H_batch psi)_i formed in registers exactly as k_pauli_apply_multi forms lambda_i (in x-mask
// order the gathers are L2 hits), so DRAM reads psi about once per batch instead of once per
// x-group; nothing is written.
template <class C>
__global__ void __launch_bounds__(kThreads) k_pauli_expval_multi(const C* __restrict__ psi, u64 n, const PauliGroupsArgs G,
                                                                 const PauliApplyTermDev* __restrict__ terms, int nterms,
                                                                 double* __restrict__ partials) {
  extern __shared__ PauliApplyTermDev sat3[];
  for (int t = threadIdx.x; t < nterms; t += kThreads) sat3[t] = terms[t];
  __syncthreads();
  double v[1] = {0.0};
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    const double2 a = wide(psi[i]);
    double2 o = make_double2(0.0, 0.0);
    for (int g = 0; g < G.ng; ++g) {
      const u64 j = i ^ G.x[g];
      const double2 b = wide(psi[j]);
      double2 s = make_double2(0.0, 0.0);
      for (int t = G.t_begin[g]; t < G.t_begin[g + 1]; ++t) {
        const double sg = (__popcll(j & sat3[t].z) & 1) ? -1.0 : 1.0;
        s.x = fma(sg, sat3[t].cc.x, s.x);
        s.y = fma(sg, sat3[t].cc.y, s.y);
      }
      o = cfma(s, b, o);
    }
    v[0] = fma(a.x, o.x, fma(a.y, o.y, v[0]));   // Re(conj(a) o)
  }
  block_reduce_store<1>(v, partials);
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

template <class C>
__global__ void __launch_bounds__(kThreads) k_pauli_expval(const C* __restrict__ a, u64 xmask, int pivot, u64 count,
                                                           const PauliTermDev* __restrict__ terms, int nterms,
                                                           double* __restrict__ partials) {
  extern __shared__ PauliTermDev st[];
  for (int t = threadIdx.x; t < nterms; t += kThreads) st[t] = terms[t];
  __syncthreads();
  double v[1] = {0.0};
  for (u64 k = u64(blockIdx.x) * kThreads + threadIdx.x; k < count; k += u64(gridDim.x) * kThreads) {
    if (xmask == 0) {
      const double2 x = wide(a[k]);
      const double p = fma(x.x, x.x, x.y * x.y);
      double s = 0.0;
      for (int t = 0; t < nterms; ++t) s += (__popcll(k & st[t].z) & 1) ? -st[t].r : st[t].r;
      v[0] = fma(p, s, v[0]);
    } else {
      const u64 lo = k & ((1ull << pivot) - 1ull);
      const u64 i = ((k ^ lo) << 1) | lo;
      const double2 ai = wide(a[i]), aj = wide(a[i ^ xmask]);
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

// Diagonal (x = 0) Pauli group with many Z terms: f(i) = sum_t r_t (-1)^{pc(i & z_t)} per amplitude
// costs nterms 64-bit POPCs, which bounds the plain kernel far below HBM (33q MaxCut, 66 ZZ terms:
// 0.32 s for one 137 GB read).  Per 4096-amplitude tile (fixed high bits H) f restricted to the low
// 12 bits is the Walsh-Hadamard transform of C_H[m] = sum_{t: z_t & 4095 = m} r_t (-1)^{pc(H & z_t)}
// (terms pre-grouped by low mask on the host, deterministic), so a tile costs ngroups term sums
// plus a 12-stage WHT: stages 0-3 in registers (thread owns L = tid*16 + j), 4-8 by warp shuffles,
// one swizzled shared-memory transpose, stages 9-11 in registers (thread owns L = b0 | tid<<1 |
// b9..11<<9, read as 32-byte amplitude pairs).  HBM-bound.
constexpr int kWhtBits = 12;
struct DiagGroupDev {
  unsigned zlo;     // low 12 bits of the group's z masks
  int first, last;  // term range [first, last)
};
struct DiagTermDev {
  u64 zhi;          // z mask without the low 12 bits
  double r;
};
__device__ __forceinline__ int wht_swz(int L) {   // double index -> swizzled double index
  const int c = L >> 1;
  return ((c ^ ((c >> 3) & 7)) << 1) | (L & 1);
}

template <class C>
__global__ void __launch_bounds__(kThreads, 2) k_pauli_diag_wht(const C* __restrict__ a, C* __restrict__ out, u64 ntiles,
                                                             const DiagGroupDev* __restrict__ groups, int ngroups,
                                                             const DiagTermDev* __restrict__ terms,
                                                             double* __restrict__ partials, double init_scale = 0.0) {
  // init_scale != 0 (K14): out = init_scale * exp(i f), write-only -- H on every qubit of |0...0>
  // followed by a run of diagonal gates, f = the Walsh expansion of the gates' phases
  const bool init = init_scale != 0.0;
  __shared__ __align__(16) double T[1 << kWhtBits];
  const int tid = threadIdx.x, lane = tid & 31;
  double acc[1] = {0.0};
  for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const u64 H = tile << kWhtBits;
    // amplitudes of layout B, issued first and consumed last so the loads overlap the transform;
    // the next tile is prefetched into L2 (two 128-byte lines per thread)
    C x[16];
    if (!init) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const u64 L = (u64(tid) << 1) | (u64(q) << 9);
        x[2 * q] = a[H + L];
        x[2 * q + 1] = a[H + L + 1];
      }
    }
    if (!init && tile + gridDim.x < ntiles) {
      const char* nxt = reinterpret_cast<const char*>(a + ((tile + gridDim.x) << kWhtBits));
      const size_t per_thread = (size_t(1) << kWhtBits) * sizeof(C) / kThreads;   // 256 B (c128) / 128 B (c64)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(nxt + tid * per_thread));
      if (per_thread > 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(nxt + tid * per_thread + 128));
    }
    // C_H scattered into the (swizzled) table
#pragma unroll
    for (int j = 0; j < 16; ++j) T[tid + j * kThreads] = 0.0;   // all entries, conflict-free
    __syncthreads();
    for (int g = tid; g < ngroups; g += kThreads) {
      double c = 0.0;
      for (int t = groups[g].first; t < groups[g].last; ++t)
        c += (__popcll(H & terms[t].zhi) & 1) ? -terms[t].r : terms[t].r;
      T[wht_swz(int(groups[g].zlo))] = c;
    }
    __syncthreads();
    // layout A: L = tid*16 + j
    double v[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {   // 16-byte accesses: conflict-free per quarter warp with the swizzle
      const double2 t2 = *reinterpret_cast<const double2*>(&T[wht_swz((tid << 4) | (2 * q))]);
      v[2 * q] = t2.x;
      v[2 * q + 1] = t2.y;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (!(j & (1 << b))) {
          const double x = v[j], y = v[j | (1 << b)];
          v[j] = x + y;
          v[j | (1 << b)] = x - y;
        }
#pragma unroll
    for (int b = 0; b < 5; ++b) {
      const bool up = (lane >> b) & 1;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const double o = __shfl_xor_sync(0xffffffffu, v[j], 1 << b);
        v[j] = up ? o - v[j] : v[j] + o;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)   // own entries: no hazard
      *reinterpret_cast<double2*>(&T[wht_swz((tid << 4) | (2 * q))]) = make_double2(v[2 * q], v[2 * q + 1]);
    __syncthreads();
    // layout B: register j' = b0 | (b9..11 << 1)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int L = (tid << 1) | (q << 9);
      const double2 t2 = *reinterpret_cast<const double2*>(&T[wht_swz(L)]);
      v[2 * q] = t2.x;
      v[2 * q + 1] = t2.y;
    }
#pragma unroll
    for (int b = 1; b < 4; ++b)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (!(j & (1 << b))) {
          const double x = v[j], y = v[j | (1 << b)];
          v[j] = x + y;
          v[j | (1 << b)] = x - y;
        }
    if (init) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const u64 L = (u64(tid) << 1) | (u64(q) << 9);
        double s0, c0, s1, c1;
        sincos(v[2 * q], &s0, &c0);
        sincos(v[2 * q + 1], &s1, &c1);
        __stcs(reinterpret_cast<double2*>(out) + H + L, make_double2(init_scale * c0, init_scale * s0));
        __stcs(reinterpret_cast<double2*>(out) + H + L + 1, make_double2(init_scale * c1, init_scale * s1));
      }
    } else if (out) {   // lambda = f psi (the adjoint's lambda initialisation, K10 for one diagonal group)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const u64 L = (u64(tid) << 1) | (u64(q) << 9);
        const double2 w0 = wide(x[2 * q]), w1 = wide(x[2 * q + 1]);
        out[H + L] = narrow<C>(make_double2(v[2 * q] * w0.x, v[2 * q] * w0.y));
        out[H + L + 1] = narrow<C>(make_double2(v[2 * q + 1] * w1.x, v[2 * q + 1] * w1.y));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const double2 w = wide(x[j]);
        acc[0] = fma(fma(w.x, w.x, w.y * w.y), v[j], acc[0]);
      }
    }
    __syncthreads();   // the next tile rewrites T
  }
  if (!out) block_reduce_store<1>(acc, partials);
}

// K10: lambda (+)= sum_t cc_t (-1)^{pc((i^x) & z_t)} psi_{i^x}   (PauliApplyTermDev: see above)

template <class C>
__global__ void __launch_bounds__(kThreads) k_pauli_apply(const C* __restrict__ psi, C* __restrict__ lam, u64 xmask,
                                                          u64 n, const PauliApplyTermDev* __restrict__ terms, int nterms,
                                                          int accumulate) {
  extern __shared__ PauliApplyTermDev sat[];
  for (int t = threadIdx.x; t < nterms; t += kThreads) sat[t] = terms[t];
  __syncthreads();
  for (u64 i = u64(blockIdx.x) * kThreads + threadIdx.x; i < n; i += u64(gridDim.x) * kThreads) {
    const u64 j = i ^ xmask;
    const double2 b = wide(psi[j]);
    double2 s = make_double2(0.0, 0.0);
    for (int t = 0; t < nterms; ++t) {
      const double sg = (__popcll(j & sat[t].z) & 1) ? -1.0 : 1.0;
      s.x = fma(sg, sat[t].cc.x, s.x);
      s.y = fma(sg, sat[t].cc.y, s.y);
    }
    double2 o = cmul(s, b);
    if (accumulate) {
      const double2 l = wide(lam[i]);
      o.x += l.x;
      o.y += l.y;
    }
    lam[i] = narrow<C>(o);
  }
}

// K11 helper: <bra| P (G (x) I) |ket> over groups (complex partial), G dense 2^K x 2^K in smem
// (always FP64: the bra-ket is a reduction, so complex64 states widen on load).
template <int K, class C>
__global__ void __launch_bounds__(kThreads) k_braket(const C* __restrict__ bra, const C* __restrict__ ket,
                                                     const DenseParams P, double* __restrict__ partials) {
  constexpr int D = 1 << K;
  __shared__ double2 M[D * D];
  const double2* mat = static_cast<const double2*>(P.mat);
  for (int i = threadIdx.x; i < D * D; i += kThreads) M[i] = mat[i];
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
      x[r] = wide(ket[off[r]]);
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < D; ++c) acc = cfma(M[r * D + c], x[c], acc);
      const double2 b = wide(bra[off[r]]);
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
template <class C>
__global__ void __launch_bounds__(kThreads) k_probs_chunked(const C* __restrict__ a, const ProbParams P, int chunks,
                                                            double* __restrict__ partials) {
  const u64 bins = 1ull << P.w;
  const u64 bin = blockIdx.x % bins;
  const int chunk = int(blockIdx.x / bins);
  const u64 pat = bin_pattern(bin, P);
  double v[1] = {0.0};
  for (u64 k = u64(chunk) * kThreads + threadIdx.x; k < P.members; k += u64(chunks) * kThreads) {
    const double2 x = wide(a[deposit(k, P.ins) | pat]);
    v[0] = fma(x.x, x.x, fma(x.y, x.y, v[0]));
  }
  block_reduce_store<1>(v, partials);
}

// one thread per bin (few members per bin)
template <class C>
__global__ void __launch_bounds__(kThreads) k_probs_perbin(const C* __restrict__ a, const ProbParams P, u64 bins,
                                                           double* __restrict__ out) {
  const u64 bin = u64(blockIdx.x) * kThreads + threadIdx.x;
  if (bin >= bins) return;
  const u64 pat = bin_pattern(bin, P);
  double s = 0.0;
  for (u64 k = 0; k < P.members; ++k) {
    const double2 x = wide(a[deposit(k, P.ins) | pat]);
    s = fma(x.x, x.x, fma(x.y, x.y, s));
  }
  out[bin] = s;
}

// Global-qubit swap over peer memory: a[i] <-> b[i] with b on the partner GPU (NVLink P2P).
// Each thread keeps 4 local and 4 remote 16-byte loads in flight (remote latency ~1-2 us).
__global__ void __launch_bounds__(kThreads) k_exchange(double2* __restrict__ a, double2* __restrict__ b, u64 n) {
  constexpr int IT = 4;
  const u64 stride = u64(gridDim.x) * kThreads * IT;
  for (u64 base = u64(blockIdx.x) * kThreads * IT + threadIdx.x; base < n; base += stride) {
    double2 x[IT], y[IT];
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const u64 i = base + u64(j) * kThreads;
      if (i < n) {
        x[j] = a[i];
        y[j] = b[i];
      }
    }
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const u64 i = base + u64(j) * kThreads;
      if (i < n) {
        a[i] = y[j];
        b[i] = x[j];
      }
    }
  }
  __threadfence_system();   // remote stores visible before the post-swap barrier
}

// Multi-bit qubit-index exchange over peer memory (dist.cpp exchange_bits): the victim local bits
// (vdep) of element i spell the partner c; element i swaps with element (i's base | gdep) of
// partner c's state.  Each pair of ranks splits its pairs on one free local bit (own[c]).  The
// counter t enumerates the local bits that are neither victims nor the split bit; consecutive t
// are consecutive amplitudes when those bits are the low ones, so every access is a full sector.
struct XchgParams {
  double2* peer[8];
  u64 vdep[8];
  u64 own[8];
  u64 gdep;
  u64 count;
  Ins ins;
  int nc;
};

template <int IT>   // IT local + IT remote 16-byte loads in flight per thread and partner
__global__ void __launch_bounds__(kThreads) k_exchange_multi(double2* __restrict__ a, const XchgParams P) {
  const u64 stride = u64(gridDim.x) * kThreads * IT;
  for (u64 t0 = u64(blockIdx.x) * kThreads * IT + threadIdx.x; t0 < P.count; t0 += stride) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c >= P.nc || !P.peer[c]) continue;
      double2 x[IT], y[IT];
      u64 il[IT], ir[IT];
#pragma unroll
      for (int j = 0; j < IT; ++j) {
        const u64 t = t0 + u64(j) * kThreads;
        if (t < P.count) {
          const u64 b = deposit(t, P.ins) | P.own[c];
          il[j] = b | P.vdep[c];
          ir[j] = b | P.gdep;
          x[j] = a[il[j]];
          y[j] = P.peer[c][ir[j]];
        }
      }
#pragma unroll
      for (int j = 0; j < IT; ++j) {
        const u64 t = t0 + u64(j) * kThreads;
        if (t < P.count) {
          a[il[j]] = y[j];
          P.peer[c][ir[j]] = x[j];
        }
      }
    }
  }
  __threadfence_system();   // remote stores visible before the post-exchange barrier
}

// NCCL fallback of the same exchange: gather / scatter the elements whose victim bits spell one
// partner (counter t over the non-victim bits, the same order on both ranks) through staging.
__global__ void __launch_bounds__(kThreads) k_pack_sel(const double2* __restrict__ a, double2* __restrict__ out,
                                                      const Ins ins, u64 vdep, u64 t_begin, u64 n, int unpack) {
  for (u64 t = u64(blockIdx.x) * kThreads + threadIdx.x; t < n; t += u64(gridDim.x) * kThreads) {
    const u64 i = deposit(t_begin + t, ins) | vdep;
    if (unpack) const_cast<double2*>(a)[i] = out[t];
    else out[t] = a[i];
  }
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
template <class C> C hc(cplx c);
template <> double2 hc<double2>(cplx c) { return d2(c); }
template <> float2 hc<float2>(cplx c) { return make_float2(float(c.real()), float(c.imag())); }

// launch KERNEL<C> on a state buffer in the handle's precision (double2* in the host API)
#define SV_F32(p) reinterpret_cast<float2*>(const_cast<double2*>(p))
#define SV_LAUNCH(h, KERNEL, CFG, A0, ...)                        \
  do {                                                            \
    if ((h)->prec == 32)                                          \
      KERNEL<float2><<<CFG>>>(SV_F32(A0), __VA_ARGS__);           \
    else                                                          \
      KERNEL<double2><<<CFG>>>(A0, __VA_ARGS__);                  \
  } while (0)
#define SV_LAUNCH2(h, KERNEL, CFG, A0, A1, ...)                   \
  do {                                                            \
    if ((h)->prec == 32)                                          \
      KERNEL<float2><<<CFG>>>(SV_F32(A0), SV_F32(A1), __VA_ARGS__); \
    else                                                          \
      KERNEL<double2><<<CFG>>>(A0, A1, __VA_ARGS__);              \
  } while (0)
#define SV_CFG(...) __VA_ARGS__

// device buffer for small per-launch tables (matrices, term lists); grows, never shrinks
void* scratch_upload(sv_handle* h, const void* src, size_t bytes);

}  // namespace

// ===========================================================================
// host launchers
// ===========================================================================
const char* kKernelClassNames[KC_COUNT] = {"pair", "diag", "dense", "fused_tile", "reduce", "apply_obs",
                                           "braket", "probs", "init", "swap"};

namespace {
// ring of 64 buffers in the handle so back-to-back async uploads do not overwrite in-flight tables
// (callers hold the handle's mutex: one mutator per handle)
void* scratch_upload(sv_handle* h, const void* src, size_t bytes) {
  sv_handle::ScratchBuf& b = h->scratch[h->scratch_slot];
  h->scratch_slot = (h->scratch_slot + 1) % 64;
  if (b.cap < bytes) {
    if (b.ptr) {
      stream_sync(h);
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
  for (auto& b : h->scratch) {
    if (b.ptr) cudaFree(b.ptr);
    b.ptr = nullptr;
    b.cap = 0;
  }
}

// Algorithmic bytes of one unfused primitive: 32 B (16 read + 16 written) per touched amplitude.
double prim_bytes(const sv_handle* h, const Prim& p) {
  if (p.skip) return 0.0;
  const double rw = 2.0 * double(amp_bytes(h));   // read + write of one amplitude
  if (p.type == PRIM_PAIR) return rw * 2.0 * double(h->n_local >> popcount64(p.fmask));
  if (p.type == PRIM_DIAG) return rw * double(h->n_local >> popcount64(p.fmask));
  return rw * double(h->n_local >> (popcount64(p.fmask) - p.nb));
}

template <class C>
static void launch_prim_t(sv_handle* h, C* a, const Prim& p) {
  // the same bytes in flight per thread in both precisions (4 x 16 B pairs or 8 x 8 B pairs)
  constexpr int kItems = sizeof(C) == 8 ? 8 : 4;
  const int nf = popcount64(p.fmask);
  if (nf > h->nl) sv_fail(SV_ERR_DEVICE, "internal: primitive fixes more bits than the shard has");
  const u64 count = h->n_local >> nf;
  const int stream = double(h->n_local) * sizeof(C) > 256.0 * (1 << 20) ? 1 : 0;   // state >> 126 MB L2
  cudaEvent_t ev[2];
  if (p.type == PRIM_PAIR) {
    PairParams<C> P;
    P.stream = stream;
    for (int i = 0; i < 4; ++i) P.m[i] = hc<C>(p.m[i]);
    P.fval = p.fval;
    P.xmask = p.xmask;
    P.count = count;
    P.ins = make_ins(p.fmask);
    stat_begin(h, KC_PAIR, prim_bytes(h, p), ev);
    if constexpr (sizeof(C) == 8) {
      if (!(p.fmask & 1ull) && count >= 2)
        k_pair_v2<4><<<grid_for(count >> 1, 4 * kThreads), kThreads, 0, h->stream>>>(a, P);
      else
        k_pair<kItems, C><<<grid_for(count, kItems * kThreads), kThreads, 0, h->stream>>>(a, P);
    } else {
      k_pair<kItems, C><<<grid_for(count, kItems * kThreads), kThreads, 0, h->stream>>>(a, P);
    }
    stat_end(h, KC_PAIR, prim_bytes(h, p), ev);
  } else if (p.type == PRIM_DIAG) {
    DiagParams<C> P;
    P.stream = stream;
    if (p.nb > 6) sv_fail(SV_ERR_DEVICE, "internal: diagonal table too large");
    for (size_t i = 0; i < p.m.size(); ++i) P.t[i] = hc<C>(p.m[i]);
    P.fval = p.fval;
    P.count = count;
    P.nb = p.nb;
    for (int j = 0; j < p.nb; ++j) P.pos[j] = (unsigned char)p.pos[j];
    P.ins = make_ins(p.fmask);
    stat_begin(h, KC_DIAG, prim_bytes(h, p), ev);
    if constexpr (sizeof(C) == 8) {
      if (!(p.fmask & 1ull) && count >= 2)
        k_diag_v2<4><<<grid_for(count >> 1, 4 * kThreads), kThreads, 0, h->stream>>>(a, P);
      else
        k_diag<kItems, C><<<grid_for(count, kItems * kThreads), kThreads, 0, h->stream>>>(a, P);
    } else {
      k_diag<kItems, C><<<grid_for(count, kItems * kThreads), kThreads, 0, h->stream>>>(a, P);
    }
    stat_end(h, KC_DIAG, prim_bytes(h, p), ev);
  } else {
    DenseParams P;
    std::vector<C> mat(p.m.size());
    for (size_t i = 0; i < p.m.size(); ++i) mat[i] = hc<C>(p.m[i]);
    P.mat = scratch_upload(h, mat.data(), mat.size() * sizeof(C));
    P.fval = p.fval;
    P.count = count;
    P.k = p.nb;
    for (int j = 0; j < p.nb; ++j) P.pos[j] = (unsigned char)p.pos[j];
    P.ins = make_ins(p.fmask);
    stat_begin(h, KC_DENSE, prim_bytes(h, p), ev);
    const unsigned g = grid_for(count, kThreads);
    switch (p.nb) {
      case 1: k_dense<1, C><<<g, kThreads, 0, h->stream>>>(a, P); break;
      case 2: k_dense<2, C><<<g, kThreads, 0, h->stream>>>(a, P); break;
      case 3: k_dense<3, C><<<g, kThreads, 0, h->stream>>>(a, P); break;
      case 4: k_dense<4, C><<<g, kThreads, 0, h->stream>>>(a, P); break;
      default: {
        if (p.nb > 12) sv_fail(SV_ERR_UNSUPPORTED, "dense matrices on more than 12 wires are not supported on the GPU path");
        const size_t smem = (size_t(2) << p.nb) * sizeof(C);   // in + out, 2^k each
        if (smem > 48 * 1024)
          CUDA_CHECK(cudaFuncSetAttribute(k_dense_big<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        unsigned gb = unsigned(std::min<u64>(count, 148ull * 16));
        k_dense_big<C><<<gb, kThreads, smem, h->stream>>>(a, P);
      }
    }
    stat_end(h, KC_DENSE, prim_bytes(h, p), ev);
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_prim(sv_handle* h, double2* a, const Prim& p) {
  if (p.skip) return;
  if (h->recording) {   // host-only planning (sv_plan_sharded)
    h->rec.push_back({REC_PRIM, p, -1});
    return;
  }
  if (h->prec == 32)
    launch_prim_t(h, reinterpret_cast<float2*>(a), p);
  else
    launch_prim_t(h, a, p);
}

void launch_init_zero(sv_handle* h, double2* a, u64 basis_local, bool set_one) {
  cudaEvent_t ev[2];
  stat_begin(h, KC_INIT, double(amp_bytes(h)) * double(h->n_local), ev);
  const size_t eb = amp_bytes(h);
  CUDA_CHECK(cudaMemsetAsync(a, 0, h->n_local * eb, h->stream));
  if (set_one) {
    static const double2 one = {1.0, 0.0};
    static const float2 one32 = {1.f, 0.f};
    const void* src = h->prec == 32 ? static_cast<const void*>(&one32) : static_cast<const void*>(&one);
    CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(a) + basis_local * eb, src, eb, cudaMemcpyHostToDevice, h->stream));
  }
  stat_end(h, KC_INIT, double(amp_bytes(h)) * double(h->n_local), ev);
}

void launch_copy(sv_handle* h, double2* dst, const double2* src, u64 n) {
  cudaEvent_t ev[2];
  const size_t eb = amp_bytes(h);
  stat_begin(h, KC_INIT, 2.0 * double(eb) * double(n), ev);
  CUDA_CHECK(cudaMemcpyAsync(dst, src, n * eb, cudaMemcpyDeviceToDevice, h->stream));
  stat_end(h, KC_INIT, 2.0 * double(eb) * double(n), ev);
}

void launch_exchange(sv_handle* h, double2* a, double2* b, u64 n) {
  if (n == 0) return;
  const unsigned g = unsigned(std::min<u64>(grid_for(n, kThreads * 4), 148ull * 8));
  k_exchange<<<g, kThreads, 0, h->stream>>>(a, b, n);
  h->launches++;
  CUDA_CHECK(cudaGetLastError());
}

void launch_exchange_multi(sv_handle* h, double2* a, double2* const* peer_by_c, const u64* vdep, const u64* own, u64 gdep,
                           int nc, u64 split_fmask, u64 count) {
  if (count == 0) return;
  XchgParams P;
  std::memset(&P, 0, sizeof(P));
  for (int c = 0; c < nc; ++c) {
    P.peer[c] = peer_by_c[c];
    P.vdep[c] = vdep[c];
    P.own[c] = own[c];
  }
  P.gdep = gdep;
  P.count = count;
  P.nc = nc;
  P.ins = make_ins(split_fmask);
  // SVB200_XCHG_IT: loads in flight per thread and partner (4 default; 8 measured for A/B)
  static const int it = getenv("SVB200_XCHG_IT") ? atoi(getenv("SVB200_XCHG_IT")) : 4;
  const unsigned g = unsigned(std::min<u64>(grid_for(count, kThreads * it), 148ull * 8));
  if (it == 8) k_exchange_multi<8><<<g, kThreads, 0, h->stream>>>(a, P);
  else if (it == 2) k_exchange_multi<2><<<g, kThreads, 0, h->stream>>>(a, P);
  else k_exchange_multi<4><<<g, kThreads, 0, h->stream>>>(a, P);
  h->launches++;
  CUDA_CHECK(cudaGetLastError());
}

void launch_pack_sel(sv_handle* h, double2* a, double2* buf, u64 victim_mask, u64 vdep, u64 t_begin, u64 n, bool unpack) {
  if (n == 0) return;
  const unsigned g = unsigned(std::min<u64>(grid_for(n, kThreads), 148ull * 16));
  k_pack_sel<<<g, kThreads, 0, h->stream>>>(a, buf, make_ins(victim_mask), vdep, t_begin, n, unpack ? 1 : 0);
  h->launches++;
  CUDA_CHECK(cudaGetLastError());
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
  stat_begin(h, KC_REDUCE, double(amp_bytes(h)) * double(h->n_local), ev);
  SV_LAUNCH(h, k_norm2, SV_CFG(g, kThreads, 0, h->stream), a, h->n_local, h->d_partials);
  stat_end(h, KC_REDUCE, double(amp_bytes(h)) * double(h->n_local), ev);
  CUDA_CHECK(cudaGetLastError());
  sum_partials(h, h->d_partials, g, 1, h->d_results);
  double out = 0;
  d2h(h, &out, h->d_results, sizeof(double));
  return out;
}

// Diagonal group through k_pauli_diag_wht: out == nullptr -> per-block partials of
// sum_i |psi_i|^2 f(i) (returns the grid); otherwise out = f psi.  Terms are grouped by their low
// 12 mask bits on the host (fixed order -> deterministic sums); real coefficients only.
static unsigned pauli_diag_wht(sv_handle* h, const double2* a, double2* out, const std::vector<PauliTerm>& terms,
                               double init_scale = 0.0) {
  const u64 lo = (u64(1) << kWhtBits) - 1;
  std::vector<size_t> order(terms.size());
  for (size_t t = 0; t < order.size(); ++t) order[t] = t;
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t x, size_t y) { return (terms[x].zmask & lo) < (terms[y].zmask & lo); });
  std::vector<DiagGroupDev> gr;
  std::vector<DiagTermDev> tm;
  for (size_t k = 0; k < order.size(); ++k) {
    const PauliTerm& t = terms[order[k]];
    const unsigned zl = unsigned(t.zmask & lo);
    if (gr.empty() || gr.back().zlo != zl) gr.push_back({zl, int(k), int(k)});
    tm.push_back({t.zmask & ~lo, t.cc.real()});
    gr.back().last = int(k) + 1;
  }
  // one upload: terms first (8-byte aligned), then the groups
  const size_t tb = tm.size() * sizeof(DiagTermDev);
  std::vector<char> blob(tb + gr.size() * sizeof(DiagGroupDev));
  std::memcpy(blob.data(), tm.data(), tb);
  std::memcpy(blob.data() + tb, gr.data(), gr.size() * sizeof(DiagGroupDev));
  auto* d_blob = (const char*)scratch_upload(h, blob.data(), blob.size());
  const u64 ntiles = h->n_local >> kWhtBits;
  const unsigned g = unsigned(std::min<u64>(ntiles, 148ull * 6));
  ensure_partials(h, g);
  cudaEvent_t ev[2];
  const double bytes = (out ? 2.0 : 1.0) * double(amp_bytes(h)) * double(h->n_local);
  stat_begin(h, out ? KC_APPLY_OBS : KC_REDUCE, bytes, ev);
  if (init_scale != 0.0) {
    k_pauli_diag_wht<double2><<<g, kThreads, 0, h->stream>>>(a, out, ntiles, (const DiagGroupDev*)(d_blob + tb),
                                                            int(gr.size()), (const DiagTermDev*)d_blob, h->d_partials,
                                                            init_scale);
  } else {
    SV_LAUNCH2(h, k_pauli_diag_wht, SV_CFG(g, kThreads, 0, h->stream), a, out, ntiles, (const DiagGroupDev*)(d_blob + tb),
              int(gr.size()), (const DiagTermDev*)d_blob, h->d_partials);
  }
  stat_end(h, out ? KC_APPLY_OBS : KC_REDUCE, bytes, ev);
  CUDA_CHECK(cudaGetLastError());
  return g;
}

// K14: the state H^n |0...0> followed by diagonal gates with total phase f(i) = sum_t r_t
// (-1)^{pc(i & z_t)} (terms in local physical bits; global bits already folded into r_t), written
// in one write-only pass: psi_i = 2^{-n/2} exp(i f(i)).  Needs n_local >= 12 (one WHT tile).
void init_uniform_phase(sv_handle* h, double2* state, const std::vector<PauliTerm>& terms, double scale) {
  if (h->nl < kWhtBits) sv_fail(SV_ERR_DEVICE, "internal: K14 init needs a full 4096-amplitude tile");
  pauli_diag_wht(h, nullptr, state, terms.empty() ? std::vector<PauliTerm>{{0, cplx(0.0)}} : terms, scale);
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
  if (xmask == 0 && terms.size() >= 8 && h->n_local >= (u64(1) << kWhtBits)) {
    const unsigned g = pauli_diag_wht(h, a, nullptr, terms);
    sum_partials(h, h->d_partials, g, 1, d_out);
    return;
  }
  const unsigned g = red_grid(count);

  ensure_partials(h, g);
  auto* d_terms = (const PauliTermDev*)scratch_upload(h, dt.data(), dt.size() * sizeof(PauliTermDev));
  size_t smem = dt.size() * sizeof(PauliTermDev);
  if (smem > 48 * 1024) {
    CUDA_CHECK(cudaFuncSetAttribute(k_pauli_expval<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CUDA_CHECK(cudaFuncSetAttribute(k_pauli_expval<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  }
  cudaEvent_t ev[2];
  const double bytes = double(amp_bytes(h)) * double(h->n_local);
  stat_begin(h, KC_REDUCE, bytes, ev);
  SV_LAUNCH(h, k_pauli_expval, SV_CFG(g, kThreads, smem, h->stream), a, xmask, pivot, count, d_terms, int(dt.size()),
            h->d_partials);
  stat_end(h, KC_REDUCE, bytes, ev);
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
  if (smem > 48 * 1024) {
    CUDA_CHECK(cudaFuncSetAttribute(k_pauli_apply<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CUDA_CHECK(cudaFuncSetAttribute(k_pauli_apply<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  }
  const unsigned g = unsigned(std::min<u64>(grid_for(h->n_local, kThreads * 4), 148ull * 64));
  const double bytes = (accumulate ? 3.0 : 2.0) * double(amp_bytes(h)) * double(h->n_local);
  cudaEvent_t ev[2];
  stat_begin(h, KC_APPLY_OBS, bytes, ev);
  SV_LAUNCH2(h, k_pauli_apply, SV_CFG(g, kThreads, smem, h->stream), psi, lam, xmask, h->n_local, d_terms,
             int(dt.size()), accumulate ? 1 : 0);
  stat_end(h, KC_APPLY_OBS, bytes, ev);
  CUDA_CHECK(cudaGetLastError());
}

// <psi|H|psi> of non-diagonal x-groups in batches of kMaxXG (x-mask order); one partial sum per
// batch into d_out[0..nbatches).  Returns the number of batches.
int pauli_groups_expval_batched(sv_handle* h, const double2* psi,
                                std::vector<std::pair<u64, std::vector<PauliTerm>>> groups, double* d_out) {
  std::stable_sort(groups.begin(), groups.end(),
                   [](const std::pair<u64, std::vector<PauliTerm>>& a, const std::pair<u64, std::vector<PauliTerm>>& b) {
                     return a.first < b.first;
                   });
  const unsigned g = red_grid(h->n_local);
  int nb = 0;
  for (size_t g0 = 0; g0 < groups.size(); g0 += kMaxXG, ++nb) {
    PauliGroupsArgs G;
    std::vector<PauliApplyTermDev> dt;
    G.ng = int(std::min<size_t>(kMaxXG, groups.size() - g0));
    for (int k = 0; k < G.ng; ++k) {
      G.x[k] = groups[g0 + k].first;
      G.t_begin[k] = int(dt.size());
      for (const auto& t : groups[g0 + k].second) dt.push_back({t.zmask, d2(t.cc)});
    }
    G.t_begin[G.ng] = int(dt.size());
    ensure_partials(h, g);
    auto* d_terms = (const PauliApplyTermDev*)scratch_upload(h, dt.data(), dt.size() * sizeof(PauliApplyTermDev));
    const size_t smem = dt.size() * sizeof(PauliApplyTermDev);
    if (smem > 48 * 1024)
      for (const void* f : {(const void*)k_pauli_expval_multi<double2>, (const void*)k_pauli_expval_multi<float2>})
        CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const double bytes = (G.ng + 1.0) * double(amp_bytes(h)) * double(h->n_local);
    cudaEvent_t ev[2];
    stat_begin(h, KC_REDUCE, bytes, ev);
    if (h->prec == 32)
      k_pauli_expval_multi<float2><<<g, kThreads, smem, h->stream>>>(SV_F32(psi), h->n_local, G, d_terms, int(dt.size()), h->d_partials);
    else
      k_pauli_expval_multi<double2><<<g, kThreads, smem, h->stream>>>(psi, h->n_local, G, d_terms, int(dt.size()), h->d_partials);
    stat_end(h, KC_REDUCE, bytes, ev);
    h->launches++;
    CUDA_CHECK(cudaGetLastError());
    sum_partials(h, h->d_partials, g, 1, d_out + nb);
  }
  return nb;
}

void pauli_groups_apply(sv_handle* h, const double2* psi, double2* lam,
                        const std::vector<std::pair<u64, std::vector<PauliTerm>>>& all_groups) {
  const unsigned g = unsigned(std::min<u64>(grid_for(h->n_local, kThreads * 4), 148ull * 64));
  // a diagonal group with many real Z terms goes through the per-tile WHT kernel (writes lam),
  // the other x-groups accumulate on top of it
  std::vector<std::pair<u64, std::vector<PauliTerm>>> groups;
  bool written = false;
  for (const auto& gr : all_groups) {
    bool diag = !written && gr.first == 0 && gr.second.size() >= 8 && h->n_local >= (u64(1) << kWhtBits);
    for (const auto& t : gr.second) diag = diag && t.cc.imag() == 0.0;
    if (diag) {
      pauli_diag_wht(h, psi, lam, gr.second);
      written = true;
    } else {
      groups.push_back(gr);
    }
  }
  // Groups in x-mask order: the up-to-16 groups of one launch then share their high x bits, so the
  // gathers psi[i ^ x_g] of a launch fall in the same L2-resident window of psi (the grid streams
  // a ~38 MB window of i at a time) and DRAM reads psi about once per launch instead of once per
  // group (config 5, 1000 random terms: 450 x-masks but 37 distinct x >> 20).
  std::stable_sort(groups.begin(), groups.end(),
                   [](const std::pair<u64, std::vector<PauliTerm>>& a, const std::pair<u64, std::vector<PauliTerm>>& b) {
                     return a.first < b.first;
                   });
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
      for (const void* f : {(const void*)k_pauli_apply_multi<double2, 0>, (const void*)k_pauli_apply_multi<float2, 0>,
                            (const void*)k_pauli_apply_multi<double2, 1>, (const void*)k_pauli_apply_multi<float2, 1>})
        CUDA_CHECK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int acc = written || g0 > 0;
    const double bytes = (G.ng + 1.0 + (acc ? 1.0 : 0.0)) * double(amp_bytes(h)) * double(h->n_local);
    cudaEvent_t ev[2];
    stat_begin(h, KC_APPLY_OBS, bytes, ev);
    // SVB200_PAULI_PF=1: issue every group's gather first -- measured slower (config 5: 0.94 vs 0.72 s)
    static const bool pf = getenv("SVB200_PAULI_PF") && std::string(getenv("SVB200_PAULI_PF")) == "1";
    if (h->prec == 32) {
      if (pf) k_pauli_apply_multi<float2, 1><<<g, kThreads, smem, h->stream>>>(SV_F32(psi), SV_F32(lam), h->n_local, G, d_terms, int(dt.size()), acc);
      else k_pauli_apply_multi<float2, 0><<<g, kThreads, smem, h->stream>>>(SV_F32(psi), SV_F32(lam), h->n_local, G, d_terms, int(dt.size()), acc);
    } else {
      if (pf) k_pauli_apply_multi<double2, 1><<<g, kThreads, smem, h->stream>>>(psi, lam, h->n_local, G, d_terms, int(dt.size()), acc);
      else k_pauli_apply_multi<double2, 0><<<g, kThreads, smem, h->stream>>>(psi, lam, h->n_local, G, d_terms, int(dt.size()), acc);
    }
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
  const double bytes = double(amp_bytes(h)) * double(h->n_local) + 24.0 * double(nnz);
  if (lam) {
    CUDA_CHECK(cudaMemsetAsync(lam, 0, h->n_local * amp_bytes(h), h->stream));
    stat_begin(h, KC_APPLY_OBS, bytes, ev);
    if (h->prec == 32)
      k_csr<true, float2><<<g, kThreads, 0, h->stream>>>(SV_F32(psi), A, SV_F32(lam), nullptr);
    else
      k_csr<true, double2><<<g, kThreads, 0, h->stream>>>(psi, A, lam, nullptr);
    stat_end(h, KC_APPLY_OBS, bytes, ev);
    CUDA_CHECK(cudaGetLastError());
  } else {
    ensure_partials(h, g);
    ensure_results(h, 1);
    stat_begin(h, KC_REDUCE, bytes, ev);
    if (h->prec == 32)
      k_csr<false, float2><<<g, kThreads, 0, h->stream>>>(SV_F32(psi), A, nullptr, h->d_partials);
    else
      k_csr<false, double2><<<g, kThreads, 0, h->stream>>>(psi, A, nullptr, h->d_partials);
    stat_end(h, KC_REDUCE, bytes, ev);
    CUDA_CHECK(cudaGetLastError());
    sum_partials(h, h->d_partials, g, 1, h->d_results);
    CUDA_CHECK(cudaMemcpyAsync(&out, h->d_results, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  }
  CUDA_CHECK(cudaFreeAsync(buf, h->stream));
  stream_sync(h);
  return out;
}

double reduce_dot_re(sv_handle* h, const double2* a, const double2* b) {
  const unsigned g = red_grid(h->n_local);
  ensure_partials(h, g);
  ensure_results(h, 1);
  cudaEvent_t ev[2];
  stat_begin(h, KC_REDUCE, 2.0 * double(amp_bytes(h)) * double(h->n_local), ev);
  SV_LAUNCH2(h, k_dot_re, SV_CFG(g, kThreads, 0, h->stream), a, b, h->n_local, h->d_partials);
  stat_end(h, KC_REDUCE, 2.0 * double(amp_bytes(h)) * double(h->n_local), ev);
  CUDA_CHECK(cudaGetLastError());
  sum_partials(h, h->d_partials, g, 1, h->d_results);
  double out = 0;
  d2h(h, &out, h->d_results, sizeof(double));
  return out;
}

void braket_prim_async(sv_handle* h, const double2* bra, const double2* ket, const Prim& gp, double* d_out) {
  if (gp.nb < 1 || gp.nb > 4) sv_fail(SV_ERR_UNSUPPORTED, "generator on more than 4 wires");
  DenseParams P;
  std::vector<double2> mat(gp.m.size());
  for (size_t i = 0; i < gp.m.size(); ++i) mat[i] = d2(gp.m[i]);
  P.mat = scratch_upload(h, mat.data(), mat.size() * sizeof(double2));   // FP64 in both precisions
  P.fval = gp.fval;
  const int nf = popcount64(gp.fmask);
  P.count = h->n_local >> nf;
  P.k = gp.nb;
  for (int j = 0; j < gp.nb; ++j) P.pos[j] = (unsigned char)gp.pos[j];
  P.ins = make_ins(gp.fmask);
  const unsigned g = red_grid(P.count);
  ensure_partials(h, size_t(g) * 2);
  const double bytes = 2.0 * double(amp_bytes(h)) * double(P.count << gp.nb);
  cudaEvent_t ev[2];
  stat_begin(h, KC_BRAKET, bytes, ev);
  if (h->prec == 32) {
    const float2 *b32 = SV_F32(bra), *k32 = SV_F32(ket);
    switch (gp.nb) {
      case 1: k_braket<1, float2><<<g, kThreads, 0, h->stream>>>(b32, k32, P, h->d_partials); break;
      case 2: k_braket<2, float2><<<g, kThreads, 0, h->stream>>>(b32, k32, P, h->d_partials); break;
      case 3: k_braket<3, float2><<<g, kThreads, 0, h->stream>>>(b32, k32, P, h->d_partials); break;
      default: k_braket<4, float2><<<g, kThreads, 0, h->stream>>>(b32, k32, P, h->d_partials); break;
    }
  } else {
    switch (gp.nb) {
      case 1: k_braket<1, double2><<<g, kThreads, 0, h->stream>>>(bra, ket, P, h->d_partials); break;
      case 2: k_braket<2, double2><<<g, kThreads, 0, h->stream>>>(bra, ket, P, h->d_partials); break;
      case 3: k_braket<3, double2><<<g, kThreads, 0, h->stream>>>(bra, ket, P, h->d_partials); break;
      default: k_braket<4, double2><<<g, kThreads, 0, h->stream>>>(bra, ket, P, h->d_partials); break;
    }
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
  const double bytes = double(amp_bytes(h)) * double(h->n_local);
  stat_begin(h, KC_PROBS, bytes, ev);
  if (P.members <= 64) {
    SV_LAUNCH(h, k_probs_perbin, SV_CFG(grid_for(bins, kThreads), kThreads, 0, h->stream), a, P, bins, d_out);
    stat_end(h, KC_PROBS, bytes, ev);
    CUDA_CHECK(cudaGetLastError());
    return;
  }
  u64 chunks = std::max<u64>(1, std::min<u64>(u64(kRedBlocks) / bins, (P.members + kThreads - 1) / kThreads));
  const u64 nblk = bins * chunks;
  ensure_partials(h, nblk);
  SV_LAUNCH(h, k_probs_chunked, SV_CFG(unsigned(nblk), kThreads, 0, h->stream), a, P, int(chunks), h->d_partials);
  stat_end(h, KC_PROBS, bytes, ev);
  CUDA_CHECK(cudaGetLastError());
  sum_partials(h, h->d_partials, int(chunks), int(bins), d_out);
}
