/*
 * svport.c -- C restatement of the reference's gate-application kernels, TEST / BASELINE
 * INFRASTRUCTURE ONLY (imported only by tests/ and bench.py's cpu_baseline / --impl reference).
 *
 * It restates Alg. 1 (apply_single_qubit, /root/reference/pkg/src/svkit/state.py:154-171) and
 * Alg. 2 (apply_controlled_single_qubit, state.py:192-226) with the same index formulas
 * (mask_high/mask_low, get_masks + on_bits, state.py:128-151 and 212-225), parallelised over
 * the disjoint pairs with OpenMP as the paper's opt-in kernel threading does (PAPER.md:471,
 * SPEC.md:111; the reference declares -fopenmp for its native tier, setup.py:10).  The
 * reference's own native tier (_cy_kernels.pyx) is absent, so this is the "port" CPU
 * baseline.  Parity of this file against the numpy oracle is checked in tests/test_cport.py.
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned long long u64;

static inline void upd(double* a, u64 i0, u64 i1, const double* m) {
  double a0r = a[2 * i0], a0i = a[2 * i0 + 1], a1r = a[2 * i1], a1i = a[2 * i1 + 1];
  a[2 * i0] = m[0] * a0r - m[1] * a0i + m[2] * a1r - m[3] * a1i;
  a[2 * i0 + 1] = m[0] * a0i + m[1] * a0r + m[2] * a1i + m[3] * a1r;
  a[2 * i1] = m[4] * a0r - m[5] * a0i + m[6] * a1r - m[7] * a1i;
  a[2 * i1 + 1] = m[4] * a0i + m[5] * a0r + m[6] * a1i + m[7] * a1r;
}

int svp_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Alg. 1: m = 2x2 interleaved complex row-major */
void svp_apply_1q(double* amps, int n, int q, const double* m, int nthreads) {
  const int q_offset = n - q - 1;
  const u64 stride = 1ull << q_offset;
  const u64 mask_high = (~0ull) << (q_offset + 1);
  const u64 mask_low = q_offset == 0 ? 0ull : (~0ull) >> (64 - q_offset); /* state.py:166-167 */
  const long long npairs = (long long)(1ull << (n - 1));
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (long long k = 0; k < npairs; ++k) {
    u64 i0 = ((2ull * (u64)k) & mask_high) | (mask_low & (u64)k);
    upd(amps, i0, i0 | stride, m);
  }
}

/* Alg. 2 with prescribed control values (aligned with ctrls as given) */
void svp_apply_ctrl_1q(double* amps, int n, const int* ctrls, const int* vals, int nc, int q, const double* m,
                       int nthreads) {
  int offs[64], nb = 0;
  u64 on_bits = 0;
  for (int i = 0; i < nc; ++i) {
    int o = n - 1 - ctrls[i];
    offs[nb++] = o;
    if (vals[i]) on_bits |= 1ull << o;
  }
  offs[nb++] = n - q - 1;
  for (int i = 1; i < nb; ++i) /* sorted(...) of state.py:213 */
    for (int j = i; j > 0 && offs[j - 1] > offs[j]; --j) {
      int t = offs[j];
      offs[j] = offs[j - 1];
      offs[j - 1] = t;
    }
  u64 masks[65];
  const u64 window = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  masks[0] = (1ull << offs[0]) - 1;
  for (int i = 1; i < nb; ++i) masks[i] = ((1ull << offs[i]) - 1) & ~((1ull << (offs[i - 1] + 1)) - 1);
  masks[nb] = window & ~((offs[nb - 1] + 1 >= 64) ? ~0ull : ((1ull << (offs[nb - 1] + 1)) - 1));
  const u64 stride = 1ull << (n - q - 1);
  const long long cnt = (long long)(1ull << (n - 1 - nc));
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (long long k = 0; k < cnt; ++k) {
    u64 i0 = (u64)k & masks[0];
    for (int i = 1; i <= nb; ++i) i0 |= ((u64)k << i) & masks[i];
    i0 |= on_bits;
    upd(amps, i0, i0 | stride, m);
  }
}
