// FP64 roof on this B200: sustained DFMA rate (the pipe the pass kernels run on), the DMMA
// (m8n8k4 f64 tensor) rate, and whether the two pipes add up when issued together.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak benchmarks/fp64_peak.cu
//   build/fp64_peak [seconds_per_case]
//
// Each case runs back to back for the given wall time (default 3 s, long enough to reach the
// board power limit), timed with CUDA events; prints one JSON line per case.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

constexpr int kIter = 4096;

// 16 independent FMA chains per thread
__global__ void __launch_bounds__(256) k_dfma(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIter; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// 8 independent accumulator tiles per warp
__global__ void __launch_bounds__(256) k_dmma(double* out, double a, double b) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3 + i;
  const double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < kIter / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(d[i], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[0] = s;
}

// both in one instruction stream: 16 DFMA chains + 4 DMMA tiles per iteration
__global__ void __launch_bounds__(256) k_mix(double* out, double a, double b, int dmma_per_iter) {
  double x[16];
  double d[4][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3 + i;
  const double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < kIter; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    if (dmma_per_iter >= 1) dmma(d[0], av, bv);
    if (dmma_per_iter >= 2) dmma(d[1], av, bv);
    if (dmma_per_iter >= 3) dmma(d[2], av, bv);
    if (dmma_per_iter >= 4) dmma(d[3], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[0] = s;
}

// pure DMUL (the other half of a complex product)
__global__ void __launch_bounds__(256) k_dmul(double* out, double a) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIter; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = x[i] * a;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}


// two register operands per DFMA (the gate-update form: x0 += t * x1, t uniform)
__global__ void __launch_bounds__(256) k_dfma2r(double* out, double a, double b) {
  double x[16], y[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    x[i] = threadIdx.x * 1e-3 + i;
    y[i] = threadIdx.x * 2e-3 - i;
  }
  for (int it = 0; it < kIter / 2; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(y[i], a, x[i]);
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = fma(x[i], b, y[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i] + y[i];
  if (s == 12345.678) out[0] = s;
}

// three register operands per DFMA
__global__ void __launch_bounds__(256) k_dfma3r(double* out, double a, double b) {
  double x[16], y[16];
  double z = a + threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    x[i] = threadIdx.x * 1e-3 + i;
    y[i] = threadIdx.x * 2e-3 - i;
  }
  for (int it = 0; it < kIter / 2; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(y[i], z, x[i]);
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = fma(x[i], z, y[i]);
    z = z * b;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i] + y[i];
  if (s == 12345.678) out[0] = s;
}

// the pass kernels' RY shear on 16 complex amplitudes in registers (8 pairs on register bit 0..3)
__global__ void __launch_bounds__(256) k_shear(double* out, double t, double s_) {
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  for (int it = 0; it < kIter / 12; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if ((r >> k) & 1) continue;
        double2& x0 = a[r];
        double2& x1 = a[r | (1 << k)];
        x0.x = fma(t, x1.x, x0.x);
        x0.y = fma(t, x1.y, x0.y);
        x1.x = fma(s_, x0.x, x1.x);
        x1.y = fma(s_, x0.y, x1.y);
        x0.x = fma(t, x1.x, x0.x);
        x0.y = fma(t, x1.y, x0.y);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

// complex phase multiply a *= d on 16 amplitudes (2 DMUL + 2 DFMA each, the RZ / Phase form)
__global__ void __launch_bounds__(256) k_cmul(double* out, double c, double sn) {
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  for (int it = 0; it < kIter / 4; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const double t1 = a[r].y * sn, t2 = a[r].x * sn;
      a[r].x = fma(a[r].x, c, -t1);
      a[r].y = fma(a[r].y, c, t2);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

template <int K>
__device__ __forceinline__ void shear_k(double2 (&a)[16], double t, double s_) {
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    if ((r >> K) & 1) continue;
    double2& x0 = a[r];
    double2& x1 = a[r | (1 << K)];
    x0.x = fma(t, x1.x, x0.x);
    x0.y = fma(t, x1.y, x0.y);
    x1.x = fma(s_, x0.x, x1.x);
    x1.y = fma(s_, x0.y, x1.y);
    x0.x = fma(t, x1.x, x0.x);
    x0.y = fma(t, x1.y, x0.y);
  }
}

// the same shear stream with a warp-uniform branch around every gate (the *D cases of the pass
// kernels: a per-thread flip selects the sign of the rotation)
__global__ void __launch_bounds__(256) k_shear_branch(double* out, double t, double s_, int fl) {
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  const int f = fl ^ (threadIdx.x >> 5);   // warp-uniform
  for (int it = 0; it < kIter / 12; ++it) {
    if (f & 1) shear_k<0>(a, -t, -s_); else shear_k<0>(a, t, s_);
    if (f & 2) shear_k<1>(a, -t, -s_); else shear_k<1>(a, t, s_);
    if (f & 4) shear_k<2>(a, -t, -s_); else shear_k<2>(a, t, s_);
    if (f & 8) shear_k<3>(a, -t, -s_); else shear_k<3>(a, t, s_);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

// ... with the sign chosen by a select instead (no branch)
__global__ void __launch_bounds__(256) k_shear_select(double* out, double t, double s_, int fl) {
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  const int f = fl ^ (threadIdx.x >> 5);
  for (int it = 0; it < kIter / 12; ++it) {
    shear_k<0>(a, (f & 1) ? -t : t, (f & 1) ? -s_ : s_);
    shear_k<1>(a, (f & 2) ? -t : t, (f & 2) ? -s_ : s_);
    shear_k<2>(a, (f & 4) ? -t : t, (f & 4) ? -s_ : s_);
    shear_k<3>(a, (f & 8) ? -t : t, (f & 8) ? -s_ : s_);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

// ... the branch condition made warp-uniform (REDUX into a uniform register: BRA.U, no BSSY)
__global__ void __launch_bounds__(256) k_shear_ubranch(double* out, double t, double s_, int fl) {
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  const int f = __reduce_or_sync(0xffffffffu, fl ^ (threadIdx.x >> 5));
  for (int it = 0; it < kIter / 12; ++it) {
    if (f & 1) shear_k<0>(a, -t, -s_); else shear_k<0>(a, t, s_);
    if (f & 2) shear_k<1>(a, -t, -s_); else shear_k<1>(a, t, s_);
    if (f & 4) shear_k<2>(a, -t, -s_); else shear_k<2>(a, t, s_);
    if (f & 8) shear_k<3>(a, -t, -s_); else shear_k<3>(a, t, s_);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

// the pass kernels' form: every gate reads its own coefficients from the by-value parameter block
// (constant bank 0) -- 64 distinct gates per loop trip
struct Cf64 {
  double2 v[64];
};
__global__ void __launch_bounds__(256) k_shear_cf(double* out, const Cf64 cf) {
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  for (int it = 0; it < kIter / 12 / 16; ++it) {
#pragma unroll
    for (int g = 0; g < 64; g += 4) {
      shear_k<0>(a, cf.v[g].x, cf.v[g].y);
      shear_k<1>(a, cf.v[g + 1].x, cf.v[g + 1].y);
      shear_k<2>(a, cf.v[g + 2].x, cf.v[g + 2].y);
      shear_k<3>(a, cf.v[g + 3].x, cf.v[g + 3].y);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

// Do the FP64 pipe and the shared-memory pipe overlap?  Warps [0, nfp) run the shear stream,
// warps [nfp, 16) stream 16-byte LDS/STS round trips through a 64 KiB tile (the pass kernels'
// phase transitions).  mode 0: both kinds, 1: FP64 warps only, 2: smem warps only.
__global__ void __launch_bounds__(512, 1) k_overlap(double* out, double t, double s_, int nfp, int mode, int smem_iters) {
  extern __shared__ __align__(16) double2 tile[];
  const int warp = threadIdx.x >> 5;
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  if (warp < nfp) {
    if (mode == 2) return;
    for (int it = 0; it < kIter / 12; ++it) {
      shear_k<0>(a, t, s_);
      shear_k<1>(a, t, s_);
      shear_k<2>(a, t, s_);
      shear_k<3>(a, t, s_);
    }
  } else {
    if (mode == 1) return;
    const int lt = threadIdx.x - nfp * 32;
    const int nt = (16 - nfp) * 32;
    for (int it = 0; it < smem_iters; ++it) {
#pragma unroll
      for (int r = 0; r < 16; ++r) tile[(lt + r * nt) & 4095] = a[r];
      asm volatile("bar.sync 1, %0;" ::"r"(nt));
#pragma unroll
      for (int r = 0; r < 16; ++r) a[r] = tile[((lt ^ 37) + r * nt) & 4095];
      asm volatile("bar.sync 1, %0;" ::"r"(nt));
    }
  }
  double sum = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) sum += a[i].x + a[i].y;
  if (sum == 12345.678) out[0] = sum;
}

// 8 distinct per-gate coefficient pairs, loaded once before the loop (loop-invariant, 32 URs)
__global__ void __launch_bounds__(256) k_shear_cf8(double* out, const Cf64 cf) {
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  const double2 c0 = cf.v[0], c1 = cf.v[1], c2 = cf.v[2], c3 = cf.v[3], c4 = cf.v[4], c5 = cf.v[5], c6 = cf.v[6],
                c7 = cf.v[7];
  for (int it = 0; it < kIter / 24; ++it) {
    shear_k<0>(a, c0.x, c0.y);
    shear_k<1>(a, c1.x, c1.y);
    shear_k<2>(a, c2.x, c2.y);
    shear_k<3>(a, c3.x, c3.y);
    shear_k<0>(a, c4.x, c4.y);
    shear_k<1>(a, c5.x, c5.y);
    shear_k<2>(a, c6.x, c6.y);
    shear_k<3>(a, c7.x, c7.y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

// per-gate coefficients staged in shared memory (LDS.128 per gate, uniform address -> broadcast)
__global__ void __launch_bounds__(256) k_shear_smemcf(double* out, const Cf64 cf) {
  __shared__ double2 sc[64];
  if (threadIdx.x < 64) sc[threadIdx.x] = cf.v[threadIdx.x];
  __syncthreads();
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  for (int it = 0; it < kIter / 12 / 16; ++it) {
#pragma unroll
    for (int g = 0; g < 64; g += 4) {
      shear_k<0>(a, sc[g].x, sc[g].y);
      shear_k<1>(a, sc[g + 1].x, sc[g + 1].y);
      shear_k<2>(a, sc[g + 2].x, sc[g + 2].y);
      shear_k<3>(a, sc[g + 3].x, sc[g + 3].y);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

// per-gate coefficients, warps desynchronised: warp w starts the 64-gate sequence at gate 4 w
__global__ void __launch_bounds__(256) k_shear_cf_desync(double* out, const Cf64 cf) {
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  const int w = (threadIdx.x >> 5) & 7;
  for (int it = 0; it < kIter / 12 / 16; ++it) {
    for (int gg = 0; gg < 64; gg += 4) {
      const int g = (gg + 8 * w) & 63;
      shear_k<0>(a, cf.v[g].x, cf.v[g].y);
      shear_k<1>(a, cf.v[g + 1].x, cf.v[g + 1].y);
      shear_k<2>(a, cf.v[g + 2].x, cf.v[g + 2].y);
      shear_k<3>(a, cf.v[g + 3].x, cf.v[g + 3].y);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
  const double secs = argc > 1 ? atof(argv[1]) : 3.0;
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  double* out;
  CK(cudaMalloc(&out, 8));
  const int blocks = sms * 4, threads = 256;
  const double nthr = double(blocks) * threads;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  struct Case {
    const char* name;
    int kind, arg;
  } cases[] = {{"dfma", 0, 0}, {"dmul", 3, 0}, {"dmma", 1, 0}, {"mix_dfma16_dmma1", 2, 1},
               {"mix_dfma16_dmma2", 2, 2}, {"mix_dfma16_dmma4", 2, 4},
               {"dfma_2reg", 4, 0},   {"dfma_3reg", 5, 0},        {"shear16", 6, 0},
               {"cmul16", 7, 0},      {"shear16_512thr", 8, 0},   {"shear16_branch", 9, 0},
               {"shear16_select", 10, 0}, {"shear16_branch_8warps", 11, 0}, {"shear16_ubranch", 12, 0},
               {"shear16_ubranch_8warps", 13, 0}, {"shear16_cf", 14, 0}, {"shear16_cf_8warps", 15, 0},
               {"shear16_cf8_invariant", 16, 0}, {"shear16_smem_cf", 17, 0}, {"shear16_smem_cf_8warps", 18, 0},
               {"shear16_cf_desync", 19, 0}};
  Cf64 cf;
  for (int g = 0; g < 64; ++g) cf.v[g] = make_double2(-0.1 + 0.001 * g, 0.19 - 0.002 * g);
  {
    // overlap test: 8 FP64 warps + 8 smem warps per SM, each kind alone, then together
    CK(cudaFuncSetAttribute(k_overlap, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    const int smem_iters = 280;
    float ms[3];
    for (int mode = 0; mode < 3; ++mode) {
      k_overlap<<<sms, 512, 65536>>>(out, -0.1, 0.19, 8, mode, smem_iters);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 20; ++r) k_overlap<<<sms, 512, 65536>>>(out, -0.1, 0.19, 8, mode, smem_iters);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms[mode], e0, e1));
    }
    std::printf("{\"case\": \"overlap_fp64_smem\", \"ms_both\": %.3f, \"ms_fp64_only\": %.3f, \"ms_smem_only\": %.3f}\n",
                ms[0] / 20, ms[1] / 20, ms[2] / 20);
  }
  for (const Case& c : cases) {
    auto launch = [&]() {
      if (c.kind == 0) k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);
      if (c.kind == 1) k_dmma<<<blocks, threads>>>(out, 0.999999, 1e-7);
      if (c.kind == 2) k_mix<<<blocks, threads>>>(out, 0.999999, 1e-7, c.arg);
      if (c.kind == 3) k_dmul<<<blocks, threads>>>(out, 0.999999);
      if (c.kind == 4) k_dfma2r<<<blocks, threads>>>(out, 0.999999, 1e-7);
      if (c.kind == 5) k_dfma3r<<<blocks, threads>>>(out, 0.999999, 1.0000001);
      if (c.kind == 6) k_shear<<<blocks, threads>>>(out, -0.1, 0.19);
      if (c.kind == 7) k_cmul<<<blocks, threads>>>(out, 0.8, 0.6);
      if (c.kind == 8) k_shear<<<sms, 256>>>(out, -0.1, 0.19);   // 8 warps per SM (one PP group)
      if (c.kind == 9) k_shear_branch<<<blocks, threads>>>(out, -0.1, 0.19, 5);
      if (c.kind == 10) k_shear_select<<<blocks, threads>>>(out, -0.1, 0.19, 5);
      if (c.kind == 11) k_shear_branch<<<sms, 256>>>(out, -0.1, 0.19, 5);
      if (c.kind == 12) k_shear_ubranch<<<blocks, threads>>>(out, -0.1, 0.19, 5);
      if (c.kind == 13) k_shear_ubranch<<<sms, 256>>>(out, -0.1, 0.19, 5);
      if (c.kind == 14) k_shear_cf<<<blocks, threads>>>(out, cf);
      if (c.kind == 15) k_shear_cf<<<sms, 256>>>(out, cf);
      if (c.kind == 16) k_shear_cf8<<<blocks, threads>>>(out, cf);
      if (c.kind == 17) k_shear_smemcf<<<blocks, threads>>>(out, cf);
      if (c.kind == 18) k_shear_smemcf<<<sms, 256>>>(out, cf);
      if (c.kind == 19) k_shear_cf_desync<<<blocks, threads>>>(out, cf);
    };
    launch();
    CK(cudaDeviceSynchronize());
    // calibrate launches for ~secs of back-to-back work
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms1 = 0;
    CK(cudaEventElapsedTime(&ms1, e0, e1));
    const int reps = int(secs * 1e3 / ms1) + 1;
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flop_dfma = 0, flop_dmma = 0;
    if (c.kind == 0) flop_dfma = 2.0 * 16 * kIter * nthr;
    if (c.kind == 3) flop_dfma = 1.0 * 16 * kIter * nthr;
    if (c.kind == 1) flop_dmma = (nthr / 32) * 8 * (kIter / 4) * (8 * 8 * 4 * 2.0);
    if (c.kind == 4 || c.kind == 5) flop_dfma = 2.0 * 32 * (kIter / 2) * nthr;
    if (c.kind == 6) flop_dfma = 2.0 * 4 * 8 * 6 * (kIter / 12) * nthr;
    if (c.kind == 8 || c.kind == 11 || c.kind == 13 || c.kind == 15 || c.kind == 18) flop_dfma = 2.0 * 4 * 8 * 6 * (kIter / 12) * double(sms) * 256;
    if (c.kind == 9 || c.kind == 10 || c.kind == 12 || c.kind == 14 || c.kind == 17 || c.kind == 19) flop_dfma = 2.0 * 4 * 8 * 6 * (kIter / 12) * nthr;
    if (c.kind == 16) flop_dfma = 2.0 * 8 * 8 * 6 * (kIter / 24) * nthr;
    if (c.kind == 7) flop_dfma = 2.0 * 16 * 4 * (kIter / 4) * nthr;   // DMUL counted as 2 like DFMA (pipe ops)
    if (c.kind == 2) {
      flop_dfma = 2.0 * 16 * kIter * nthr;
      flop_dmma = (nthr / 32) * c.arg * kIter * (8 * 8 * 4 * 2.0);
    }
    const double s = ms * 1e-3 / reps;
    std::printf("{\"case\": \"%s\", \"ms_per_launch\": %.4f, \"reps\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, "
                "\"total_tflops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d}\n",
                c.name, s * 1e3, reps, flop_dfma / s * 1e-12, flop_dmma / s * 1e-12, (flop_dfma + flop_dmma) / s * 1e-12,
                sms, clk / 1000);
    std::fflush(stdout);
  }
  return 0;
}
