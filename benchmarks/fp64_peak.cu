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
               {"mix_dfma16_dmma2", 2, 2}, {"mix_dfma16_dmma4", 2, 4}};
  for (const Case& c : cases) {
    auto launch = [&]() {
      if (c.kind == 0) k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);
      if (c.kind == 1) k_dmma<<<blocks, threads>>>(out, 0.999999, 1e-7);
      if (c.kind == 2) k_mix<<<blocks, threads>>>(out, 0.999999, 1e-7, c.arg);
      if (c.kind == 3) k_dmul<<<blocks, threads>>>(out, 0.999999);
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
