// Runtime pass compiler (fused_jit.cpp): one NVRTC-compiled kernel per fused-pass structure.
#pragma once

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "sv_internal.h"

namespace fused {

struct Program;
struct JitKernel;

// per pass of a program: the compiled kernel (shared across programs with the same structure)
// and the values that parameterise it
struct JitPass {
  std::shared_ptr<JitKernel> kernel;            // nullptr: the pass runs on the interpreter
  std::vector<std::pair<int, int>> cf_refs;     // parameter block slot -> (pass-local op, c[] index)
  std::vector<std::pair<int, int>> tab_refs;    // device tables in order: (pass-local op, length)
  std::vector<double2> cf;                      // the parameter block
  int tab_base = 0;                             // first entry in Program::jit_tabs
  bool split = false;                           // tile in 3 rotating half buffers (1.5 tiles of smem)
  bool pp = false;                              // ping-pong loop: 512 threads, 1 CTA/SM, 3 tile buffers
};

// generated source of one pass (empty: not expressible, e.g. parameter block too large)
bool jit_enabled();   // SVB200_JIT != 0: passes run as generated kernels (planner keeps structure value-free)
bool jit_db();
bool jit_pp();   // direct full-tile passes use the ping-pong tile loop (fused_dev.cuh run_pass_pp)
int jit_ctas_per_sm();   // generated kernels use the double-buffered 1-CTA-per-SM tile loop
std::string jit_pass_source(const Program& prog, int pass, bool two, bool db, std::vector<std::pair<int, int>>* cf_refs,
                            std::vector<std::pair<int, int>>* tab_refs);
// compile / look up every pass kernel of prog (no-op when already prepared); throws SvError on failure
void jit_prepare(Program& prog, bool two);
bool jit_launch(const JitPass& jp, int device, unsigned grid, int threads, size_t smem, cudaStream_t st,
                double2* state, double2* state_hi, const void* dpass, const void* phases, const double2* tabs,
                double2* gen);
void jit_stats(int64_t* compiled, int64_t* compile_us, int64_t* cached);

}  // namespace fused
