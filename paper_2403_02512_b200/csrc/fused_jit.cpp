// Runtime pass compiler for the K7 fusion engine.
//
// The prebuilt tile kernel (fused.cu, k_fused) interprets a pass's op records: per op it loads
// the record from shared memory, tests the predicate and dispatches through a jump table.  That
// interpretation is ~2/3 of the instructions the kernel issues (profiles/r1_ncu_fused_pass_v14.md:
// FP64 34.8 %, BRA + UISETP + LOP3 + LDS + IMAD + LEA ~43 %), and the dispatch boundaries stop the
// compiler from overlapping one gate's FMAs with the next gate's.
//
// Here every planned pass becomes its own kernel: the pass's op sequence is emitted as straight-line
// CUDA (the same fused_dev.cuh building blocks, with register bits, masks and patterns as literals)
// and compiled for sm_100a with NVRTC at plan time.  Gate coefficients are NOT in the source: they
// travel as a by-value kernel parameter block (constant bank 0, read directly by the DFMAs), and
// diagonal / 4x4 tables through a small device table, so a kernel depends only on the pass's
// *structure* -- circuits re-run with new parameters (VQE / QAOA optimisation loops, the rows of a
// multi-observable adjoint sweep) reuse the compiled kernels.  Kernels are cached process-wide by
// their source text; distinct passes compile in parallel.
//
// Data movement, tiles, phases and results are exactly those of k_fused<*, false, *>; the pass
// compiler only removes the interpreter.  SVB200_JIT=0 selects the interpreter (A/B timing).
#include <fcntl.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <sys/types.h>
#include <unistd.h>

#include <cerrno>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "fused.h"
#include "fused_jit.h"

namespace fused {
namespace {

const char* kDevSrc =
#include "fused_dev_src.inc"
    ;

std::string hex64(u64 v) {
  char b[32];
  std::snprintf(b, sizeof(b), "0x%llxull", v);
  return b;
}

int swz_h(int s) { return s ^ (((s >> 3) ^ (s >> 6) ^ (s >> 9)) & 7); }

const int kPairK0[6] = {0, 0, 0, 1, 1, 2};
const int kPairK1[6] = {1, 2, 3, 2, 3, 3};

// Source generator for one pass.  Records, in emission order, which op coefficients go into the
// parameter block (cf_refs) and which coefficient tables go into the device table (tab_refs).
constexpr int fdev_gen_sub = 4;   // == fdev::kGenSub (fused.cu checks): accumulators per warp and slot

struct Gen {
  bool pp = false;   // ping-pong loop: one accumulator per warp and slot (its smem is full)
  std::ostringstream o;
  std::vector<std::pair<int, int>> cf_refs;   // (pass-local op, c[] index)
  std::vector<std::pair<int, int>> tab_refs;  // (pass-local op, table length)
  int tab_len = 0;

  std::map<std::pair<int, int>, int> cf_slot, tab_off;   // one slot per (op, entry) even when emitted twice
  // j = -1: entry 1 of the op's coefficient table (the odd-parity value of a parity table)
  std::string C(int op, int j) {
    static const bool one = getenv("SVB200_JIT_EXP_ONECF") && std::string(getenv("SVB200_JIT_EXP_ONECF")) == "1";
    if (one) {   // timing experiment only (wrong results): every op reads the same coefficient slot
      if (cf_refs.empty()) cf_refs.push_back({op, j});
      return "cf.v[0]";
    }
    auto it = cf_slot.find({op, j});
    if (it == cf_slot.end()) {
      cf_refs.push_back({op, j});
      it = cf_slot.emplace(std::make_pair(op, j), int(cf_refs.size()) - 1).first;
    }
    return "cf.v[" + std::to_string(it->second) + "]";
  }
  std::string T(int op, int len) {
    auto it = tab_off.find({op, len});
    if (it == tab_off.end()) {
      tab_refs.push_back({op, len});
      it = tab_off.emplace(std::make_pair(op, len), tab_len).first;
      tab_len += len;
    }
    return "(tabs + " + std::to_string(it->second) + ")";
  }
};

// table index constant of a DIAGG / GEND op: off-register table bits from the thread's physical
// base, register table bits carrying a dynamic flip toggle their table bit
std::string tconst_expr(const FOp& op, int W[4]) {
  std::string e = "0";
  for (int k = 0; k < 4; ++k) W[k] = 0;
  for (int j = 0; j < op.nt; ++j) {
    const int rg = op.treg[j];
    if (rg == 0xFF) {
      e += " | (int((pb >> " + std::to_string(op.tphys[j]) + ") & 1ull) << " + std::to_string(j) + ")";
    } else {
      W[rg] |= 1 << j;
      e = "(" + e + ") ^ (((fthr >> " + std::to_string(rg) + ") & 1) << " + std::to_string(j) + ")";
    }
  }
  return e;
}

// Versioned phases: the thread-dependent predicates of a phase (the patterns of thread-predicated X
// gates and of thread-controlled ops, the parities of parity phases) are evaluated once at the
// phase start and the phase's op sequence is emitted once per outcome, so inside a version every
// per-thread flip is a compile-time constant -- no branch between gates (a warp-uniform branch
// between two gates costs ~20 % of the FP64 rate, benchmarks/fp64_peak.cu shear16_branch).
struct VPred {
  int kind;   // 0: (pb & m) == v; 1: parity(pb & m)
  u64 m, v;
};
struct VCtx {
  std::vector<VPred> preds;
  int ver = 0;    // outcome bits, one per predicate
  int fthr = 0;   // the per-thread flip mask so far (compile-time in this version)
  bool eval(int kind, u64 m, u64 v) const {
    for (size_t i = 0; i < preds.size(); ++i)
      if (preds[i].kind == kind && preds[i].m == m && preds[i].v == v) return (ver >> i) & 1;
    return false;
  }
};

// Warp-uniform predicates: when no predicate of a phase involves a lane bit, every predicate is the
// same across a warp; the phase evaluates them once into a uniform register (one REDUX.OR), so the
// flips, the thread-controlled ops and the *D cases branch on uniform values (BRA.U, no
// divergence bookkeeping: a uniform branch between two gates costs ~4 % of the FP64 rate instead
// of ~22 %, benchmarks/fp64_peak.cu shear16_ubranch vs shear16_branch).
struct UPreds {
  std::vector<VPred> preds;
  std::string of(int kind, u64 m, u64 v) const {
    for (size_t i = 0; i < preds.size(); ++i)
      if (preds[i].kind == kind && preds[i].m == m && preds[i].v == v) return "((vp_ >> " + std::to_string(i) + ") & 1)";
    return std::string();
  }
};

// dyn: register bits that may carry a per-thread flip at this op (fthr starts at 0 every phase)
// vc: versioned phase (predicates and flips are compile-time), or nullptr
// up: the phase's predicates in the uniform register vp_, or nullptr
bool emit_op(Gen& g, int i, const FOp& op, bool parity_tab, int& dyn, VCtx* vc = nullptr, const UPreds* up = nullptr) {
  std::ostringstream& o = g.o;
  const int cs = op.cs;
  bool has_pred = op.pm != 0 || op.pv != 0;
  if (vc) {
    if (op.fk && vc->eval(0, op.fpm, op.fpv)) vc->fthr ^= op.fk;
    const bool active = !has_pred || vc->eval(0, op.pm, op.pv);
    if (cs >= CS_XFLIP && cs < CS_XFLIP + 4) {
      if (active) vc->fthr ^= 1 << (cs - CS_XFLIP);
      return true;
    }
    if (!active) return true;   // thread-controlled op off for this version (a GEN op adds 0)
    has_pred = false;
    dyn = 0;
    o << "    {\n      const int fthr = " << vc->fthr << ";\n";
  } else {
    o << "    {\n";
    if (op.fk) {
      if (up) o << "      if " << up->of(0, op.fpm, op.fpv) << " fthr ^= " << op.fk << ";\n";
      else o << "      if ((pb & " << hex64(op.fpm) << ") == " << hex64(op.fpv) << ") fthr ^= " << op.fk << ";\n";
      dyn |= op.fk;
    }
    if (cs >= CS_XFLIP && cs < CS_XFLIP + 4) dyn |= 1 << (cs - CS_XFLIP);
  }
  const std::string pred = up && has_pred ? up->of(0, op.pm, op.pv) : "((pb & " + hex64(op.pm) + ") == " + hex64(op.pv) + ")";
  const std::string cm = std::to_string(int(op.cm));
  const std::string cvd = "(" + std::to_string(int(op.cv)) + " ^ (fthr & " + cm + "))";
  if (cs >= CS_GEN1) {
    o << "      double re = 0.0, im = 0.0;\n";
    o << "      if (" << (has_pred ? pred : std::string("true")) << ") {\n";
    if (cs < CS_GEN2) {
      const int k = (cs - CS_GEN1) / 4, t = (cs - CS_GEN1) % 4;
      const std::string c0 = g.C(i, 0), c1 = g.C(i, 1), c2 = g.C(i, 2), c3 = g.C(i, 3);
      o << "        const bool sw = (fthr >> " << k << ") & 1;\n";
      o << "        fdev::gen1<" << k << ", " << t << ">(a, sw ? " << c3 << " : " << c0 << ", sw ? " << c2 << " : " << c1
        << ", sw ? " << c1 << " : " << c2 << ", sw ? " << c0 << " : " << c3 << ", " << cm << ", " << cvd
        << ", re, im);\n";
    } else if (cs < CS_GEND) {
      const int pi = (cs - CS_GEN2) / 4, t = (cs - CS_GEN2) % 4;
      const int k0 = kPairK0[pi], k1 = kPairK1[pi];
      o << "        const int f = ((fthr >> " << k0 << ") & 1) | (((fthr >> " << k1 << ") & 1) << 1);\n";
      o << "        fdev::gen2<" << k0 << ", " << k1 << ", " << t << ">(a, " << g.T(i, 16) << ", " << cm << ", " << cvd
        << ", f, re, im);\n";
    } else if (cs < CS_GEND + 4 && parity_tab) {
      // parity table (Z / Z..Z generators): S_even + d S_odd, d from the parameter block
      const int t = cs - CS_GEND;
      int W[4];
      const std::string tc = tconst_expr(op, W);
      int M = 0;
      for (int k = 0; k < 4; ++k)
        if (W[k]) M |= 1 << k;
      o << "        fdev::gen_parity<" << t << ", " << M << ">(a, " << g.C(i, -1) << ", __popc(" << tc << ") & 1, " << cm
        << ", " << cvd << ", re, im);\n";
    } else if (cs < CS_GEND + 4) {
      const int t = cs - CS_GEND;
      int W[4];
      const std::string tc = tconst_expr(op, W);
      o << "        fdev::gen_diag_tab<" << t << ", " << W[0] << ", " << W[1] << ", " << W[2] << ", " << W[3] << ">(a, "
        << g.T(i, 1 << op.nt) << ", " << tc << ", " << cm << ", " << cvd << ", re, im);\n";
    } else {
      return false;
    }
    o << "      }\n";
    o << "      fdev::gen_commit<" << (g.pp ? 1 : fdev_gen_sub) << ">(re, im, acc_warp, " << op.slot << ");\n";
    o << "    }\n";
    return true;
  }
  if (has_pred) o << "      if " << pred << " {\n";
  if (cs >= CS_PAIR1 && cs < CS_PAIR1 + 16) {
    const int k = cs / 4, mt = cs % 4;
    if (mt != MT_X)
      o << "      fdev::pair1<" << k << ", " << mt << ">(a, " << g.C(i, 0) << ", " << g.C(i, 1) << ", " << g.C(i, 2)
        << ", " << g.C(i, 3) << ");\n";
  } else if (cs >= CS_PAIR1D && cs < CS_PAIR1D + 16) {
    const int k = (cs - CS_PAIR1D) / 4, mt = op.mtype;
    if (mt != MT_X) {
      const std::string c0 = g.C(i, 0), c1 = g.C(i, 1), c2 = g.C(i, 2), c3 = g.C(i, 3);
      o << "      if ((fthr >> " << k << ") & 1) fdev::pair1<" << k << ", " << mt << ">(a, " << c3 << ", " << c2 << ", "
        << c1 << ", " << c0 << ");\n";
      o << "      else fdev::pair1<" << k << ", " << mt << ">(a, " << c0 << ", " << c1 << ", " << c2 << ", " << c3
        << ");\n";
    }
  } else if (cs >= CS_PHASE1 && cs < CS_PHASE1 + 8) {
    o << "      fdev::phase1<" << (cs - CS_PHASE1) / 2 << ", " << (cs - CS_PHASE1) % 2 << ">(a, " << g.C(i, 0) << ");\n";
  } else if (cs >= CS_PHASE1D && cs < CS_PHASE1D + 8) {
    const int k = (cs - CS_PHASE1D) / 2;
    const std::string c0 = g.C(i, 0);
    o << "      if (((fthr >> " << k << ") & 1) ^ " << int(op.v) << ") fdev::phase1<" << k << ", 1>(a, " << c0 << ");\n";
    o << "      else fdev::phase1<" << k << ", 0>(a, " << c0 << ");\n";
  } else if (cs == CS_SCALAR) {
    o << "      _Pragma(\"unroll\") for (int r = 0; r < fdev::kRegs; ++r) fdev::cmul_ip(a[r], " << g.C(i, 0) << ");\n";
  } else if (cs >= CS_XFLIP && cs < CS_XFLIP + 4) {
    o << "      fthr ^= " << (1 << (cs - CS_XFLIP)) << ";\n";
  } else if (cs >= CS_SHEAR && cs < CS_SHEAR + 16) {
    const int k = (cs - CS_SHEAR) / 4, sub = (cs - CS_SHEAR) % 4;
    const std::string c0 = g.C(i, 0);
    if (sub == SH_RY) o << "      fdev::pair_shear<" << k << ", false>(a, " << c0 << ".x, " << c0 << ".y);\n";
    if (sub == SH_RX) o << "      fdev::pair_shear<" << k << ", true>(a, " << c0 << ".x, " << c0 << ".y);\n";
    if (sub == SH_RYD) {
      o << "      if ((fthr >> " << k << ") & 1) fdev::pair_shear<" << k << ", false>(a, -" << c0 << ".x, -" << c0
        << ".y);\n";
      o << "      else fdev::pair_shear<" << k << ", false>(a, " << c0 << ".x, " << c0 << ".y);\n";
    }
  } else if (cs >= CS_TAN && cs < CS_TAN + 16) {
    const int k = (cs - CS_TAN) / 4, sub = (cs - CS_TAN) % 4;
    o << "      fdev::pair_tan<" << k << ", " << ((sub & 1) ? "true" : "false") << ", " << ((sub & 2) ? "true" : "false")
      << ">(a, " << g.C(i, 0) << ".x);\n";
  } else if (cs == CS_RDIAG) {
    for (int r = 0; r < 16; ++r)
      if ((op.xm >> r) & 1) o << "      fdev::cmul_ip(a[" << r << "], " << g.C(i, 16 + r) << ");\n";
  } else if (cs >= CS_TAND && cs < CS_TAND + 8) {
    const int k = (cs - CS_TAND) / 2;
    const char* cot = (cs - CS_TAND) % 2 ? "true" : "false";
    const std::string c0 = g.C(i, 0);
    o << "      if ((fthr >> " << k << ") & 1) fdev::pair_tan<" << k << ", false, " << cot << ", true>(a, " << c0
      << ".x);\n";
    o << "      else fdev::pair_tan<" << k << ", false, " << cot << ">(a, " << c0 << ".x);\n";
  } else if (cs >= CS_PARITY && cs < CS_PARITY + 16) {
    const int M = cs - CS_PARITY;
    std::string tp = "(__popc(fthr & " + std::to_string(M) + ") + " + std::to_string(int(op.v));
    if (op.xm && vc) tp += std::string(" + ") + (vc->eval(1, op.xm, 0) ? "1" : "0");
    else if (op.xm && up) tp += " + " + up->of(1, op.xm, 0);
    else if (op.xm) tp += " + __popcll(pb & " + hex64(op.xm) + ")";
    tp += ") & 1";
    o << "      fdev::parity_phase<" << M << ">(a, " << g.C(i, 0) << ", " << tp << ");\n";
  } else if (cs >= CS_PAIRGR && cs < CS_PAIRGR + 15 && op.mtype == MT_X &&
             (vc || __builtin_popcount(cs - CS_PAIRGR + 1) == 1 || (dyn & (cs - CS_PAIRGR + 1)) == 0)) {
    // register-controlled X: register renaming (static control bits) or selects (flipped ones);
    // a multi-bit xmask needs its i0 pattern static
    const int xr = cs - CS_PAIRGR + 1, cc = op.cm & ~xr & 15;
    const int fs = vc ? vc->fthr : 0;   // versioned: the flips are folded into the pattern
    o << "      fdev::swap_x<" << xr << ", " << cc << ", " << ((op.cv ^ fs) & cc) << ", " << (dyn & cc) << ", "
      << ((op.cv ^ fs) & xr) << ">(a, fthr);\n";
  } else if (cs >= CS_PAIRGR && cs < CS_PAIRGR + 15) {
    o << "      fdev::pairg<" << (cs - CS_PAIRGR + 1) << ", fdev::kMtReal>(a, " << g.C(i, 0) << ", " << g.C(i, 1) << ", "
      << g.C(i, 2) << ", " << g.C(i, 3) << ", " << cm << ", " << cvd << ");\n";
  } else if (cs >= CS_PAIRG && cs < CS_PAIRG + 15) {
    o << "      fdev::pairg<" << (cs - CS_PAIRG + 1) << ", fdev::kMtGeneral>(a, " << g.C(i, 0) << ", " << g.C(i, 1)
      << ", " << g.C(i, 2) << ", " << g.C(i, 3) << ", " << cm << ", " << cvd << ");\n";
  } else if (cs == CS_DIAGG) {
    int W[4];
    const std::string tc = tconst_expr(op, W);
    o << "      fdev::diag_tab<" << W[0] << ", " << W[1] << ", " << W[2] << ", " << W[3] << ">(a, " << g.T(i, 1 << op.nt)
      << ", " << tc << ", " << cm << ", " << cvd << ");\n";
  } else if (cs >= CS_DENSE2 && cs < CS_DENSE2 + 6) {
    const int k0 = kPairK0[cs - CS_DENSE2], k1 = kPairK1[cs - CS_DENSE2];
    o << "      {\n        const int f = ((fthr >> " << k0 << ") & 1) | (((fthr >> " << k1 << ") & 1) << 1);\n";
    o << "        fdev::dense2<" << k0 << ", " << k1 << ">(a, " << g.T(i, 16) << ", " << cm << ", " << cvd
      << ", f);\n      }\n";
  } else {
    return false;
  }
  if (has_pred) o << "      }\n";
  o << "    }\n";
  return true;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// compiled-kernel cache (process-wide, keyed by the generated source)
// ---------------------------------------------------------------------------------------------
struct JitKernel {
  std::string src;
  bool ok = false;
  std::string log;
  std::vector<char> cubin;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int smem_set[64] = {0};   // per device: dynamic shared memory attribute already set
  std::mutex mu;
};

namespace {
std::mutex g_jit_mu;
std::map<std::string, std::shared_ptr<JitKernel>> g_jit;
std::atomic<int64_t> g_jit_compiled{0};
std::atomic<int64_t> g_jit_compile_us{0};

// On-disk cubin cache shared by the processes of one user (tests, smoke, bench): the file name
// is a 64-bit FNV-1a hash of the full source + compiler version + options, and the file stores the
// full source too, so a hash collision is detected and ignored.  SVB200_JIT_CACHE=<dir> (default
// $XDG_CACHE_HOME/svb200_jit, else $TMPDIR/svb200_jit-<uid>); "0" disables.  The directory is
// created 0700 and used only when it is ours and not writable by group/others: a cubin planted
// by another local user is never loaded.
const char* kOptsKey = "sm_100a|c++17|lineinfo|restrict|default-device";

std::string cache_dir() {
  const char* e = getenv("SVB200_JIT_CACHE");
  if (e && std::string(e) == "0") return std::string();
  if (e && *e) return e;
  const char* x = getenv("XDG_CACHE_HOME");
  if (x && *x) return std::string(x) + "/svb200_jit";
  const char* t = getenv("TMPDIR");
  return std::string(t && *t ? t : "/tmp") + "/svb200_jit-" + std::to_string(unsigned(getuid()));
}

// create (mode 0700) if missing, then require: a real directory, owned by us, no group/other write
bool cache_dir_ok(const std::string& dir) {
  if (dir.empty()) return false;
  if (mkdir(dir.c_str(), 0700) != 0 && errno != EEXIST) return false;
  struct stat st;
  if (lstat(dir.c_str(), &st) != 0 || !S_ISDIR(st.st_mode)) return false;
  return st.st_uid == getuid() && (st.st_mode & (S_IWGRP | S_IWOTH)) == 0;
}

u64 fnv1a(const std::string& s) {
  u64 h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

bool cache_load(const std::string& path, const std::string& full, std::vector<char>& cubin) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  uint64_t ns = 0, nc = 0;
  bool ok = std::fread(&ns, 8, 1, f) == 1 && ns == full.size();
  std::string src;
  if (ok) {
    src.resize(ns);
    ok = std::fread(&src[0], 1, ns, f) == ns && src == full && std::fread(&nc, 8, 1, f) == 1 && nc > 0 &&
         nc < (uint64_t(1) << 30);
  }
  if (ok) {
    cubin.resize(nc);
    ok = std::fread(cubin.data(), 1, nc, f) == nc;
  }
  std::fclose(f);
  return ok;
}

void cache_store(const std::string& path, const std::string& full, const std::vector<char>& cubin) {
  static std::atomic<unsigned> counter{0};
  const std::string tmp = path + ".tmp" + std::to_string(long(getpid())) + "." + std::to_string(counter++);
  const int fd = open(tmp.c_str(), O_WRONLY | O_CREAT | O_EXCL, 0600);
  if (fd < 0) return;
  FILE* f = fdopen(fd, "wb");
  if (!f) {
    close(fd);
    std::remove(tmp.c_str());
    return;
  }
  const uint64_t ns = full.size(), nc = cubin.size();
  bool ok = std::fwrite(&ns, 8, 1, f) == 1 && std::fwrite(full.data(), 1, ns, f) == ns &&
            std::fwrite(&nc, 8, 1, f) == 1 && std::fwrite(cubin.data(), 1, nc, f) == nc;
  ok = (std::fclose(f) == 0) && ok;
  if (ok) std::rename(tmp.c_str(), path.c_str());   // atomic publish
  else std::remove(tmp.c_str());
}

void compile_kernel(JitKernel& k) {
  const auto t0 = std::chrono::steady_clock::now();
  // configuration #defines lead the generated text; they must precede the shared header
  const size_t cut = k.src.find("struct SvCf");
  const std::string full = k.src.substr(0, cut) + std::string(kDevSrc) + "\n" + k.src.substr(cut);
  int major = 0, minor = 0;
  nvrtcVersion(&major, &minor);
  const std::string keyed = full + "\n//" + kOptsKey + "|nvrtc" + std::to_string(major) + "." + std::to_string(minor);
  const std::string dir = cache_dir();
  const bool dir_ok = cache_dir_ok(dir);
  char hb[32];
  std::snprintf(hb, sizeof(hb), "%016llx", fnv1a(keyed));
  const std::string path = dir_ok ? dir + "/" + hb + ".svc" : std::string();
  if (!path.empty() && cache_load(path, keyed, k.cubin)) {
    k.ok = true;
    return;
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, full.c_str(), "svb200_pass.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    k.log = "nvrtcCreateProgram failed";
    return;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--restrict", "-default-device"};
  const nvrtcResult r = nvrtcCompileProgram(prog, 5, opts);
  size_t ls = 0;
  nvrtcGetProgramLogSize(prog, &ls);
  if (ls > 1) {
    k.log.resize(ls);
    nvrtcGetProgramLog(prog, &k.log[0]);
  }
  if (r == NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    k.cubin.resize(n);
    nvrtcGetCUBIN(prog, k.cubin.data());
    k.ok = n > 0;
  }
  nvrtcDestroyProgram(&prog);
  if (k.ok && !path.empty()) cache_store(path, keyed, k.cubin);
  g_jit_compiled += 1;
  g_jit_compile_us += std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

bool jit_enabled() {
  static const bool on = !(getenv("SVB200_JIT") && std::string(getenv("SVB200_JIT")) == "0");
  return on;
}

// SVB200_JIT_MODE=db: one CTA per SM with two tile buffers (the next tile streams in during the
// current one's phases) instead of two single-buffer CTAs per SM
bool jit_db() {
  static const bool db = getenv("SVB200_JIT_MODE") && std::string(getenv("SVB200_JIT_MODE")) == "db";
  return db;
}

// SVB200_JIT_VMAX: most thread predicates a phase may have and still be emitted once per outcome
// (2^VMAX copies of its ops); 0 turns versioning off
int jit_vmax() {
  static const int v = getenv("SVB200_JIT_VMAX") ? std::max(0, std::min(4, atoi(getenv("SVB200_JIT_VMAX")))) : 0;
  return v;
}

// SVB200_JIT_UNIFORM=0: per-thread predicate evaluation instead of one warp-uniform REDUX per phase
bool jit_uniform_preds() {
  static const bool on = !(getenv("SVB200_JIT_UNIFORM") && std::string(getenv("SVB200_JIT_UNIFORM")) == "0");
  return on;
}

// SVB200_JIT_PP=1: direct passes use the ping-pong loop instead of two free-running CTAs per SM.
// Measured on the 30-qubit bench circuit: 0.410 s (PP) vs 0.401 s (two CTAs) -- the lockstep hides
// the shared-memory round trips, but its arithmetic segments then run on 8 warps; off by default.
bool jit_pp() {
  static const bool on = getenv("SVB200_JIT_PP") && std::string(getenv("SVB200_JIT_PP")) == "1";
  return on;
}

// resident CTAs per SM of the single-buffer form (SVB200_JIT_CTAS, default 2)
int jit_ctas_per_sm() {
  static const int n = getenv("SVB200_JIT_CTAS") ? std::max(1, std::min(3, atoi(getenv("SVB200_JIT_CTAS")))) : 2;
  return n;
}

std::string jit_pass_source(const Program& prog, int pass, bool two, bool db, std::vector<std::pair<int, int>>* cf_refs,
                            std::vector<std::pair<int, int>>* tab_refs) {
  const FPassArgs& A = prog.passes[pass];
  Gen g;
  std::ostringstream& o = g.o;
  std::ostringstream body;
  static const bool direct_on = !(getenv("SVB200_JIT_DIRECT") && std::string(getenv("SVB200_JIT_DIRECT")) == "0");
  const bool direct = direct_on && A.direct && !db && A.n_phases > 0;
  // measured: hiding the rest of the next tile's load this way does not pay (0.539 vs 0.529 s on
  // the bench circuit) -- the passes are bound by their compute phases, not the load -- so off
  static const bool split_on = getenv("SVB200_JIT_SPLIT") && std::string(getenv("SVB200_JIT_SPLIT")) == "1";
  const bool split = split_on && direct && jit_ctas_per_sm() <= 2 && !jit_pp();
  // ping-pong tile loop (fused_dev.cuh run_pass_pp): direct passes on full 12-bit tiles
  const bool pp = jit_pp() && direct && A.b == kMaxB && A.nthr == kMaxB - kRB;
  g.pp = pp;
  // first phase straight from global memory after an L2 prefetch (fused_dev.cuh run_pass DFL)
  static const bool dfl_on = getenv("SVB200_JIT_DFL") && std::string(getenv("SVB200_JIT_DFL")) == "1";
  const bool dfl = dfl_on && direct && !pp && !split;
  if (getenv("SVB200_JIT_EXP_NOSMEM") && std::string(getenv("SVB200_JIT_EXP_NOSMEM")) == "1") o << "  double2 ap_[16];\n";
  if (direct) {
    // the thread's physical store bits in the last phase (its lane bits land on physical 0..2)
    const FPhase& L = prog.phases[A.phase_begin + A.n_phases - 1];
    o << "  u64 st_thr = 0;\n";
    for (int j = 0; j < A.nthr; ++j)
      o << "  if ((threadIdx.x >> " << j << ") & 1) st_thr |= " << hex64(1ull << A.tpos_st[L.thr[j]]) << ";\n";
  }
  for (int ph = 0; ph < A.n_phases; ++ph) {
    const FPhase& F = prog.phases[A.phase_begin + ph];
    const bool last_direct = direct && ph == A.n_phases - 1;
    int W[4];
    for (int k = 0; k < 4; ++k) W[k] = swz_h(1 << F.reg[k]);
    o << "  {   // phase " << ph << (last_direct ? " (direct store)" : "") << "\n";
    static const bool tab_thr = getenv("SVB200_JIT_THRTAB") && std::string(getenv("SVB200_JIT_THRTAB")) == "1";
    if (tab_thr && !pp) {
      o << "    FDEV_PHASE_LOAD(s_ph[" << ph << "], " << W[0] << ", " << W[1] << ", " << W[2] << ", " << W[3] << ")\n";
    } else {
      // the thread's slot: swizzled offset and physical bits as literal-mask expressions of tid
      std::string se = "0", pe = "0ull";
      for (int j = 0; j < A.nthr; ++j) {
        const std::string bit = "((threadIdx.x >> " + std::to_string(j) + ") & 1)";
        se += " ^ (" + bit + " ? " + std::to_string(swz_h(1 << F.thr[j])) + " : 0)";
        pe += " | (" + bit + " ? " + hex64(1ull << A.tpos[F.thr[j]]) + " : 0ull)";
      }
      static const bool exp_nosmem = getenv("SVB200_JIT_EXP_NOSMEM") && std::string(getenv("SVB200_JIT_EXP_NOSMEM")) == "1";
      if (dfl && ph == 0) {
        o << "    FDEV_PHASE_LOAD_G(" << se << ", " << pe;
        for (int k = 0; k < 4; ++k) o << ", " << hex64(1ull << A.tpos[F.reg[k]]);
        o << ")\n    next_load();\n";
      } else if (exp_nosmem && ph > 0) {   // timing experiment only (wrong results): no smem round trip between phases
        o << "    const int s0 = (" << se << "); const u64 pb = base | (" << pe << "); double2 a[16];\n";
        o << "    _Pragma(\"unroll\") for (int r = 0; r < 16; ++r) a[r] = ap_[r];\n    int fthr = 0; (void)pb; (void)s0; (void)fthr;\n";
      } else {
        o << "    FDEV_PHASE_LOAD_X(" << se << ", " << pe << ", " << W[0] << ", " << W[1] << ", " << W[2] << ", " << W[3]
          << ")\n";
      }
    }
    if (pp) o << "    FDEV_STEP_I(" << 2 * ph << ");\n";   // end of segment T_ph
    // DFL: the barrier still separates this phase's reads from the next tile's first store
    if (last_direct) o << (pp ? "    next_load();\n" : (dfl ? "    __syncthreads();\n" : "    __syncthreads();\n    next_load();\n"));
    auto parity_tab_of = [&](const FOp& op) {
      bool ptab = false;
      if (op.cs >= CS_GEND && op.cs < CS_GEND + 4 && op.nt >= 1) {
        // the table's structure (parity form), not its values, decides the code: generators are
        // fixed per gate kind, so this is stable across parameters
        const double2* t = prog.coef.data() + op.tab;
        ptab = t[0].x == 1.0 && t[0].y == 0.0;
        for (int e = 0; e < (1 << op.nt) && ptab; ++e) {
          const double2 want = (__builtin_popcount(e) & 1) ? t[1] : make_double2(1.0, 0.0);
          ptab = t[e].x == want.x && t[e].y == want.y;
        }
      }
      return ptab;
    };
    auto emit_store = [&]() {
      if (last_direct) {
        o << "    FDEV_PHASE_STORE_GLOBAL" << (two ? "2(" : "(") << int(F.flip);
        for (int k = 0; k < 4; ++k) o << ", " << hex64(1ull << A.tpos_st[F.reg[k]]);
        o << ")\n";
        if (pp) o << "    FDEV_STEP_I(" << 2 * ph + 1 << ");\n";   // end of segment C_ph
      } else {
        if (pp) o << "    FDEV_STEP_I(" << 2 * ph + 1 << ");\n";   // end of segment C_ph; the store opens T_ph+1
        static const bool exp_nosmem = getenv("SVB200_JIT_EXP_NOSMEM") && std::string(getenv("SVB200_JIT_EXP_NOSMEM")) == "1";
        // the next phase keeps the warp-bit positions: warp-local exchange (fused_plan.cpp)
        bool warp_local = ph + 1 < A.n_phases && A.nthr == kMaxB - kRB;
        if (warp_local) {
          const FPhase& N = prog.phases[A.phase_begin + ph + 1];
          for (int j = 5; j < A.nthr; ++j) warp_local = warp_local && N.thr[j] == F.thr[j];
        }
        // top thread bits kept by the next phase: 1 -> each 128-thread half, 2 -> each 64-thread
        // quarter of the CTA exchanges only within itself (named barrier over the group)
        int kept = 0;
        if (!warp_local && !pp && ph + 1 < A.n_phases && A.nthr == kMaxB - kRB) {
          const FPhase& N = prog.phases[A.phase_begin + ph + 1];
          while (kept < 2 && N.thr[A.nthr - 1 - kept] == F.thr[A.nthr - 1 - kept]) ++kept;
        }
        if (exp_nosmem) o << "    _Pragma(\"unroll\") for (int r = 0; r < 16; ++r) ap_[r] = a[r];\n";
        else if (kept > 0)
          o << "    FDEV_PHASE_STORE_GROUP(" << int(F.flip) << ", " << W[0] << ", " << W[1] << ", " << W[2] << ", " << W[3]
            << ", " << (kept == 1 ? "1 + (threadIdx.x >> 7), 128" : "3 + (threadIdx.x >> 6), 64") << ")\n";
        else o << "    FDEV_PHASE_STORE" << (warp_local ? "_WARP(" : "(") << int(F.flip) << ", " << W[0] << ", " << W[1] << ", "
               << W[2] << ", " << W[3] << ")\n";
      }
    };
    // the phase's thread-dependent predicates; versioned when few and warp-uniform (no lane bits)
    VCtx vc;
    bool versioned = jit_vmax() > 0;
    {
      u64 lanes = 0;
      for (int j = 0; j < 5 && j < A.nthr; ++j) lanes |= 1ull << A.tpos[F.thr[j]];
      auto add = [&](int kind, u64 m, u64 v) {
        if (m & lanes) versioned = false;
        for (const VPred& q : vc.preds)
          if (q.kind == kind && q.m == m && q.v == v) return;
        vc.preds.push_back({kind, m, v});
      };
      for (int oi = F.op_begin; oi < F.op_end; ++oi) {
        const FOp& op = prog.ops[oi];
        if (op.fk) add(0, op.fpm, op.fpv);
        if (op.pm != 0 || op.pv != 0) add(0, op.pm, op.pv);
        if (op.cs >= CS_PARITY && op.cs < CS_PARITY + 16 && op.xm) add(1, op.xm, 0);
      }
      if (vc.preds.empty() || int(vc.preds.size()) > jit_vmax()) versioned = false;
    }
    if (!versioned) {
      // lane-free predicates (at most 32): evaluated once per phase into a warp-uniform register
      UPreds up;
      bool uni = jit_uniform_preds() && !vc.preds.empty() && vc.preds.size() <= 32;
      {
        u64 lanes = 0;
        for (int j = 0; j < 5 && j < A.nthr; ++j) lanes |= 1ull << A.tpos[F.thr[j]];
        for (const VPred& q : vc.preds)
          if (q.m & lanes) uni = false;
      }
      if (uni) {
        up.preds = vc.preds;
        o << "    const unsigned vp_ = __reduce_or_sync(0xffffffffu, 0u";
        for (size_t q = 0; q < up.preds.size(); ++q) {
          const VPred& P = up.preds[q];
          if (P.kind == 0) o << " | (((pb & " << hex64(P.m) << ") == " << hex64(P.v) << ") ? " << (1u << q) << "u : 0u)";
          else o << " | (unsigned(__popcll(pb & " << hex64(P.m) << ") & 1) << " << q << ")";
        }
        o << ");\n";
      }
      int dyn = 0;
      static const bool exp_noops = getenv("SVB200_JIT_EXP_NOOPS") && std::string(getenv("SVB200_JIT_EXP_NOOPS")) == "1";
      for (int oi = F.op_begin; oi < F.op_end && !exp_noops; ++oi)   // (NOOPS: timing experiment, wrong results)
        if (!emit_op(g, oi - A.op_begin, prog.ops[oi], parity_tab_of(prog.ops[oi]), dyn, nullptr, uni ? &up : nullptr))
          return std::string();
      emit_store();
    } else {
      o << "    const int ver_ = 0";
      for (size_t q = 0; q < vc.preds.size(); ++q) {
        const VPred& P = vc.preds[q];
        if (P.kind == 0) o << " | (((pb & " << hex64(P.m) << ") == " << hex64(P.v) << ") ? " << (1 << q) << " : 0)";
        else o << " | ((__popcll(pb & " << hex64(P.m) << ") & 1) << " << q << ")";
      }
      o << ";\n    switch (ver_) {\n";
      for (int v = 0; v < (1 << vc.preds.size()); ++v) {
        vc.ver = v;
        vc.fthr = 0;
        o << "    " << (v + 1 < (1 << int(vc.preds.size())) ? "case " + std::to_string(v) : std::string("default")) << ": {\n";
        int dyn = 0;
        for (int oi = F.op_begin; oi < F.op_end; ++oi)
          if (!emit_op(g, oi - A.op_begin, prog.ops[oi], parity_tab_of(prog.ops[oi]), dyn, &vc)) return std::string();
        o << "    {\n    const int fthr = " << vc.fthr << ";\n";
        emit_store();
        o << "    }\n    break;\n    }\n";
      }
      o << "    }\n";
    }
    o << "  }\n";
  }
  const size_t ncf = std::max<size_t>(g.cf_refs.size(), 1);
  // kernel parameter space: 32764 bytes (sm_70+, CUDA 12.1+); the fixed arguments use < 1 KiB
  if (ncf * sizeof(double2) + sizeof(void*) * 5 + 1024 > 32000) return std::string();
  std::ostringstream k;
  if (const char* st = getenv("SVB200_JIT_STAGGER")) {   // experiment: "ns,sel" (sel 0: upper half of the grid, 1: odd CTAs)
    int ns = 0, sel = 0;
    std::sscanf(st, "%d,%d", &ns, &sel);
    if (ns > 0) {
      k << "#define FDEV_STAGGER_NS " << ns << "\n";
      k << "#define FDEV_STAGGER_SEL " << (sel ? "(blockIdx.x & 1)" : "(blockIdx.x >= gridDim.x / 2)") << "\n";
    }
  }
  if (split) k << "#define FDEV_SPLIT 1\n#define FDEV_HB " << (1 << (A.b - 1)) << "\n";
  if (pp) k << "#define FDEV_PP 1\n";
  if (getenv("SVB200_JIT_EXP_NOMEM") && std::string(getenv("SVB200_JIT_EXP_NOMEM")) == "1") k << "#define FDEV_EXP_NOMEM 1\n";
  static const bool pp_free = getenv("SVB200_JIT_PP_FREE") && std::string(getenv("SVB200_JIT_PP_FREE")) == "1";
  if (pp && pp_free) k << "#define FDEV_PP_FREE 1\n";
  static const bool segprof = getenv("SVB200_JIT_SEGPROF") && std::string(getenv("SVB200_JIT_SEGPROF")) == "1";
  if (pp && segprof) k << "#define FDEV_SEGPROF 1\n";
  static const bool plain_st = getenv("SVB200_JIT_STCS") && std::string(getenv("SVB200_JIT_STCS")) == "0";
  if (plain_st) k << "#define FDEV_PLAIN_STORE 1\n";
  k << "struct SvCf { double2 v[" << ncf << "]; };\n";
  if (pp) k << "extern \"C\" __global__ void __launch_bounds__(512, 1)\n";
  else k << "extern \"C\" __global__ void __launch_bounds__(256, " << (db ? 1 : jit_ctas_per_sm()) << ")\n";
  k << "svb200_pass(double2* __restrict__ state, double2* __restrict__ state_hi, const fdev::DPass P,\n"
       "            const fdev::DPhase* __restrict__ phases, const double2* __restrict__ tabs,\n"
       "            double2* __restrict__ gen_partials, const SvCf cf) {\n";
  if (pp) {
    k << "  (void)phases;\n";
    k << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n";
    k << "  double2* __restrict__ tile = reinterpret_cast<double2*>(smem_raw);   // 3 buffers; tile_off picks one\n";
    k << "  auto body = [&](const int tile_off, const u64 base, double2* __restrict__ acc_warp, auto next_load) {\n";
    k << "  (void)acc_warp; (void)tabs; (void)next_load;\n";
    k << o.str();
    k << "  };\n";
    k << "  fdev::run_pass_pp<" << (two ? "true" : "false") << ">(state, state_hi, P, gen_partials, body);\n}\n";
  } else {
    k << "  auto body = [&](double2* __restrict__ tile, double2* __restrict__ tile_hi,\n"
         "                  const fdev::DPhase* __restrict__ s_ph, const u64 base, double2* __restrict__ acc_warp,\n"
         "                  auto next_load) {\n";
    k << "  (void)acc_warp; (void)tabs; (void)next_load; (void)tile_hi;\n";
    k << o.str();
    k << "  };\n";
    k << "  fdev::run_pass<" << (two ? "true" : "false") << ", " << (db ? "true" : "false") << ", "
      << (direct ? "true" : "false") << ", decltype(body), " << (split ? "true" : "false") << ", "
      << (dfl ? "true" : "false") << ">(state, state_hi, P, phases, gen_partials, body);\n}\n";
  }

  if (cf_refs) *cf_refs = g.cf_refs;
  if (tab_refs) *tab_refs = g.tab_refs;
  return k.str();
}

// Compile (or find) the kernels of every pass of a program; fills prog.jit (nullptr = interpreter).
void jit_prepare(Program& prog, bool two) {
  if (prog.jit_ready && prog.jit_two == two) return;
  prog.jit.assign(prog.passes.size(), JitPass());
  prog.jit_tabs.clear();
  prog.jit_ready = true;
  prog.jit_two = two;
  if (!jit_enabled()) return;
  std::vector<std::shared_ptr<JitKernel>> todo;
  for (size_t p = 0; p < prog.passes.size(); ++p) {
    JitPass& jp = prog.jit[p];
    std::string src = jit_pass_source(prog, int(p), two, jit_db(), &jp.cf_refs, &jp.tab_refs);
    if (src.empty()) continue;
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = g_jit.find(src);
    if (it == g_jit.end()) {
      auto k = std::make_shared<JitKernel>();
      k->src = src;
      it = g_jit.emplace(src, k).first;
      todo.push_back(k);
    }
    jp.kernel = it->second;
    jp.split = src.find("#define FDEV_SPLIT") != std::string::npos;
    jp.pp = src.find("#define FDEV_PP") != std::string::npos;
  }
  if (const char* dump = getenv("SVB200_JIT_DUMP")) {   // debugging: write the generated sources
    for (size_t i = 0; i < todo.size(); ++i) {
      const std::string fn = std::string(dump) + "/pass_" + std::to_string(g_jit_compiled.load() + int64_t(i)) + ".cu";
      if (FILE* f = std::fopen(fn.c_str(), "w")) {
        std::fputs(kDevSrc, f);
        std::fputs(todo[i]->src.c_str(), f);
        std::fclose(f);
      }
    }
  }
  if (!todo.empty()) {
    // distinct pass structures compile in parallel (NVRTC programs are independent)
    const int nth = std::max(1, std::min<int>(int(todo.size()), int(std::thread::hardware_concurrency())));
    std::atomic<size_t> next{0};
    std::vector<std::thread> ths;
    for (int t = 0; t < nth; ++t)
      ths.emplace_back([&]() {
        for (size_t i = next++; i < todo.size(); i = next++) compile_kernel(*todo[i]);
      });
    for (auto& th : ths) th.join();
    for (auto& k : todo)
      if (!k->ok) {
        std::lock_guard<std::mutex> lk(g_jit_mu);
        g_jit.erase(k->src);
        sv_fail(SV_ERR_DEVICE, "pass compiler (NVRTC) failed:\n" + k->log.substr(0, 4000));
      }
  }
  // per-pass parameter blocks and the device table layout (values are fixed per program)
  for (size_t p = 0; p < prog.passes.size(); ++p) {
    JitPass& jp = prog.jit[p];
    if (!jp.kernel) continue;
    const FPassArgs& A = prog.passes[p];
    jp.cf.assign(std::max<size_t>(jp.cf_refs.size(), 1), make_double2(0.0, 0.0));
    for (size_t r = 0; r < jp.cf_refs.size(); ++r) {
      const FOp& op = prog.ops[A.op_begin + jp.cf_refs[r].first];
      const int j = jp.cf_refs[r].second;   // -1: coef[tab + 1]; 16 + r: coef[tab + r]; else inline c[j]
      jp.cf[r] = j < 0 ? prog.coef[op.tab + 1] : (j >= 16 ? prog.coef[op.tab + j - 16] : op.c[j]);
    }
    jp.tab_base = int(prog.jit_tabs.size());
    for (const auto& tr : jp.tab_refs) {
      const FOp& op = prog.ops[A.op_begin + tr.first];
      for (int j = 0; j < tr.second; ++j) prog.jit_tabs.push_back(prog.coef[op.tab + j]);
    }
  }
}

bool jit_launch(const JitPass& jp, int device, unsigned grid, int threads, size_t smem, cudaStream_t st, double2* state,
                double2* state_hi, const void* dpass, const void* phases, const double2* tabs, double2* gen) {
  JitKernel& k = *jp.kernel;
  {
    std::lock_guard<std::mutex> lk(k.mu);
    if (!k.lib) {
      CUDA_CHECK(cudaLibraryLoadData(&k.lib, k.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
      CUDA_CHECK(cudaLibraryGetKernel(&k.kern, k.lib, "svb200_pass"));
    }
    if (device < 0 || device >= 64) sv_fail(SV_ERR_DEVICE, "device ordinal out of range");
    if (k.smem_set[device] < int(smem)) {
      CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k.kern),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      k.smem_set[device] = int(smem);
    }
  }
  const double2* tb = tabs + jp.tab_base;
  void* args[] = {&state, &state_hi, const_cast<void*>(dpass), const_cast<void**>(&phases),
                  const_cast<const double2**>(&tb), &gen, const_cast<double2*>(jp.cf.data())};
  CUDA_CHECK(cudaLaunchKernel(reinterpret_cast<const void*>(k.kern), dim3(grid), dim3(threads), args, smem, st));
  return true;
}

void jit_stats(int64_t* compiled, int64_t* compile_us, int64_t* cached) {
  *compiled = g_jit_compiled.load();
  *compile_us = g_jit_compile_us.load();
  std::lock_guard<std::mutex> lk(g_jit_mu);
  *cached = int64_t(g_jit.size());
}

}  // namespace fused
