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
struct Gen {
  std::ostringstream o;
  std::vector<std::pair<int, int>> cf_refs;   // (pass-local op, c[] index)
  std::vector<std::pair<int, int>> tab_refs;  // (pass-local op, table length)
  int tab_len = 0;

  // j = -1: entry 1 of the op's coefficient table (the odd-parity value of a parity table)
  std::string C(int op, int j) {
    cf_refs.push_back({op, j});
    return "cf.v[" + std::to_string(cf_refs.size() - 1) + "]";
  }
  std::string T(int op, int len) {
    tab_refs.push_back({op, len});
    const int off = tab_len;
    tab_len += len;
    return "(tabs + " + std::to_string(off) + ")";
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

bool emit_op(Gen& g, int i, const FOp& op, bool parity_tab) {
  std::ostringstream& o = g.o;
  const int cs = op.cs;
  o << "    {\n";
  if (op.fk) o << "      if ((pb & " << hex64(op.fpm) << ") == " << hex64(op.fpv) << ") fthr ^= " << op.fk << ";\n";
  const bool has_pred = op.pm != 0 || op.pv != 0;
  const std::string pred = "((pb & " + hex64(op.pm) + ") == " + hex64(op.pv) + ")";
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
    o << "      fdev::gen_commit(re, im, acc_warp, " << op.slot << ");\n";
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
  } else if (cs >= CS_PARITY && cs < CS_PARITY + 16) {
    const int M = cs - CS_PARITY;
    std::string tp = "(__popc(fthr & " + std::to_string(M) + ") + " + std::to_string(int(op.v));
    if (op.xm) tp += " + __popcll(pb & " + hex64(op.xm) + ")";
    tp += ") & 1";
    o << "      fdev::parity_phase<" << M << ">(a, " << g.C(i, 0) << ", " << tp << ");\n";
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
  const bool split = split_on && direct && jit_ctas_per_sm() <= 2;
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
    if (tab_thr) {
      o << "    FDEV_PHASE_LOAD(s_ph[" << ph << "], " << W[0] << ", " << W[1] << ", " << W[2] << ", " << W[3] << ")\n";
    } else {
      // the thread's slot: swizzled offset and physical bits as literal-mask expressions of tid
      std::string se = "0", pe = "0ull";
      for (int j = 0; j < A.nthr; ++j) {
        const std::string bit = "((threadIdx.x >> " + std::to_string(j) + ") & 1)";
        se += " ^ (" + bit + " ? " + std::to_string(swz_h(1 << F.thr[j])) + " : 0)";
        pe += " | (" + bit + " ? " + hex64(1ull << A.tpos[F.thr[j]]) + " : 0ull)";
      }
      o << "    FDEV_PHASE_LOAD_X(" << se << ", " << pe << ", " << W[0] << ", " << W[1] << ", " << W[2] << ", " << W[3]
        << ")\n";
    }
    if (last_direct) o << "    __syncthreads();\n    next_load();\n";
    for (int oi = F.op_begin; oi < F.op_end; ++oi) {
      const FOp& op = prog.ops[oi];
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
      if (!emit_op(g, oi - A.op_begin, op, ptab)) return std::string();
    }
    if (last_direct) {
      o << "    FDEV_PHASE_STORE_GLOBAL" << (two ? "2(" : "(") << int(F.flip);
      for (int k = 0; k < 4; ++k) o << ", " << hex64(1ull << A.tpos_st[F.reg[k]]);
      o << ")\n";
    } else {
      o << "    FDEV_PHASE_STORE(" << int(F.flip) << ", " << W[0] << ", " << W[1] << ", " << W[2] << ", " << W[3] << ")\n";
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
  static const bool plain_st = getenv("SVB200_JIT_STCS") && std::string(getenv("SVB200_JIT_STCS")) == "0";
  if (plain_st) k << "#define FDEV_PLAIN_STORE 1\n";
  k << "struct SvCf { double2 v[" << ncf << "]; };\n";
  k << "extern \"C\" __global__ void __launch_bounds__(256, " << (db ? 1 : jit_ctas_per_sm()) << ")\n";
  k << "svb200_pass(double2* __restrict__ state, double2* __restrict__ state_hi, const fdev::DPass P,\n"
       "            const fdev::DPhase* __restrict__ phases, const double2* __restrict__ tabs,\n"
       "            double2* __restrict__ gen_partials, const SvCf cf) {\n";
  k << "  auto body = [&](double2* __restrict__ tile, double2* __restrict__ tile_hi,\n"
       "                  const fdev::DPhase* __restrict__ s_ph, const u64 base, double2* __restrict__ acc_warp,\n"
       "                  auto next_load) {\n";
  k << "  (void)acc_warp; (void)tabs; (void)next_load; (void)tile_hi;\n";
  k << o.str();
  k << "  };\n";
  k << "  fdev::run_pass<" << (two ? "true" : "false") << ", " << (db ? "true" : "false") << ", "
    << (direct ? "true" : "false") << ", decltype(body), " << (split ? "true" : "false")
    << ">(state, state_hi, P, phases, gen_partials, body);\n}\n";

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
      jp.cf[r] = jp.cf_refs[r].second < 0 ? prog.coef[op.tab + 1] : op.c[jp.cf_refs[r].second];
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
