// C-ABI of libsvb200 (include/svb200.h): handle lifecycle, validation with the reference's
// error taxonomy, op-list execution, measurements and the adjoint-Jacobian driver.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstring>
#include <functional>
#include <map>
#include <new>

#include "dist.h"
#include "fused_jit.h"
#include "prim_util.h"
#include "sv_internal.h"

namespace {
thread_local std::string g_last_error;
}

[[noreturn]] void sv_fail(int status, const std::string& msg) { throw SvError{status, msg}; }

void sv_cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    sv_fail(SV_ERR_CAPACITY, std::string("device allocation failed: ") + what);
  }
  sv_fail(SV_ERR_DEVICE, std::string(cudaGetErrorString(e)) + " in " + what);
}

void sv_nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  sv_fail(SV_ERR_DEVICE, std::string("NCCL: ") + ncclGetErrorString(r) + " in " + what);
}

#define API_BEGIN try {
#define API_END                                  \
  return SV_OK;                                  \
  }                                              \
  catch (const SvError& e) {                     \
    g_last_error = e.msg;                        \
    return e.status;                             \
  }                                              \
  catch (const std::bad_alloc&) {                \
    g_last_error = "host allocation failed";     \
    return SV_ERR_CAPACITY;                      \
  }                                              \
  catch (const std::exception& e) {              \
    g_last_error = e.what();                     \
    return SV_ERR_DEVICE;                        \
  }

// ---------------------------------------------------------------------------
// scratch / stats helpers
// ---------------------------------------------------------------------------
void ensure_partials(sv_handle* h, size_t doubles) {
  if (h->partials_cap >= doubles) return;
  if (h->d_partials) {
    stream_sync(h);
    CUDA_CHECK(cudaFree(h->d_partials));
  }
  size_t cap = std::max<size_t>(doubles, 4096);
  CUDA_CHECK(cudaMalloc(&h->d_partials, cap * sizeof(double)));
  h->partials_cap = cap;
}

void ensure_results(sv_handle* h, size_t doubles) {
  if (h->results_cap >= doubles) return;
  if (h->d_results) {
    stream_sync(h);
    CUDA_CHECK(cudaFree(h->d_results));
  }
  size_t cap = std::max<size_t>(doubles, 1024);
  CUDA_CHECK(cudaMalloc(&h->d_results, cap * sizeof(double)));
  h->results_cap = cap;
}

// Wait for the handle's stream.  Sharded handles poll instead of blocking: a peer that failed (or
// died) leaves this rank's NCCL kernels waiting forever, so after SVB200_NCCL_TIMEOUT seconds
// (default 600) -- or as soon as NCCL reports an asynchronous error -- the communicator is
// aborted (ncclCommAbort, which also tears down the waiting kernels) and the call fails with a
// device error instead of hanging every rank.
void host_prof_mark(const char* what) {
  static const bool on = getenv("SVB200_HOST_PROF") && std::string(getenv("SVB200_HOST_PROF")) == "1";
  if (!on) return;
  static auto last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[host_prof] %-28s +%.3f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

void stream_sync(sv_handle* h) {
  if (!h->comm) {
    CUDA_CHECK(cudaStreamSynchronize(h->stream));
    return;
  }
  static const double timeout_s = getenv("SVB200_NCCL_TIMEOUT") ? atof(getenv("SVB200_NCCL_TIMEOUT")) : 600.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(h->stream);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) CUDA_CHECK(e);
    ncclResult_t ae = ncclSuccess;
    ncclCommGetAsyncError(h->comm, &ae);
    const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ae != ncclSuccess && ae != ncclInProgress) || waited > timeout_s) {
      dist_abort(h);
      sv_fail(SV_ERR_DEVICE, ae != ncclSuccess && ae != ncclInProgress
                                 ? std::string("NCCL asynchronous error: ") + ncclGetErrorString(ae) + "; communicator aborted"
                                 : "no progress for " + std::to_string(int(waited)) +
                                       " s (a peer rank failed?); communicator aborted");
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

static double* ensure_pinned(sv_handle* h, size_t doubles);

// Small device->host result copy through the handle's pinned buffer + stream_sync: a copy into
// pageable memory would block inside cudaMemcpyAsync, out of the watchdog's reach.
void d2h(sv_handle* h, void* host, const void* dev, size_t bytes) {
  double* pin = ensure_pinned(h, (bytes + sizeof(double) - 1) / sizeof(double));
  CUDA_CHECK(cudaMemcpyAsync(pin, dev, bytes, cudaMemcpyDeviceToHost, h->stream));
  stream_sync(h);
  std::memcpy(host, pin, bytes);
}

static double* ensure_pinned(sv_handle* h, size_t doubles) {
  if (h->h_pinned_cap < doubles) {
    if (h->h_pinned) cudaFreeHost(h->h_pinned);
    size_t cap = std::max<size_t>(doubles, 1024);
    CUDA_CHECK(cudaMallocHost(&h->h_pinned, cap * sizeof(double)));
    h->h_pinned_cap = cap;
  }
  return h->h_pinned;
}

static cudaEvent_t pool_event(sv_handle* h) {
  if (!h->event_pool.empty()) {
    cudaEvent_t e = h->event_pool.back();
    h->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CUDA_CHECK(cudaEventCreate(&e));
  return e;
}

void stat_begin(sv_handle* h, int cls, double bytes, cudaEvent_t* ev) {
  (void)cls;
  (void)bytes;
  if (!h->profiling) return;
  ev[0] = pool_event(h);
  ev[1] = pool_event(h);
  CUDA_CHECK(cudaEventRecord(ev[0], h->stream));
}

void stat_end(sv_handle* h, int cls, double bytes, cudaEvent_t* ev) {
  h->launches++;
  h->kc_launches[cls] += 1;
  h->kc_bytes[cls] += bytes;
  if (!h->profiling) return;
  CUDA_CHECK(cudaEventRecord(ev[1], h->stream));
  h->pending.push_back({cls, bytes, ev[0], ev[1]});
}

static void drain_timings(sv_handle* h) {
  if (h->pending.empty()) return;
  stream_sync(h);
  for (auto& p : h->pending) {
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, p.start, p.stop));
    h->kc_ms[p.cls] += ms;
    h->event_pool.push_back(p.start);
    h->event_pool.push_back(p.stop);
  }
  h->pending.clear();
}

// ---------------------------------------------------------------------------
// op execution
// ---------------------------------------------------------------------------
// Every entry point makes the handle's GPU current for the calling thread, so handles on
// different GPUs can be driven from worker threads of one process (observable batching).
static void check_handle(const sv_handle* h) {
  if (!h) sv_fail(SV_ERR_VALIDATION, "null device handle (released?)");
  if (!h->recording) CUDA_CHECK(cudaSetDevice(h->device));
}

static void exec_prims(sv_handle* h, const std::vector<double2*>& states, std::vector<Prim>& prims, int fuse) {
  if (prims.empty()) return;
  fold_diag_phases(prims);
  if (fuse && !h->recording && h->prec == 64) {   // the fusion engine is complex128-only
    // fused passes may relabel qubits inside their tiles: the qubit at local position p ends at perm[p]
    const std::vector<int> perm = apply_prims_fused(h, states, prims);
    for (int o = 0; o < h->n; ++o)
      if (h->phys[o] < h->nl) h->phys[o] = perm[h->phys[o]];
  } else {
    for (double2* st : states)
      for (const Prim& p : prims) launch_prim(h, st, p);
  }
  prims.clear();
}

// Lower and run an op list on `states` (psi, plus lambdas during the adjoint sweep all share
// the layout).  Global-qubit targets trigger a layout swap first (dist.cpp).
// Sharded schedule: lower everything to primitives on LOGICAL bit offsets, then repeatedly run
// the largest batch of primitives whose dense targets are local (a primitive may only move
// past deferred ones it commutes with); when nothing is runnable, swap the global qubit the
// next primitive needs with the local qubit whose next dense use is furthest away (Belady).
// Controls and diagonal bits on global qubits never need a swap (resolve_global).
// `exec` receives each batch already relabeled to physical positions and resolved against
// this rank's global bits (the forward pass and the fused adjoint sweep share this schedule).
// this rank's view of a batch: global controls / diagonal bits resolved, skipped prims dropped
static void resolve_batch(sv_handle* h, std::vector<Prim>& batch) {
  std::vector<Prim> out;
  out.reserve(batch.size());
  for (Prim& p : batch) {
    resolve_global(p, h->nl, h->rank);
    if (!p.skip) out.push_back(p);
  }
  batch.swap(out);
}

static void schedule_sharded(sv_handle* h, const std::vector<double2*>& states, const std::vector<Prim>& L,
                             const std::function<void(std::vector<Prim>&)>& exec) {
  std::vector<PrimReq> req(L.size());
  for (size_t i = 0; i < L.size(); ++i) req[i] = prim_requirements(L[i]);
  std::vector<int> rem(L.size());
  for (size_t i = 0; i < L.size(); ++i) rem[i] = int(i);
  while (!rem.empty()) {
    DeferredSet def;
    std::vector<int> batch, rest;
    for (int i : rem) {
      bool local = true;
      for (int o = 0; o < h->n; ++o)
        if (((req[i].dense >> o) & 1) && h->phys[o] >= h->nl) local = false;
      if (local && !def.blocks(req[i])) {
        batch.push_back(i);
      } else {
        def.add(req[i]);
        rest.push_back(i);
      }
    }
    if (!batch.empty()) {
      // physical positions; controls / diagonal bits on global positions are NOT resolved here:
      // the batch is identical on every rank, and exec resolves it (resolve_global) or runs it
      // rank-uniformly (fused programs evaluate global bits in the kernel)
      std::vector<Prim> phys_prims;
      for (int i : batch) {
        Prim p = L[i];
        relabel_prim(p, h->phys.data());
        if (!p.skip) phys_prims.push_back(p);
      }
      exec(phys_prims);
      rem.swap(rest);
      continue;
    }
    // stuck: bring the first primitive's global dense targets local
    std::vector<int> next_use(h->n, 1 << 30);
    for (size_t k = 0; k < rem.size(); ++k)
      for (int o = 0; o < h->n; ++o)
        if (((req[rem[k]].dense >> o) & 1) && next_use[o] > int(k)) next_use[o] = int(k);
    std::vector<int> keep;
    for (int o = 0; o < h->n; ++o)
      if ((req[rem[0]].dense >> o) & 1) keep.push_back(o);
    dist_bring_local(h, states, keep, next_use);
  }
}

static void run_ops_sharded(sv_handle* h, const std::vector<double2*>& states, const sv_op* ops, int n_ops,
                            int fuse) {
  std::vector<Prim> L;
  for (int i = 0; i < n_ops; ++i) {
    int col = 0;
    for (auto& pc : lower_op(ops[i], h->n, col, false, nullptr))
      if (!pc.fwd.skip) L.push_back(pc.fwd);
  }
  static const bool uniform_on = !(getenv("SVB200_RANK_UNIFORM") && std::string(getenv("SVB200_RANK_UNIFORM")) == "0");
  schedule_sharded(h, states, L, [&](std::vector<Prim>& batch) {
    if (uniform_on && fuse && !h->recording && h->prec == 64 && h->nl >= 5) {
      // one program for every rank (global bits evaluated in the kernel): in-tile relabeling allowed
      fold_diag_phases(batch);
      const std::vector<int> perm = apply_prims_fused(h, states, batch, nullptr, nullptr, true, true);
      for (int o = 0; o < h->n; ++o)
        if (h->phys[o] < h->nl) h->phys[o] = perm[h->phys[o]];
      batch.clear();
      return;
    }
    resolve_batch(h, batch);
    exec_prims(h, states, batch, fuse);
  });
}

// Single GPU: undo the qubit relabeling that fused passes leave behind (qubit at logical offset o
// back to physical position o) with ONE fused program of bit-SWAP primitives and no relabeling of
// its own -- SWAPs inside a tile are free register renamings, so this is a few pure-bandwidth
// passes (3 for the 30-qubit bench circuit's final layout) instead of one kernel per transposition.
static bool identity_layout(const sv_handle* h) {
  for (int o = 0; o < h->n; ++o)
    if (h->phys[o] != o) return false;
  return true;
}

static void canonicalize_single(sv_handle* h, const std::vector<double2*>& states) {
  if (identity_layout(h)) return;
  std::vector<int> at(h->nl);   // physical position -> logical offset
  for (int o = 0; o < h->n; ++o) at[h->phys[o]] = o;
  std::vector<Prim> swaps;
  for (int p = 0; p < h->nl; ++p)
    while (at[p] != p) {
      const int q = at[p];   // the qubit that belongs at q sits at p: exchange positions p and q
      Prim s;
      s.type = PRIM_PAIR;
      s.fmask = (1ull << p) | (1ull << q);
      s.fval = 1ull << p;
      s.xmask = s.fmask;
      s.m = {cplx(0), cplx(1), cplx(1), cplx(0)};
      swaps.push_back(s);
      std::swap(at[p], at[q]);
    }
  if (h->prec == 64) {
    apply_prims_fused(h, states, swaps, nullptr, nullptr, false);
  } else {
    for (double2* st : states)
      for (const Prim& p : swaps) launch_prim(h, st, p);
  }
  for (int o = 0; o < h->n; ++o) h->phys[o] = o;
}

// K14: from |0...0>, an op list that starts with H on every qubit followed by
// diagonal gates is ONE write-only pass: psi = 2^(-n/2) exp(i f), f = the Walsh expansion of the
// diagonal gates' phases (the reference's uniform start, state.py:41-45, plus e.g. QAOA's first
// cost layer), evaluated per 4096-amplitude tile by the WHT kernel.  Returns how many leading ops
// it consumed (0: not applicable -- the ops then run as usual).
static int try_uniform_prefix(sv_handle* h, const sv_op* ops, int n_ops) {
  static const bool off = getenv("SVB200_K14") && std::string(getenv("SVB200_K14")) == "0";
  if (off || !h->zero_state || h->recording || h->prec != 64 || h->nl < 12 || n_ops < h->n || !identity_layout(h))
    return 0;
  std::vector<char> seen(h->n, 0);
  for (int k = 0; k < h->n; ++k) {
    const sv_op& op = ops[k];
    if (op.kind != SV_GATE_H || op.n_wires != 1 || op.n_ctrls != 0) return 0;
    if (seen[op.wires[0]]) return 0;
    seen[op.wires[0]] = 1;
  }
  std::map<u64, double> walsh;   // physical bit mask -> coefficient of (-1)^pc(i & mask) in the phase
  int end = h->n;
  for (; end < n_ops; ++end) {
    int col = 0;
    const auto pieces = lower_op(ops[end], h->n, col, false, h->phys.data());
    bool diag = !pieces.empty();
    for (const auto& pc : pieces) {
      if (pc.fwd.type != PRIM_DIAG || pc.fwd.nb > 6 || popcount64(pc.fwd.fmask) > 4) diag = false;
      for (const cplx& t : pc.fwd.m)
        if (std::abs(std::abs(t) - 1.0) > 1e-12) diag = false;   // unit-modulus phases only
    }
    if (!diag) break;
    for (const auto& pc : pieces) {
      const Prim& p = pc.fwd;
      std::vector<int> bits(p.pos, p.pos + p.nb);   // S = table bits + control bits
      for (int b = 0; b < 64; ++b)
        if (((p.fmask >> b) & 1) && std::find(bits.begin(), bits.end(), b) == bits.end()) bits.push_back(b);
      const int k = int(bits.size());
      std::vector<double> theta(size_t(1) << k, 0.0);
      for (size_t x = 0; x < theta.size(); ++x) {
        u64 z = 0;
        for (int j = 0; j < k; ++j)
          if ((x >> j) & 1) z |= 1ull << bits[j];
        if ((z & p.fmask) != p.fval) continue;
        size_t t = 0;
        for (int j = 0; j < p.nb; ++j)
          if ((z >> p.pos[j]) & 1) t |= size_t(1) << j;
        theta[x] = std::arg(p.m[t]);
      }
      for (size_t sidx = 0; sidx < theta.size(); ++sidx) {   // Walsh coefficients over S
        double c = 0.0;
        for (size_t x = 0; x < theta.size(); ++x) c += (popcount64(x & sidx) & 1) ? -theta[x] : theta[x];
        c /= double(theta.size());
        if (c == 0.0) continue;
        u64 mask = 0;
        for (int j = 0; j < k; ++j)
          if ((sidx >> j) & 1) mask |= 1ull << bits[j];
        walsh[mask] += c;
      }
    }
  }
  std::vector<PauliTerm> terms;
  const u64 lmask = (h->nl >= 64) ? ~0ull : ((1ull << h->nl) - 1);
  for (const auto& e : walsh) {
    const bool neg = popcount64(u64(h->rank) & (e.first >> h->nl)) & 1;   // global bits: this rank's values
    terms.push_back({e.first & lmask, cplx(neg ? -e.second : e.second, 0.0)});
  }
  init_uniform_phase(h, h->state, terms, std::pow(2.0, -0.5 * double(h->n)));
  return end;
}

static void run_ops(sv_handle* h, const std::vector<double2*>& states, const sv_op* ops, int n_ops, int fuse) {
  if (fuse && states.size() == 1 && states[0] == h->state) {
    const int done = try_uniform_prefix(h, ops, n_ops);
    ops += done;
    n_ops -= done;
  }
  h->zero_state = false;
  // plans and generated kernels are keyed by the physical layout: an apply on a relabeled state
  // first restores the canonical layout, so repeated applies reuse the same program
  if (h->world == 1 && fuse && !h->recording && n_ops > 0) canonicalize_single(h, states);
  if (h->world > 1) {
    run_ops_sharded(h, states, ops, n_ops, fuse);
    return;
  }
  std::vector<Prim> pending;
  for (int i = 0; i < n_ops; ++i) {
    const sv_op& op = ops[i];
    int dummy = 0;
    auto pieces = lower_op(op, h->n, dummy, false, h->phys.data());
    if (h->world > 1) {
      bool need = false;
      for (auto& pc : pieces) need |= prim_needs_swap(pc.fwd, h->nl);
      if (need) {
        exec_prims(h, states, pending, fuse);
        dist_make_local(h, states, std::vector<int>(op.wires, op.wires + op.n_wires));
        dummy = 0;
        pieces = lower_op(op, h->n, dummy, false, h->phys.data());
      }
    }
    for (auto& pc : pieces) {
      resolve_global(pc.fwd, h->nl, h->rank);
      if (!pc.fwd.skip) pending.push_back(pc.fwd);
    }
  }
  exec_prims(h, states, pending, fuse);
}

static void validate_ops(const sv_handle* h, const sv_op* ops, int n_ops) {
  if (n_ops < 0 || (n_ops > 0 && !ops)) sv_fail(SV_ERR_VALIDATION, "bad op list");
  for (int i = 0; i < n_ops; ++i) validate_op(ops[i], h->n);
}

// ---------------------------------------------------------------------------
// observables
// ---------------------------------------------------------------------------
struct PauliGroup {
  u64 x;
  std::vector<PauliTerm> terms;
};

// Terms of a PAULI / HAMILTONIAN observable in physical bits, grouped by x-mask (one read per group).
static std::vector<PauliGroup> pauli_groups(sv_handle* h, const sv_obs& o, const std::vector<double2*>& states) {
  if (o.type != SV_OBS_PAULI && o.type != SV_OBS_HAMILTONIAN) sv_fail(SV_ERR_VALIDATION, "not a Pauli observable");
  if (o.n_terms < 0 || (o.n_terms && (!o.term_len))) sv_fail(SV_ERR_VALIDATION, "malformed observable");
  if (o.type == SV_OBS_HAMILTONIAN && o.n_terms && !o.coeffs) sv_fail(SV_ERR_VALIDATION, "Hamiltonian without coefficients");
  struct Raw {
    std::vector<int> xw;
    u64 xl = 0, zl = 0;   // logical offsets
    int ny = 0;
    double c = 1.0;
  };
  std::vector<Raw> raw(o.n_terms);
  int at = 0;
  for (int t = 0; t < o.n_terms; ++t) {
    Raw& r = raw[t];
    r.c = (o.type == SV_OBS_HAMILTONIAN) ? o.coeffs[t] : 1.0;
    for (int f = 0; f < o.term_len[t]; ++f, ++at) {
      int w = o.term_wires[at];
      char p = o.term_paulis[at];
      if (w < 0 || w >= h->n)
        sv_fail(SV_ERR_VALIDATION, "wire " + std::to_string(w) + " out of range for " + std::to_string(h->n) + "-qubit register");
      u64 bit = 1ull << (h->n - 1 - w);
      if ((r.xl | r.zl) & bit) sv_fail(SV_ERR_VALIDATION, "duplicate wire within Pauli word");
      if (p == 'X') {
        r.xl |= bit;
        r.xw.push_back(w);
      } else if (p == 'Y') {
        r.xl |= bit;
        r.zl |= bit;
        r.ny++;
        r.xw.push_back(w);
      } else if (p == 'Z') {
        r.zl |= bit;
      } else if (p == 'I') {
        r.zl |= 0;   // identity factor still reserves the wire for the duplicate check
        r.xl |= 0;
      } else {
        sv_fail(SV_ERR_VALIDATION, std::string("unknown Pauli '") + p + "'");
      }
    }
  }
  // bring X/Y wires onto local bits (swaps permute every state sharing the layout)
  if (h->world > 1) {
    std::vector<int> xw;
    for (auto& r : raw)
      for (int w : r.xw) xw.push_back(w);
    std::sort(xw.begin(), xw.end());
    xw.erase(std::unique(xw.begin(), xw.end()), xw.end());
    dist_make_local_set(h, states, xw);
  }
  std::map<u64, PauliGroup> groups;
  const cplx ipow[4] = {cplx(1, 0), cplx(0, 1), cplx(-1, 0), cplx(0, -1)};
  for (auto& r : raw) {
    u64 xp = 0, zp = 0;
    for (int o2 = 0; o2 < h->n; ++o2) {
      int p = h->phys[o2];
      if ((r.xl >> o2) & 1) xp |= 1ull << p;
      if ((r.zl >> o2) & 1) zp |= 1ull << p;
    }
    cplx cc = r.c * ipow[r.ny & 3];
    u64 local = (h->nl >= 64) ? ~0ull : ((1ull << h->nl) - 1);
    if (zp & ~local) {
      u64 zg = (zp & ~local) >> h->nl;
      if (popcount64(zg & u64(h->rank)) & 1) cc = -cc;
      zp &= local;
    }
    auto& g = groups[xp];
    g.x = xp;
    g.terms.push_back({zp, cc});
  }
  std::vector<PauliGroup> out;
  for (auto& kv : groups) out.push_back(kv.second);
  return out;
}

// <psi|O|psi> summed on the host in fixed group order (device partials are deterministic)
// CSR structure checks (SPEC.md:273 invariants; malformed CSR -> validation error)
static void validate_csr(const sv_handle* h, const sv_obs& o) {
  if (o.csr_dim != (int64_t(1) << h->n))
    sv_fail(SV_ERR_VALIDATION, "CSR dimension " + std::to_string(o.csr_dim) + " != 2^" + std::to_string(h->n));
  if (!o.csr_indptr || o.csr_nnz < 0 || (o.csr_nnz > 0 && (!o.csr_indices || !o.csr_data)))
    sv_fail(SV_ERR_VALIDATION, "malformed CSR: missing arrays");
  if (o.csr_indptr[0] != 0 || o.csr_indptr[o.csr_dim] != o.csr_nnz)
    sv_fail(SV_ERR_VALIDATION, "malformed CSR: row pointers must start at 0 and end at nnz");
  for (int64_t r = 0; r < o.csr_dim; ++r)
    if (o.csr_indptr[r + 1] < o.csr_indptr[r]) sv_fail(SV_ERR_VALIDATION, "malformed CSR: row pointers not monotone");
  for (int64_t k = 0; k < o.csr_nnz; ++k)
    if (o.csr_indices[k] < 0 || o.csr_indices[k] >= o.csr_dim)
      sv_fail(SV_ERR_VALIDATION, "malformed CSR: column index out of range");
  if (h->world != 1)
    sv_fail(SV_ERR_UNSUPPORTED, "sparse observables on sharded states are not supported (single-GPU states only)");
}

static double expval_impl(sv_handle* h, const sv_obs& o) {
  if (o.type == SV_OBS_SPARSE) {
    validate_csr(h, o);
    return csr_apply_or_expval(h, o, h->state, nullptr);
  }
  if (o.type == SV_OBS_DENSE) {
    if (o.n_wires < 1 || !o.wires || !o.matrix) sv_fail(SV_ERR_VALIDATION, "malformed dense observable");
    sv_op op{};
    op.kind = SV_GATE_MATRIX;
    op.n_wires = o.n_wires;
    op.wires = o.wires;
    op.matrix = o.matrix;
    validate_op(op, h->n);
    std::vector<int> tw(o.wires, o.wires + o.n_wires);
    dist_make_local_set(h, {h->state}, tw);
    std::vector<cplx> m(size_t(1) << (2 * o.n_wires));
    for (size_t i = 0; i < m.size(); ++i) m[i] = cplx(o.matrix[2 * i], o.matrix[2 * i + 1]);
    Prim g = make_dense_prim(tw, m, h->n, {}, {}, h->phys.data());
    ensure_results(h, 2);
    double z[2];
    if (g.nb <= 4) {
      braket_prim_async(h, h->state, h->state, g, h->d_results);
      d2h(h, z, h->d_results, 2 * sizeof(double));
    } else {
      // 5+ wires: lambda = O psi in one extra buffer (smem DENSE kernel), then Re<psi|lambda>
      size_t free_b = 0, total_b = 0;
      CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
      const size_t bytes = h->n_local * amp_bytes(h);
      double lacking = (bytes + (64ull << 20) > free_b) ? 1.0 : 0.0;
      dist_allreduce_sum(h, &lacking, 1);
      if (lacking > 0) sv_fail(SV_ERR_CAPACITY, "dense observable on more than 4 wires needs one extra state buffer");
      double2* lam = nullptr;
      CUDA_CHECK(cudaMalloc(&lam, bytes));
      try {
        launch_copy(h, lam, h->state, h->n_local);
        launch_prim(h, lam, g);
        z[0] = reduce_dot_re(h, h->state, lam);
      } catch (...) {
        cudaFree(lam);
        throw;
      }
      CUDA_CHECK(cudaFree(lam));
    }
    double v = z[0];
    dist_allreduce_sum(h, &v, 1);
    return v;
  }
  auto groups = pauli_groups(h, o, {h->state});
  ensure_results(h, groups.size() + 1);
  // SVB200_EXPVAL_BATCH=1: non-diagonal x-groups in batches of 16 that share their psi reads through
  // L2 (k_pauli_expval_multi).  Measured slower on the config-5 Hamiltonian (28q, 1000 terms: 0.42 vs
  // 0.39 s): the per-group kernel's pair form does half the amplitude work with real weights, and
  // without it the batch is bound by its term loop, not DRAM -- so one launch per group stays.
  static const bool batch_on = getenv("SVB200_EXPVAL_BATCH") && std::string(getenv("SVB200_EXPVAL_BATCH")) == "1";
  size_t nres = 0;
  std::vector<std::pair<u64, std::vector<PauliTerm>>> offdiag;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    if (batch_on && groups[gi].x != 0 && groups.size() > 1) {
      offdiag.push_back({groups[gi].x, groups[gi].terms});
      continue;
    }
    pauli_group_expval_async(h, h->state, groups[gi].x, groups[gi].terms, h->d_results + nres);
    ++nres;
  }
  if (!offdiag.empty()) nres += size_t(pauli_groups_expval_batched(h, h->state, offdiag, h->d_results + nres));
  std::vector<double> vals(nres);
  if (nres) {
    d2h(h, vals.data(), h->d_results, nres * sizeof(double));
  }
  dist_allreduce_sum(h, vals.data(), vals.size());
  double s = 0.0;
  for (double v : vals) s += v;
  return s;
}

// lam = O psi (out of place), the lambda initialisation of the adjoint sweep
static void apply_observable(sv_handle* h, const sv_obs& o, const double2* psi, double2* lam,
                             const std::vector<double2*>& all_states) {
  if (o.type == SV_OBS_SPARSE) {
    validate_csr(h, o);
    csr_apply_or_expval(h, o, psi, lam);
    return;
  }
  if (o.type == SV_OBS_DENSE) {
    std::vector<int> tw(o.wires, o.wires + o.n_wires);
    dist_make_local_set(h, all_states, tw);
    std::vector<cplx> m(size_t(1) << (2 * o.n_wires));
    for (size_t i = 0; i < m.size(); ++i) m[i] = cplx(o.matrix[2 * i], o.matrix[2 * i + 1]);
    Prim g = make_dense_prim(tw, m, h->n, {}, {}, h->phys.data());
    launch_copy(h, lam, psi, h->n_local);
    launch_prim(h, lam, g);
    return;
  }
  auto groups = pauli_groups(h, o, all_states);
  if (groups.empty()) {
    CUDA_CHECK(cudaMemsetAsync(lam, 0, h->n_local * amp_bytes(h), h->stream));
    return;
  }
  std::vector<std::pair<u64, std::vector<PauliTerm>>> gl;
  for (auto& g : groups) gl.push_back({g.x, g.terms});
  pauli_groups_apply(h, psi, lam, gl);
}

static void free_aux(sv_handle* h) {
  for (auto* p : h->aux) dist_forget(h, p);
  for (auto* p : h->aux) cudaFree(p);
  h->aux.clear();
}

// Fused adjoint sweep (K11 on the K7 engine): psi (h->state) and lambda (its own array) are
// treated as one 2^(nl+1) state whose top bit -- pinned, never relabeled -- selects the array, so
// "apply U^dagger to both" is a plain fused program on nl+1 bits and each <lambda|G_k|psi> is a
// GEN op evaluated inside the tile: many gates and generators per HBM pass, no state copies.
// One sweep per observable from the saved final state.  Sharded handles run the same sweep
// through the sharded schedule (both arrays swap together; controls and diagonal tables on global
// bits resolve per rank) and sum the per-rank bra-kets with one allreduce.  Generators on <= 2
// targets (adjoint_fused checks).
static double adjoint_fused_row(sv_handle* h, const sv_op* ops, int n_ops, const sv_obs& obs, int ncols, double2* lam,
                                double* jac_row) {
  apply_observable(h, obs, h->state, lam, {h->state, lam});                      // lambda = O psi
  host_prof_mark("row: lambda enqueued");
  // reverse sweep on LOGICAL bit offsets; generators become bra-kets whose psi/lambda selector
  // (xmask) is set per batch to the top bit of the two-array state
  std::vector<Prim> prims;
  std::vector<double> prefactor(ncols, 0.0);
  std::vector<int> col_start(n_ops);
  int col = 0;
  for (int i = 0; i < n_ops; ++i) {
    col_start[i] = col;
    lower_op(ops[i], h->n, col, true, nullptr);
  }
  for (int i = n_ops - 1; i >= 0; --i) {
    int c0 = col_start[i];
    auto pieces = lower_op(ops[i], h->n, c0, true, nullptr);
    for (int pi = int(pieces.size()) - 1; pi >= 0; --pi) {
      Piece& pc = pieces[pi];
      if (pc.has_gen) {
        Prim g = pc.gen.g;
        g.type = PRIM_GEN;
        g.xmask = 0;
        g.slot = pc.gen.column;
        // diagonal generators (Z, ZZ, |1><1|) become table bra-kets: targets need not be in registers
        const size_t d = size_t(1) << g.nb;
        bool diag = true;
        for (size_t r = 0; r < d && diag; ++r)
          for (size_t c = 0; c < d; ++c)
            if (r != c && g.m[r * d + c] != 0.0) diag = false;
        if (diag) {
          std::vector<cplx> t(d);
          for (size_t r = 0; r < d; ++r) t[r] = g.m[r * d + r];
          u64 tb = 0;
          for (int j = 0; j < g.nb; ++j) tb |= 1ull << g.pos[j];
          g.type = PRIM_GEND;
          g.fmask &= ~tb;
          g.fval &= ~tb;
          g.m = t;
        }
        prefactor[pc.gen.column] = pc.gen.prefactor;
        prims.push_back(g);
      }
      if (!pc.inv.skip) prims.push_back(pc.inv);
    }
  }
  // im[0..ncols) = Im<lambda_k|G_k|psi_k> (this rank's part), im[ncols] = Re<psi|lambda> = <O>
  std::vector<double> im(ncols + 1, 0.0);
  host_prof_mark("row: prims built");
  im[ncols] = reduce_dot_re(h, h->state, lam);
  host_prof_mark("row: <psi|lambda> (synced)");
  const std::vector<double2*> both = {h->state, lam};
  static const bool uniform_on = !(getenv("SVB200_RANK_UNIFORM") && std::string(getenv("SVB200_RANK_UNIFORM")) == "0");
  const bool uniform = uniform_on && h->world > 1;
  schedule_sharded(h, both, prims, [&](std::vector<Prim>& batch) {
    if (uniform) {
      // rank-uniform program on the nl+1-bit two-array state: the psi/lambda selector takes
      // position nl, so global positions move up by one (gbits = rank << (nl + 1) in the kernels)
      const int nl0 = h->nl;
      auto up = [&](u64 m) { return (m & ((1ull << nl0) - 1)) | ((m >> nl0) << (nl0 + 1)); };
      for (Prim& p : batch) {
        p.fmask = up(p.fmask);
        p.fval = up(p.fval);
        for (int j = 0; j < p.nb; ++j)
          if (p.pos[j] >= nl0) ++p.pos[j];
      }
    } else {
      resolve_batch(h, batch);
    }
    const int top = h->nl;
    for (Prim& p : batch)
      if (p.type == PRIM_GEN || p.type == PRIM_GEND) p.xmask = 1ull << top;
    fold_diag_phases(batch);
    std::vector<std::pair<int, cplx>> gens;
    h->nl += 1;
    h->n_local *= 2;
    std::vector<int> perm;
    try {
      // psi = h->state, lambda = lam: one logical 2^(nl+1) state whose top bit (pinned) picks the array
      perm = apply_prims_fused(h, {h->state}, batch, &gens, lam, true, uniform);
    } catch (...) {
      h->nl -= 1;
      h->n_local /= 2;
      throw;
    }
    h->nl -= 1;
    h->n_local /= 2;
    if (perm[top] != top) sv_fail(SV_ERR_DEVICE, "internal: the psi/lambda bit was relabeled");
    for (int o = 0; o < h->n; ++o)
      if (h->phys[o] < top) h->phys[o] = perm[h->phys[o]];   // qubit at p moved to perm[p]
    for (auto& g : gens) im[g.first] += g.second.imag();
    batch.clear();
  });
  host_prof_mark("row: sweep returned");
  stream_sync(h);
  host_prof_mark("row: synced");
  dist_allreduce_sum(h, im.data(), im.size());
  for (int c = 0; c < ncols; ++c) jac_row[c] = -2.0 * prefactor[c] * im[c];
  return im[ncols];
}

static bool adjoint_fused(sv_handle* h, const sv_op* ops, int n_ops, const sv_obs* obs, int n_obs, int ncols,
                          double* jac, double* expvals) {
  // tiles need >= 32 threads (2^(b-4)) for the warp-level generator reduction: nl + 1 >= 9
  if (n_obs < 1 || h->nl + 1 < 9) return false;
  for (int i = 0; i < n_ops; ++i) {
    int c = 0;
    for (auto& pc : lower_op(ops[i], h->n, c, true, nullptr))
      if (pc.has_gen && pc.gen.g.nb > 2) return false;
  }
  // lambda (+ the saved final psi for several observables) are allocated once per handle and
  // kept (the SPEC's "preallocation of all required memory"), so repeated Jacobians do not pay
  // for mapping tens of GiB each call
  const size_t half = h->n_local * sizeof(double2);
  const int need = n_obs > 1 ? 2 : 1;
  size_t free_b = 0, total_b = 0;
  CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
  const int have = (h->adj_lam ? 1 : 0) + (h->adj_saved ? 1 : 0);
  double lacking = (size_t(std::max(0, need - have)) * half + (64ull << 20) > free_b) ? 1.0 : 0.0;
  dist_allreduce_sum(h, &lacking, 1);   // every rank must take the same path (collectives inside)
  if (lacking > 0) return false;
  if (!h->adj_lam) CUDA_CHECK(cudaMalloc(&h->adj_lam, half));
  if (need > 1 && !h->adj_saved) CUDA_CHECK(cudaMalloc(&h->adj_saved, half));

  host_prof_mark("adjoint: start");
  run_ops(h, {h->state}, ops, n_ops, 1);                       // forward pass (once)
  host_prof_mark("adjoint: forward enqueued");
  std::vector<double> ev(n_obs);
  double2* buf = h->adj_lam;   // lambda
  double2* saved = h->adj_saved;
  {
    const std::vector<int> phys_final = h->phys;
    if (n_obs > 1) launch_copy(h, saved, h->state, h->n_local);
    for (int k = 0; k < n_obs; ++k) {
      if (k > 0) {                                             // restart from the final state
        launch_copy(h, h->state, saved, h->n_local);
        h->phys = phys_final;
      }
      ev[k] = adjoint_fused_row(h, ops, n_ops, obs[k], ncols, buf, jac + size_t(k) * ncols);
    }
    if (expvals)
      for (int k = 0; k < n_obs; ++k) expvals[k] = ev[k];
  }
  return true;
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* sv_last_error(void) { return g_last_error.c_str(); }

int sv_device_count(int* out) {
  API_BEGIN
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *out = c;
  API_END
}

static void create_common(sv_handle* h, int n_qubits, int device) {
  if (n_qubits < 1) sv_fail(SV_ERR_VALIDATION, "n_qubits must be a positive integer, got " + std::to_string(n_qubits));
  if (n_qubits > 62) sv_fail(SV_ERR_CAPACITY, "n_qubits=" + std::to_string(n_qubits) + " exceeds the 62-qubit addressing limit");
  h->n = n_qubits;
  h->nl = n_qubits - h->g;
  if (h->nl < 1) sv_fail(SV_ERR_VALIDATION, "too many shards for " + std::to_string(n_qubits) + " qubits");
  h->n_local = 1ull << h->nl;
  h->device = device;
  h->phys.resize(n_qubits);
  for (int o = 0; o < n_qubits; ++o) h->phys[o] = o;
  CUDA_CHECK(cudaSetDevice(device));
  size_t free_b = 0, total_b = 0;
  CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
  const double need = double(h->n_local) * amp_bytes(h);
  if (h->nl >= 40 || need > double(free_b))
    sv_fail(SV_ERR_CAPACITY, "cannot allocate 2**" + std::to_string(h->nl) + " amplitudes (" + std::to_string(need / 1e9) +
                                 " GB) on device " + std::to_string(device) + " with " + std::to_string(free_b / 1e9) +
                                 " GB free");
  CUDA_CHECK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  CUDA_CHECK(cudaMalloc(&h->state, h->n_local * amp_bytes(h)));
  launch_init_zero(h, h->state, 0, h->rank == 0);
  stream_sync(h);
  h->zero_state = true;
}

static void release_adjoint_buffers(sv_handle* h) {
  if (h->adj_lam) dist_forget(h, h->adj_lam);
  if (h->adj_saved) dist_forget(h, h->adj_saved);
  if (h->adj_lam) cudaFree(h->adj_lam);
  if (h->adj_saved) cudaFree(h->adj_saved);
  h->adj_lam = h->adj_saved = nullptr;
}

static void destroy_handle(sv_handle* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  free_aux(h);
  release_adjoint_buffers(h);
  release_scratch(h);
  release_fused(h);
  dist_destroy(h);
  if (h->state) cudaFree(h->state);
  if (h->d_partials) cudaFree(h->d_partials);
  if (h->d_results) cudaFree(h->d_results);
  if (h->h_pinned) cudaFreeHost(h->h_pinned);
  for (auto& p : h->pending) {
    cudaEventDestroy(p.start);
    cudaEventDestroy(p.stop);
  }
  for (auto e : h->event_pool) cudaEventDestroy(e);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

int sv_create(int n_qubits, int device, sv_handle** out) {
  sv_handle* h = nullptr;
  API_BEGIN
  if (!out) sv_fail(SV_ERR_VALIDATION, "null output handle");
  *out = nullptr;
  h = new sv_handle();
  create_common(h, n_qubits, device);
  *out = h;
  h = nullptr;
  API_END
}

int sv_create_ex(int n_qubits, int device, int precision_bits, sv_handle** out) {
  sv_handle* h = nullptr;
  API_BEGIN
  if (!out) sv_fail(SV_ERR_VALIDATION, "null output handle");
  *out = nullptr;
  if (precision_bits != 64 && precision_bits != 32)
    sv_fail(SV_ERR_VALIDATION, "precision_bits must be 64 (complex128) or 32 (complex64)");
  h = new sv_handle();
  h->prec = precision_bits;
  create_common(h, n_qubits, device);
  *out = h;
  h = nullptr;
  API_END
}

int sv_set_state_c64(sv_handle* h, const float* amps, uint64_t n_amps) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->prec != 32) sv_fail(SV_ERR_VALIDATION, "complex128 state: use sv_set_state");
  if (!amps) sv_fail(SV_ERR_VALIDATION, "null amplitude buffer");
  if (n_amps != (1ull << h->n))
    sv_fail(SV_ERR_VALIDATION, "amplitude array length " + std::to_string(n_amps) + " does not match 2**" + std::to_string(h->n));
  dist_reset_layout(h);
  h->zero_state = false;
  CUDA_CHECK(cudaMemcpyAsync(h->state, amps, h->n_local * sizeof(float2), cudaMemcpyHostToDevice, h->stream));
  stream_sync(h);
  API_END
}

int sv_get_state_c64(sv_handle* h, float* out, uint64_t n_amps) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->prec != 32) sv_fail(SV_ERR_VALIDATION, "complex128 state: use sv_get_state");
  if (!out) sv_fail(SV_ERR_VALIDATION, "null output buffer");
  if (n_amps != (1ull << h->n))
    sv_fail(SV_ERR_VALIDATION, "output length " + std::to_string(n_amps) + " does not match 2**" + std::to_string(h->n));
  // complex64 handles never run the fusion engine, so the layout is the identity here
  CUDA_CHECK(cudaMemcpyAsync(out, h->state, h->n_local * sizeof(float2), cudaMemcpyDeviceToHost, h->stream));
  stream_sync(h);
  API_END
}

int sv_nccl_unique_id(void* out128) {
  API_BEGIN
  ncclUniqueId id;
  NCCL_CHECK(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  API_END
}

int sv_create_sharded(int n_qubits, int rank, int world, int device, const void* nccl_id, sv_handle** out) {
  sv_handle* h = nullptr;
  try {
    if (!out) sv_fail(SV_ERR_VALIDATION, "null output handle");
    *out = nullptr;
    if (world < 1 || (world & (world - 1))) sv_fail(SV_ERR_VALIDATION, "n_shards must be a power of two");
    if (rank < 0 || rank >= world) sv_fail(SV_ERR_VALIDATION, "rank out of range");
    h = new sv_handle();
    h->rank = rank;
    h->world = world;
    h->g = __builtin_ctz(unsigned(world));
    create_common(h, n_qubits, device);
    if (world > 1) dist_init(h, nccl_id);
    *out = h;
    return SV_OK;
  } catch (const SvError& e) {
    g_last_error = e.msg;
    destroy_handle(h);
    return e.status;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    destroy_handle(h);
    return SV_ERR_DEVICE;
  }
}

int sv_destroy(sv_handle* h) {
  API_BEGIN
  if (h && !h->recording) CUDA_CHECK(cudaSetDevice(h->device));
  destroy_handle(h);
  API_END
}

int sv_info(const sv_handle* h, int64_t* out6) {
  API_BEGIN
  check_handle(h);
  out6[0] = h->n;
  out6[1] = h->nl;
  out6[2] = h->rank;
  out6[3] = h->world;
  out6[4] = h->device;
  out6[5] = h->prec;
  API_END
}

int sv_reset(sv_handle* h) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  dist_reset_layout(h);
  launch_init_zero(h, h->state, 0, h->rank == 0);
  stream_sync(h);
  h->zero_state = true;
  API_END
}

int sv_set_basis_state(sv_handle* h, uint64_t index) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->n < 64 && index >= (1ull << h->n)) sv_fail(SV_ERR_VALIDATION, "basis index out of range");
  dist_reset_layout(h);
  h->zero_state = false;
  const u64 owner = index >> h->nl;
  launch_init_zero(h, h->state, index & (h->n_local - 1), owner == u64(h->rank));
  stream_sync(h);
  API_END
}

int sv_set_state(sv_handle* h, const double* amps, uint64_t n_amps) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  if (!amps) sv_fail(SV_ERR_VALIDATION, "null amplitude buffer");
  if (n_amps != (1ull << h->n))
    sv_fail(SV_ERR_VALIDATION, "amplitude array length " + std::to_string(n_amps) + " does not match 2**" + std::to_string(h->n));
  if (h->prec != 64) sv_fail(SV_ERR_VALIDATION, "complex64 state: use sv_set_state_c64");
  dist_reset_layout(h);
  h->zero_state = false;
  const double* src = amps + 2 * (u64(h->rank) << h->nl);
  CUDA_CHECK(cudaMemcpyAsync(h->state, src, h->n_local * sizeof(double2), cudaMemcpyHostToDevice, h->stream));
  stream_sync(h);
  API_END
}

int sv_get_state(sv_handle* h, double* out, uint64_t n_amps) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  if (!out) sv_fail(SV_ERR_VALIDATION, "null output buffer");
  if (n_amps != (1ull << h->n))
    sv_fail(SV_ERR_VALIDATION, "output length " + std::to_string(n_amps) + " does not match 2**" + std::to_string(h->n));
  if (h->prec != 64) sv_fail(SV_ERR_VALIDATION, "complex64 state: use sv_get_state_c64");
  if (h->world == 1) canonicalize_single(h, {h->state});
  else dist_canonicalize(h, {h->state});
  if (h->world == 1) {
    CUDA_CHECK(cudaMemcpyAsync(out, h->state, h->n_local * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
    stream_sync(h);
  } else {
    dist_gather_state(h, out);
  }
  API_END
}

int sv_norm(sv_handle* h, double* out) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  double s = reduce_norm2(h, h->state);
  dist_allreduce_sum(h, &s, 1);
  *out = std::sqrt(s);
  API_END
}

int sv_apply_ops(sv_handle* h, const sv_op* ops, int n_ops, int fuse) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  validate_ops(h, ops, n_ops);   // trainable flags are irrelevant for plain application
  run_ops(h, {h->state}, ops, n_ops, fuse);
  stream_sync(h);
  API_END
}

int sv_apply_single_qubit(sv_handle* h, int q, const double* m2x2) {
  API_BEGIN
  check_handle(h);
  if (q < 0 || q >= h->n)
    sv_fail(SV_ERR_VALIDATION, "qubit " + std::to_string(q) + " out of range for " + std::to_string(h->n) + "-qubit register");
  if (!m2x2) sv_fail(SV_ERR_VALIDATION, "null matrix");
  sv_op op{};
  op.kind = SV_GATE_MATRIX;
  op.n_wires = 1;
  op.wires = &q;
  op.matrix = m2x2;
  std::lock_guard<std::mutex> lk(h->mu);
  run_ops(h, {h->state}, &op, 1, 0);
  stream_sync(h);
  API_END
}

int sv_apply_controlled_single_qubit(sv_handle* h, const int32_t* ctrls, int n_ctrls, int q, const double* m2x2,
                                     const int32_t* ctrl_values) {
  API_BEGIN
  check_handle(h);
  if (q < 0 || q >= h->n)
    sv_fail(SV_ERR_VALIDATION, "qubit " + std::to_string(q) + " out of range for " + std::to_string(h->n) + "-qubit register");
  if (!m2x2) sv_fail(SV_ERR_VALIDATION, "null matrix");
  sv_op op{};
  op.kind = SV_GATE_CONTROLLED_MATRIX;
  op.n_wires = 1;
  op.wires = &q;
  op.n_ctrls = n_ctrls;
  op.ctrls = ctrls;
  op.ctrl_values = ctrl_values;
  op.matrix = m2x2;
  validate_op(op, h->n);
  std::lock_guard<std::mutex> lk(h->mu);
  run_ops(h, {h->state}, &op, 1, 0);
  stream_sync(h);
  API_END
}

int sv_apply_matrix(sv_handle* h, const int32_t* wires, int n_wires, const double* matrix) {
  API_BEGIN
  check_handle(h);
  if (!matrix) sv_fail(SV_ERR_VALIDATION, "null matrix");
  sv_op op{};
  op.kind = SV_GATE_MATRIX;
  op.n_wires = n_wires;
  op.wires = wires;
  op.matrix = matrix;
  validate_op(op, h->n);
  std::lock_guard<std::mutex> lk(h->mu);
  run_ops(h, {h->state}, &op, 1, 0);
  stream_sync(h);
  API_END
}

int sv_expval(sv_handle* h, const sv_obs* obs, double* out) {
  API_BEGIN
  check_handle(h);
  if (!obs || !out) sv_fail(SV_ERR_VALIDATION, "null observable");
  std::lock_guard<std::mutex> lk(h->mu);
  *out = expval_impl(h, *obs);
  API_END
}

// variance: a Pauli word squares to I, so Var = 1 - <P>^2; otherwise
// lambda = O psi (one extra state buffer) gives <O^2> = |lambda|^2 (O Hermitian) and <O> =
// Re<psi|lambda>, both local partial sums allreduced across shards.
int sv_var(sv_handle* h, const sv_obs* obs, double* out) {
  API_BEGIN
  check_handle(h);
  if (!obs || !out) sv_fail(SV_ERR_VALIDATION, "null observable");
  std::lock_guard<std::mutex> lk(h->mu);
  if (obs->type == SV_OBS_PAULI) {
    const double e = expval_impl(h, *obs);
    *out = 1.0 - e * e;
  } else {
    // lambda lives in the handle's adjoint buffer (allocated once, kept; registered for peer
    // swaps like any adjoint lambda and unmapped collectively when the handle releases it)
    const size_t bytes = h->n_local * sizeof(double2);
    size_t free_b = 0, total_b = 0;
    CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    double lacking = (!h->adj_lam && bytes + (64ull << 20) > free_b) ? 1.0 : 0.0;
    dist_allreduce_sum(h, &lacking, 1);
    if (lacking > 0) sv_fail(SV_ERR_CAPACITY, "variance needs one extra state buffer");
    expval_impl(h, *obs);   // validates the observable (and its wires) like expval
    if (!h->adj_lam) CUDA_CHECK(cudaMalloc(&h->adj_lam, bytes));
    double2* lam = h->adj_lam;
    apply_observable(h, *obs, h->state, lam, {h->state, lam});
    double v[2] = {reduce_norm2(h, lam), reduce_dot_re(h, h->state, lam)};
    dist_allreduce_sum(h, v, 2);
    *out = v[0] - v[1] * v[1];
  }
  API_END
}

static std::vector<int> measured_wires(const sv_handle* h, const int32_t* wires, int n_wires, const char* what) {
  std::vector<int> w;
  if (n_wires <= 0) {
    for (int q = 0; q < h->n; ++q) w.push_back(q);
    return w;
  }
  for (int i = 0; i < n_wires; ++i) {
    if (wires[i] < 0 || wires[i] >= h->n)
      sv_fail(SV_ERR_VALIDATION, "wire " + std::to_string(wires[i]) + " out of range for " + std::to_string(h->n) +
                                     "-qubit register");
    for (int j = 0; j < i; ++j)
      if (wires[j] == wires[i]) sv_fail(SV_ERR_VALIDATION, std::string("duplicate wires in ") + what);
    w.push_back(wires[i]);
  }
  return w;
}

int sv_probs(sv_handle* h, const int32_t* wires, int n_wires, double* out) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  const std::vector<int> w = measured_wires(h, wires, n_wires, "probabilities");
  if (w.size() > 40) sv_fail(SV_ERR_CAPACITY, "probability vector too large");
  dist_probs(h, w, out);
  API_END
}

// Deterministic sampling (sample_root SPEC.md:455-462): the marginal
// distribution comes from the device reduction (dist_probs: every rank holds the same vector),
// the inverse-CDF draw is the fixed procedure documented in svb200.h, so a sharded state and a
// single-GPU state give the same rows for the same seed.
static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

int sv_sample(sv_handle* h, const int32_t* wires, int n_wires, uint64_t shots, uint64_t seed, int64_t* out) {
  API_BEGIN
  check_handle(h);
  if (shots == 0) sv_fail(SV_ERR_VALIDATION, "shots must be >= 1");
  if (!out) sv_fail(SV_ERR_VALIDATION, "null output buffer");
  std::lock_guard<std::mutex> lk(h->mu);
  const std::vector<int> w = measured_wires(h, wires, n_wires, "sample");
  if (w.size() > 30) sv_fail(SV_ERR_CAPACITY, "sampling supports at most 30 measured wires");
  const size_t bins = size_t(1) << w.size();
  std::vector<double> c(bins);
  dist_probs(h, w, c.data());
  for (size_t b = 1; b < bins; ++b) c[b] += c[b - 1];   // sequential inclusive prefix
  const double total = c[bins - 1];
  for (uint64_t i = 0; i < shots; ++i) {
    const uint64_t x = splitmix64(seed + (i + 1) * 0x9E3779B97F4A7C15ull);
    const double u = double(x >> 11) * (1.0 / 9007199254740992.0) * total;
    size_t b = size_t(std::upper_bound(c.begin(), c.end(), u) - c.begin());
    if (b >= bins) b = bins - 1;
    out[i] = int64_t(b);
  }
  API_END
}

int sv_adjoint_jacobian(sv_handle* h, const sv_op* ops, int n_ops, const sv_obs* obs, int n_obs, int fuse, double* jac,
                        double* expvals) {
  API_BEGIN
  check_handle(h);
  std::lock_guard<std::mutex> lk(h->mu);
  validate_ops(h, ops, n_ops);
  if (n_obs < 0 || (n_obs > 0 && !obs)) sv_fail(SV_ERR_VALIDATION, "bad observable list");
  // lower once (logical layout) to learn columns and validate differentiability
  int ncols = 0;
  for (int i = 0; i < n_ops; ++i) lower_op(ops[i], h->n, ncols, true, nullptr);
  if (fuse && h->prec == 64 && adjoint_fused(h, ops, n_ops, obs, n_obs, ncols, jac, expvals)) return SV_OK;
  // capacity: one lambda per observable; the fused path's kept buffers go first
  release_adjoint_buffers(h);
  size_t free_b = 0, total_b = 0;
  CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
  const double need = double(n_obs) * double(h->n_local) * amp_bytes(h);
  if (need > double(free_b))
    sv_fail(SV_ERR_CAPACITY, "adjoint sweep needs " + std::to_string(n_obs) + " extra state copies (" +
                                 std::to_string(need / 1e9) + " GB) but only " + std::to_string(free_b / 1e9) + " GB are free");
  free_aux(h);
  for (int k = 0; k < n_obs; ++k) {
    double2* p = nullptr;
    CUDA_CHECK(cudaMalloc(&p, h->n_local * amp_bytes(h)));
    h->aux.push_back(p);
  }
  std::vector<double2*> lam_states = h->aux;
  std::vector<double2*> all = {h->state};
  all.insert(all.end(), lam_states.begin(), lam_states.end());

  // forward pass
  run_ops(h, {h->state}, ops, n_ops, fuse);
  // lambda_k = O_k psi ; expvals from Re<psi|lambda_k> via the expval kernels
  std::vector<double> ev(n_obs, 0.0);
  for (int k = 0; k < n_obs; ++k) ev[k] = expval_impl(h, obs[k]);
  for (int k = 0; k < n_obs; ++k) apply_observable(h, obs[k], h->state, lam_states[k], all);

  // reverse sweep
  adjoint_sweep(h, ops, n_ops, lam_states, ncols, fuse, jac);
  if (expvals)
    for (int k = 0; k < n_obs; ++k) expvals[k] = ev[k];
  free_aux(h);
  API_END
}

int sv_synchronize(sv_handle* h) {
  API_BEGIN
  check_handle(h);
  stream_sync(h);
  API_END
}

void* sv_stream(sv_handle* h) { return h ? (void*)h->stream : nullptr; }

int64_t sv_launch_count(const sv_handle* h) { return h ? h->launches : -1; }

int sv_set_profiling(sv_handle* h, int enabled) {
  API_BEGIN
  check_handle(h);
  drain_timings(h);
  h->profiling = enabled != 0;
  API_END
}

int sv_kernel_stats(sv_handle* h, double* out, int max_classes, int* n_classes, char* names, int names_len) {
  API_BEGIN
  check_handle(h);
  drain_timings(h);
  int n = std::min<int>(max_classes, KC_COUNT);
  for (int k = 0; k < n; ++k) {
    out[3 * k + 0] = h->kc_launches[k];
    out[3 * k + 1] = h->kc_ms[k];
    out[3 * k + 2] = h->kc_bytes[k];
  }
  if (n_classes) *n_classes = n;
  if (names && names_len > 0) {
    std::string s;
    for (int k = 0; k < KC_COUNT; ++k) s += std::string(kKernelClassNames[k]) + (k + 1 < KC_COUNT ? "," : "");
    std::strncpy(names, s.c_str(), names_len - 1);
    names[names_len - 1] = 0;
  }
  API_END
}

int sv_reset_stats(sv_handle* h) {
  API_BEGIN
  check_handle(h);
  drain_timings(h);
  for (int k = 0; k < KC_COUNT; ++k) h->kc_launches[k] = h->kc_ms[k] = h->kc_bytes[k] = 0;
  API_END
}

// the prim list exec_prims would fuse for this op list on one GPU (identity layout)
static std::vector<Prim> host_prims(int n_qubits, const sv_op* ops, int n_ops) {
  if (n_qubits < 1 || n_qubits > 62) sv_fail(SV_ERR_VALIDATION, "bad qubit count");
  if (n_ops < 0 || (n_ops > 0 && !ops)) sv_fail(SV_ERR_VALIDATION, "bad op list");
  std::vector<Prim> prims;
  int col = 0;
  for (int i = 0; i < n_ops; ++i) {
    validate_op(ops[i], n_qubits);
    for (auto& pc : lower_op(ops[i], n_qubits, col, false, nullptr))
      if (!pc.fwd.skip) prims.push_back(pc.fwd);
  }
  fold_diag_phases(prims);
  return prims;
}

int sv_plan_summary(int n_qubits, const sv_op* ops, int n_ops, int64_t* out4) {
  API_BEGIN
  PlanStats s = plan_stats(n_qubits, host_prims(n_qubits, ops, n_ops));
  out4[0] = s.passes;
  out4[1] = s.ops;
  out4[2] = s.tile_bits;
  out4[3] = s.phases;
  API_END
}

int sv_plan_fp64(int n_qubits, const sv_op* ops, int n_ops, double* flops_per_amp) {
  API_BEGIN
  *flops_per_amp = plan_stats(n_qubits, host_prims(n_qubits, ops, n_ops)).fp64_flops_per_amp;
  API_END
}

int sv_jit_stats(int64_t* out3) {
  API_BEGIN
  if (!out3) sv_fail(SV_ERR_VALIDATION, "null output");
  fused::jit_stats(&out3[0], &out3[1], &out3[2]);
  API_END
}

int sv_plan_compile(int n_qubits, const sv_op* ops, int n_ops, int two_array, int64_t* out4) {
  API_BEGIN
  if (n_qubits < 5 || n_qubits > 62) sv_fail(SV_ERR_VALIDATION, "bad qubit count");
  plan_compile(n_qubits, host_prims(n_qubits, ops, n_ops), two_array != 0, out4);
  API_END
}

// Host-only: run the sharded driver for `rank` of `world` in recording mode (no device memory,
// no NCCL) and return what it would execute -- local primitives and global-qubit swaps -- plus
// the canonicalising swaps at the end.  tests/test_sharded_cpu.py replays it on gloo ranks.
int sv_plan_sharded(int n_qubits, int rank, int world, const sv_op* ops, int n_ops, int64_t* ints, int64_t ints_cap,
                    double* dbls, int64_t dbls_cap, int64_t* sizes2) {
  API_BEGIN
  if (world < 1 || (world & (world - 1))) sv_fail(SV_ERR_VALIDATION, "n_shards must be a power of two");
  if (rank < 0 || rank >= world) sv_fail(SV_ERR_VALIDATION, "rank out of range");
  if (n_qubits < 1 || n_qubits > 62) sv_fail(SV_ERR_VALIDATION, "bad qubit count");
  sv_handle v;
  v.recording = true;
  v.rank = rank;
  v.world = world;
  v.g = __builtin_ctz(unsigned(world));
  v.n = n_qubits;
  v.nl = n_qubits - v.g;
  if (v.nl < 1) sv_fail(SV_ERR_VALIDATION, "too many shards");
  v.n_local = 1ull << v.nl;
  v.phys.resize(n_qubits);
  for (int o = 0; o < n_qubits; ++o) v.phys[o] = o;
  validate_ops(&v, ops, n_ops);
  run_ops(&v, {nullptr}, ops, n_ops, 0);
  dist_canonicalize(&v, {nullptr});
  std::vector<int64_t> I = {1, v.n, v.nl, v.rank, v.world, int64_t(v.rec.size())};
  std::vector<double> D;
  for (const RecStep& s : v.rec) {
    I.push_back(s.kind);
    if (s.kind == REC_GSWAP) {
      I.push_back(s.G);
      continue;
    }
    if (s.kind == REC_XSWAP) {
      I.push_back(int64_t(s.Gs.size()));
      for (size_t i = 0; i < s.Gs.size(); ++i) {
        I.push_back(s.Gs[i]);
        I.push_back(s.ps[i]);
      }
      continue;
    }
    const Prim& p = s.p;
    I.push_back(p.type);
    I.push_back(int64_t(p.fmask));
    I.push_back(int64_t(p.fval));
    I.push_back(int64_t(p.xmask));
    I.push_back(p.nb);
    for (int t = 0; t < p.nb; ++t) I.push_back(p.pos[t]);
    I.push_back(int64_t(D.size()) / 2);
    I.push_back(int64_t(p.m.size()));
    for (auto& c : p.m) {
      D.push_back(c.real());
      D.push_back(c.imag());
    }
  }
  for (int o = 0; o < v.n; ++o) I.push_back(v.phys[o]);
  sizes2[0] = int64_t(I.size());
  sizes2[1] = int64_t(D.size());
  if (ints && int64_t(I.size()) <= ints_cap) std::memcpy(ints, I.data(), I.size() * sizeof(int64_t));
  if (dbls && int64_t(D.size()) <= dbls_cap) std::memcpy(dbls, D.data(), D.size() * sizeof(double));
  API_END
}

int sv_plan_program(int n_qubits, const sv_op* ops, int n_ops, int64_t* ints, int64_t ints_cap, double* dbls,
                    int64_t dbls_cap, int64_t* sizes2) {
  API_BEGIN
  std::vector<int64_t> I;
  std::vector<double> D;
  plan_program_serialized(n_qubits, host_prims(n_qubits, ops, n_ops), I, D);
  sizes2[0] = int64_t(I.size());
  sizes2[1] = int64_t(D.size());
  if (ints && int64_t(I.size()) <= ints_cap) std::memcpy(ints, I.data(), I.size() * sizeof(int64_t));
  if (dbls && int64_t(D.size()) <= dbls_cap) std::memcpy(dbls, D.data(), D.size() * sizeof(double));
  API_END
}

}  // extern "C"

// ---------------------------------------------------------------------------
// adjoint reverse sweep (unfused reference schedule; the fused tile sweep lives in fused.cu)
// ---------------------------------------------------------------------------
void adjoint_sweep(sv_handle* h, const sv_op* ops, int n_ops, const std::vector<double2*>& lams, int ncols, int fuse,
                   double* jac) {
  const int n_obs = int(lams.size());
  std::vector<double2*> all = {h->state};
  all.insert(all.end(), lams.begin(), lams.end());
  // complex <lambda_k|G|psi> per (column, obs) accumulated into d_results
  ensure_results(h, size_t(ncols) * n_obs * 2 + 2);
  std::vector<double> prefactor(ncols, 0.0);
  // lower in forward order to know columns; then walk backwards
  struct Rec {
    int op;
    Piece pc;
  };
  int col = 0;
  std::vector<std::vector<Piece>> lowered(n_ops);
  std::vector<int> col_start(n_ops);
  for (int i = 0; i < n_ops; ++i) {
    col_start[i] = col;
    lowered[i] = lower_op(ops[i], h->n, col, true, nullptr);   // columns only; re-lowered with layout below
  }
  (void)fuse;
  for (int i = n_ops - 1; i >= 0; --i) {
    const sv_op& op = ops[i];
    int c0 = col_start[i];
    auto pieces = lower_op(op, h->n, c0, true, h->phys.data());
    if (h->world > 1) {
      bool need = false;
      for (auto& pc : pieces) need |= prim_needs_swap(pc.inv, h->nl) || (pc.has_gen && prim_needs_swap(pc.gen.g, h->nl));
      if (need) {
        dist_make_local(h, all, std::vector<int>(op.wires, op.wires + op.n_wires));
        c0 = col_start[i];
        pieces = lower_op(op, h->n, c0, true, h->phys.data());
      }
    }
    for (int pi = int(pieces.size()) - 1; pi >= 0; --pi) {
      Piece& pc = pieces[pi];
      if (pc.has_gen) {
        Prim g = pc.gen.g;
        resolve_global(g, h->nl, h->rank);
        prefactor[pc.gen.column] = pc.gen.prefactor;
        for (int k = 0; k < n_obs; ++k) {
          double* dst = h->d_results + 2 * (size_t(pc.gen.column) * n_obs + k);
          if (g.skip)
            CUDA_CHECK(cudaMemsetAsync(dst, 0, 2 * sizeof(double), h->stream));
          else
            braket_prim_async(h, lams[k], h->state, g, dst);
        }
      }
      Prim inv = pc.inv;
      resolve_global(inv, h->nl, h->rank);
      if (!inv.skip)
        for (double2* st : all) launch_prim(h, st, inv);
    }
  }
  std::vector<double> z(size_t(ncols) * n_obs * 2, 0.0);
  if (!z.empty()) {
    d2h(h, z.data(), h->d_results, z.size() * sizeof(double));
  }
  dist_allreduce_sum(h, z.data(), z.size());
  for (int k = 0; k < n_obs; ++k)
    for (int c = 0; c < ncols; ++c) jac[size_t(k) * ncols + c] = -2.0 * prefactor[c] * z[2 * (size_t(c) * n_obs + k) + 1];
}
