// Sharded execution over NCCL: qubit-index swaps between a global (shard-index) bit and a
// local bit, reductions with ncclAllReduce, root-free state gather for I/O.
//
// Reference semantics: ShardedState with global qubits = top log2(n_shards) bits
// (SPEC.md:429-443); gates on local qubits need no messages; results equal
// the monolithic ones.  The SPEC's block exchange is replaced by
// index swaps as BASELINE.json's north_star asks, so its message-count law does not apply.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "dist.h"

namespace {
constexpr u64 kStagingAmps = 1ull << 27;   // 2 GiB staging: two 1 GiB slots (NCCL p2p reaches ~600 GB/s only at >= 512 MiB messages, benchmarks/p2p_bw.py)

struct DistState {
  SwapStats stats;
};

inline u64 local_mask(int nl) { return nl >= 64 ? ~0ull : ((1ull << nl) - 1); }

int logical_at(const sv_handle* h, int p) {
  for (int o = 0; o < h->n; ++o)
    if (h->phys[o] == p) return o;
  return -1;
}

// swap two LOCAL physical bits with a SWAP pair primitive on every state (no communication)
void local_bit_swap(sv_handle* h, const std::vector<double2*>& states, int p, int q) {
  if (p == q) return;
  Prim s;
  s.type = PRIM_PAIR;
  s.fmask = (1ull << p) | (1ull << q);
  s.fval = 1ull << p;                 // i0 has bit p = 1, bit q = 0; partner flips both
  s.xmask = s.fmask;
  s.m = {cplx(0), cplx(1), cplx(1), cplx(0)};
  for (double2* st : states) launch_prim(h, st, s);
  int op = logical_at(h, p), oq = logical_at(h, q);
  h->phys[op] = q;
  h->phys[oq] = p;
}

// stream-ordered barrier over all ranks (a 1-int allreduce on the handle's stream)
void device_barrier(sv_handle* h) {
  NCCL_CHECK(ncclAllReduce(h->d_barrier, h->d_barrier, 1, ncclInt, ncclSum, h->comm, h->stream));
}

// Collective: export `buf` (a cudaMalloc base) with CUDA IPC, all-gather the handles and map
// every other rank's copy (world <= 8: a multi-bit exchange talks to any rank of its group).
// Returns 1 when every rank mapped all its peers (else nothing stays mapped on any rank).
int register_peers(sv_handle* h, double2* buf) {
  int ok = h->world <= 8 ? 1 : 0;
  cudaIpcMemHandle_t mine;
  std::memset(&mine, 0, sizeof(mine));
  if (ok && cudaIpcGetMemHandle(&mine, buf) != cudaSuccess) {
    cudaGetLastError();
    ok = 0;
  }
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  char* d_handles = nullptr;
  CUDA_CHECK(cudaMalloc(&d_handles, hb * (h->world + 1)));
  CUDA_CHECK(cudaMemcpyAsync(d_handles + hb * h->world, &mine, hb, cudaMemcpyHostToDevice, h->stream));
  NCCL_CHECK(ncclAllGather(d_handles + hb * h->world, d_handles, hb, ncclChar, h->comm, h->stream));
  std::vector<cudaIpcMemHandle_t> all(h->world);
  d2h(h, all.data(), d_handles, hb * h->world);
  CUDA_CHECK(cudaFree(d_handles));
  sv_handle::PeerMap pm;
  pm.local = buf;
  for (int r = 0; r < 8; ++r) pm.by_rank[r] = nullptr;
  for (int r = 0; ok && r < h->world; ++r) {
    if (r == h->rank) continue;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    pm.by_rank[r] = static_cast<double2*>(p);
  }
  int* d_ok = h->d_barrier + 1;
  CUDA_CHECK(cudaMemcpyAsync(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  NCCL_CHECK(ncclAllReduce(d_ok, d_ok, 1, ncclInt, ncclMin, h->comm, h->stream));
  d2h(h, &ok, d_ok, sizeof(int));
  if (ok) {
    h->peers.push_back(pm);
  } else {
    for (int r = 0; r < 8; ++r)
      if (pm.by_rank[r]) cudaIpcCloseMemHandle(pm.by_rank[r]);
  }
  return ok;
}

// the peer map of `buf` (registering it on first use, collectively); false when unavailable.
// Returned by value: registering another buffer may reallocate h->peers.
bool peers_of(sv_handle* h, double2* buf, sv_handle::PeerMap* out) {
  if (!h->p2p) return false;
  for (const auto& pm : h->peers)
    if (pm.local == buf) {
      *out = pm;
      return true;
    }
  if (!register_peers(h, buf)) return false;
  *out = h->peers.back();
  return true;
}

// Exchange global positions Gs[i] with local positions ps[i] (i < k <= 3), all at once: an amplitude
// whose bits at ps spell c (bit i <-> ps[i]) moves to the rank whose bits at Gs spell c, at the same
// local index with the ps bits set to this rank's bits at Gs.  k = 1 is a qubit-index swap with
// one partner (half the shard crosses NVLink); k = log2 P is one all-to-all over all ranks
// ((1 - 2^-k) of the shard) -- cheaper than k sequential single-bit swaps (k / 2 of the shard) and
// with no local bit-permutation pass: the victims stay where they are.
//   peer memory (default): one kernel reads and writes the partners' states mapped over NVLink,
//     each rank pair splitting its pairs on a free local bit; two stream-ordered barriers;
//   fallback (NCCL): per partner (XOR schedule, deadlock-free), gather the elements through the
//     staging buffer, ncclSend/ncclRecv, scatter -- the same element placement, so both paths
//     give bit-identical states.
void exchange_bits(sv_handle* h, const std::vector<double2*>& states, const std::vector<int>& Gs,
                   const std::vector<int>& ps) {
  const int k = int(Gs.size());
  if (k == 0) return;
  if (k > 3 || int(ps.size()) != k) sv_fail(SV_ERR_DEVICE, "internal: bad exchange");
  auto relayout = [&]() {
    std::vector<int> og(k), op(k);
    for (int i = 0; i < k; ++i) {
      og[i] = logical_at(h, Gs[i]);
      op[i] = logical_at(h, ps[i]);
    }
    for (int i = 0; i < k; ++i) {
      h->phys[og[i]] = ps[i];
      h->phys[op[i]] = Gs[i];
    }
  };
  if (h->recording) {
    RecStep st;
    st.kind = REC_XSWAP;
    st.Gs = Gs;
    st.ps = ps;
    h->rec.push_back(st);
    relayout();
    return;
  }
  const int nc = 1 << k;
  u64 vmask = 0, vdep[8] = {0};
  for (int c = 0; c < nc; ++c)
    for (int i = 0; i < k; ++i)
      if ((c >> i) & 1) vdep[c] |= 1ull << ps[i];
  for (int i = 0; i < k; ++i) vmask |= 1ull << ps[i];
  int g = 0, rank_of[8];
  for (int i = 0; i < k; ++i) g |= ((h->rank >> (Gs[i] - h->nl)) & 1) << i;
  for (int c = 0; c < nc; ++c) {
    int r = h->rank;
    for (int i = 0; i < k; ++i) r = (r & ~(1 << (Gs[i] - h->nl))) | (((c >> i) & 1) << (Gs[i] - h->nl));
    rank_of[c] = r;
  }
  const u64 moved = (h->n_local >> k) * u64(nc - 1);   // amplitudes leaving this rank
  cudaEvent_t ev[2];
  bool p2p = h->p2p;
  std::vector<sv_handle::PeerMap> maps(states.size());
  for (size_t si = 0; si < states.size() && p2p; ++si) p2p = peers_of(h, states[si], &maps[si]);
  for (size_t si = 0; si < states.size(); ++si) {
    double2* st = states[si];
    // peer memory: the partners' earlier kernels on their states are done -- the wait absorbs any
    // skew between the ranks' programs, so it stays outside the swap's timed region
    if (p2p) device_barrier(h);
    stat_begin(h, KC_SWAP, 32.0 * double(moved), ev);
    static const bool old_top = getenv("SVB200_XCHG_TOP") && std::string(getenv("SVB200_XCHG_TOP")) == "1";
    if (p2p && old_top && k == 1 && ps[0] == h->nl - 1) {
      // A/B reference: the round-1 contiguous half-shard exchange (victim on the top local bit)
      const int b = g;
      const u64 half = h->n_local >> 1, share = half >> 1, lo = b ? share : 0;
      double2* peer = maps[si].by_rank[rank_of[1 - g]];
      launch_exchange(h, st + ((1 - b) ? half : 0) + lo, peer + (b ? half : 0) + lo, b ? half - share : share);
      device_barrier(h);
    } else if (p2p) {
      // pairs with partner c split on the highest local bit that is not a victim
      int q = h->nl - 1;
      while ((vmask >> q) & 1) --q;
      double2* peer[8];
      u64 own[8];
      for (int c = 0; c < nc; ++c) {
        peer[c] = c == g ? nullptr : maps[si].by_rank[rank_of[c]];
        own[c] = h->rank < rank_of[c] ? 0ull : (1ull << q);
      }
      launch_exchange_multi(h, st, peer, vdep, own, vdep[g], nc, vmask | (1ull << q), h->n_local >> (k + 1));
      device_barrier(h);   // their stores into ours are visible
    } else {
      const u64 per = h->n_local >> k;   // amplitudes exchanged with each partner
      const u64 chunk = h->staging_amps / 2;
      double2* sbuf = h->staging;
      double2* rbuf = h->staging + chunk;
      for (int step = 1; step < nc; ++step) {
        const int c = g ^ step;
        for (u64 t = 0; t < per; t += chunk) {
          const u64 len = std::min<u64>(chunk, per - t);
          launch_pack_sel(h, st, sbuf, vmask, vdep[c], t, len, false);
          NCCL_CHECK(ncclGroupStart());
          NCCL_CHECK(ncclSend(sbuf, len * 2, ncclDouble, rank_of[c], h->comm, h->stream));
          NCCL_CHECK(ncclRecv(rbuf, len * 2, ncclDouble, rank_of[c], h->comm, h->stream));
          NCCL_CHECK(ncclGroupEnd());
          launch_pack_sel(h, st, rbuf, vmask, vdep[c], t, len, true);
        }
      }
    }
    stat_end(h, KC_SWAP, 32.0 * double(moved), ev);
  }
  relayout();
}

// exchange the top local bit (nl-1) with global position G = nl + j
void global_swap_top(sv_handle* h, const std::vector<double2*>& states, int G) {
  exchange_bits(h, states, {G}, {h->nl - 1});
}

// bring logical offset o (currently global) local, evicting a local qubit not in `keep`
void make_one_local(sv_handle* h, const std::vector<double2*>& states, int o, const std::vector<int>& keep_offsets) {
  const int G = h->phys[o];
  if (G < h->nl) return;
  auto kept = [&](int p) {
    int lo = logical_at(h, p);
    return std::find(keep_offsets.begin(), keep_offsets.end(), lo) != keep_offsets.end();
  };
  int victim = -1;
  for (int p = h->nl - 1; p >= 0; --p)
    if (!kept(p)) {
      victim = p;
      break;
    }
  if (victim < 0) sv_fail(SV_ERR_CAPACITY, "gate acts on more qubits than one shard holds locally");
  exchange_bits(h, states, {G}, {victim});
}
}  // namespace

void dist_init(sv_handle* h, const void* nccl_id) {
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  NCCL_CHECK(ncclCommInitRank(&h->comm, h->world, id, h->rank));
  h->staging_amps = std::min<u64>(kStagingAmps, std::max<u64>(h->n_local >> 1, 2));
  CUDA_CHECK(cudaMalloc(&h->staging, h->staging_amps * sizeof(double2)));
  CUDA_CHECK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_recv[i], cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&h->ev_copy[i], cudaEventDisableTiming));
  }
  CUDA_CHECK(cudaMalloc(&h->d_barrier, 64 * sizeof(int)));
  CUDA_CHECK(cudaMemsetAsync(h->d_barrier, 0, 64 * sizeof(int), h->stream));
  // Peer-memory swaps: map every partner's state (rank ^ 2^j) through CUDA IPC now; other
  // swapped buffers (adjoint lambdas) register on their first swap.  Any rank failing to map
  // (no P2P path, SVB200_P2P_SWAP=0) turns the feature off on every rank: NCCL send/recv.
  const char* env = std::getenv("SVB200_P2P_SWAP");
  int want = (env && env[0] == '0') ? 0 : 1;
  int* d_ok = h->d_barrier + 1;
  CUDA_CHECK(cudaMemcpyAsync(d_ok, &want, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  NCCL_CHECK(ncclAllReduce(d_ok, d_ok, 1, ncclInt, ncclMin, h->comm, h->stream));
  d2h(h, &want, d_ok, sizeof(int));
  h->p2p = want && register_peers(h, h->state);
}

void dist_forget(sv_handle* h, double2* buf) {
  if (!h->p2p || !h->comm) return;
  for (size_t i = 0; i < h->peers.size(); ++i)
    if (h->peers[i].local == buf) {
      // every rank is done with every mapping of this buffer before any rank unmaps or frees it
      if (ncclAllReduce(h->d_barrier, h->d_barrier, 1, ncclInt, ncclSum, h->comm, h->stream) == ncclSuccess)
        try {
          stream_sync(h);   // bounded wait: a dead peer aborts the communicator instead of hanging
        } catch (const SvError&) {
        }
      for (int r = 0; r < 8; ++r)
        if (h->peers[i].by_rank[r]) cudaIpcCloseMemHandle(h->peers[i].by_rank[r]);
      h->peers.erase(h->peers.begin() + long(i));
      return;
    }
}

void dist_abort(sv_handle* h) {
  if (!h->comm) return;
  ncclCommAbort(h->comm);
  h->comm = nullptr;
  h->p2p = false;   // peer mappings stay until destroy; no further exchanges
}

void dist_destroy(sv_handle* h) {
  const cudaError_t q = h->comm ? cudaStreamQuery(h->stream) : cudaSuccess;
  if (q != cudaSuccess && q != cudaErrorNotReady) {
    cudaGetLastError();
    dist_abort(h);   // a failed device context: destroying would wait on peers forever
  }
  if (h->p2p && h->comm) {
    // no rank unmaps (or frees) a state its partner may still be exchanging with
    if (ncclAllReduce(h->d_barrier, h->d_barrier, 1, ncclInt, ncclSum, h->comm, h->stream) == ncclSuccess)
      try {
        stream_sync(h);
      } catch (const SvError&) {
      }
  }
  for (auto& pm : h->peers)
    for (int r = 0; r < 8; ++r)
      if (pm.by_rank[r]) cudaIpcCloseMemHandle(pm.by_rank[r]);
  h->peers.clear();
  h->p2p = false;
  if (h->d_barrier) {
    cudaFree(h->d_barrier);
    h->d_barrier = nullptr;
  }
  if (h->comm) {
    ncclCommDestroy(h->comm);
    h->comm = nullptr;
  }
  if (h->staging) {
    cudaFree(h->staging);
    h->staging = nullptr;
  }
  for (int i = 0; i < 2; ++i) {
    if (h->ev_recv[i]) cudaEventDestroy(h->ev_recv[i]);
    if (h->ev_copy[i]) cudaEventDestroy(h->ev_copy[i]);
    h->ev_recv[i] = h->ev_copy[i] = nullptr;
  }
  if (h->copy_stream) {
    cudaStreamDestroy(h->copy_stream);
    h->copy_stream = nullptr;
  }
}

bool prim_needs_swap(const Prim& p, int nl) {
  if (p.skip) return false;
  if (p.type == PRIM_PAIR) return (p.xmask & ~local_mask(nl)) != 0;
  if (p.type == PRIM_DENSE)
    for (int j = 0; j < p.nb; ++j)
      if (p.pos[j] >= nl) return true;
  return false;
}

// Bring every global qubit in `keep` local with ONE exchange (exchange_bits), plus -- while an
// exchange is happening anyway -- the other global qubits needed again before some local qubit
// would be (Belady: victims are the local qubits not in `keep` whose next use is furthest; ties
// prefer positions >= 3 (whole 128-byte runs stay together) and then the highest position).
void dist_bring_local(sv_handle* h, const std::vector<double2*>& states, const std::vector<int>& keep,
                      const std::vector<int>& next_use) {
  std::vector<int> in;
  for (int o : keep)
    if (h->phys[o] >= h->nl) in.push_back(o);
  if (in.empty()) return;
  std::vector<std::pair<int, int>> cand;   // (next use, local position)
  for (int p = 0; p < h->nl; ++p) {
    const int lo = logical_at(h, p);
    if (std::find(keep.begin(), keep.end(), lo) != keep.end()) continue;
    cand.push_back({next_use[lo], p});
  }
  // victims on physical bits 0..2 would split the exchange's 128-byte runs (16-byte remote
  // accesses) and bits 3..6 its 2 KiB runs: positions >= 7 first, then 3..6, then 0..2, Belady
  // (furthest next use) within a tier
  auto tier = [](int p) { return p >= 7 ? 0 : (p >= 3 ? 1 : 2); };
  std::sort(cand.begin(), cand.end(), [&](const std::pair<int, int>& a, const std::pair<int, int>& b) {
    if (tier(a.second) != tier(b.second)) return tier(a.second) < tier(b.second);
    if (a.first != b.first) return a.first > b.first;
    return a.second > b.second;
  });
  if (cand.size() < in.size()) sv_fail(SV_ERR_CAPACITY, "operation spans more qubits than a shard holds locally");
  std::vector<std::pair<int, int>> extra;   // (next use, logical offset) of the other global qubits
  for (int G = h->nl; G < h->n; ++G) {
    const int o = logical_at(h, G);
    if (std::find(in.begin(), in.end(), o) == in.end() && next_use[o] < (1 << 30)) extra.push_back({next_use[o], o});
  }
  std::sort(extra.begin(), extra.end());
  size_t vi = in.size();
  for (const auto& e : extra)
    if (vi < cand.size() && cand[vi].first > e.first) {
      in.push_back(e.second);
      ++vi;
    }
  for (size_t b = 0; b < in.size(); b += 3) {   // at most 3 bits per exchange (P <= 8 in one go)
    std::vector<int> Gs, ps;
    for (size_t i = b; i < std::min(in.size(), b + 3); ++i) {
      Gs.push_back(h->phys[in[i]]);
      ps.push_back(cand[i].second);
    }
    exchange_bits(h, states, Gs, ps);
  }
}

void dist_swap_in(sv_handle* h, const std::vector<double2*>& states, int o, const std::vector<int>& keep,
                  const std::vector<int>& next_use) {
  const int G = h->phys[o];
  if (G < h->nl) return;
  int victim = -1, best = -1;
  for (int p = h->nl - 1; p >= 0; --p) {
    const int lo = logical_at(h, p);
    if (std::find(keep.begin(), keep.end(), lo) != keep.end()) continue;
    // furthest next use wins; ties prefer the top local bit (no local swap needed)
    if (next_use[lo] > best) {
      best = next_use[lo];
      victim = p;
    }
  }
  if (victim < 0) sv_fail(SV_ERR_CAPACITY, "operation spans more qubits than a shard holds locally");
  exchange_bits(h, states, {G}, {victim});
}

void dist_make_local(sv_handle* h, const std::vector<double2*>& states, const std::vector<int>& wires) {
  dist_make_local_set(h, states, wires);
}

void dist_make_local_set(sv_handle* h, const std::vector<double2*>& states, const std::vector<int>& wires) {
  if (h->world == 1) return;
  std::vector<int> offs;
  for (int w : wires) offs.push_back(h->n - 1 - w);
  if (int(offs.size()) > h->nl) sv_fail(SV_ERR_CAPACITY, "operation spans more qubits than a shard holds locally");
  for (int o : offs) make_one_local(h, states, o, offs);
}

// Restore the identity layout (fused passes and sharded swaps leave qubits relabeled).
void dist_canonicalize(sv_handle* h, const std::vector<double2*>& states) {
  // global positions first: logical offset G must sit at physical G
  for (int G = h->nl; G < h->n; ++G) {
    if (h->phys[G] == G) continue;
    int p = h->phys[G];
    if (p >= h->nl) {            // logical G sits on another global position: bring it local first
      global_swap_top(h, states, p);
      p = h->phys[G];            // now the top local bit
    }
    local_bit_swap(h, states, p, h->nl - 1);
    global_swap_top(h, states, G);
  }
  // then the local permutation (selection sort with local swaps)
  for (int o = 0; o < h->nl; ++o)
    if (h->phys[o] != o) local_bit_swap(h, states, h->phys[o], o);
}

void dist_reset_layout(sv_handle* h) {
  for (int o = 0; o < h->n; ++o) h->phys[o] = o;
}

void dist_gather_state(sv_handle* h, double* out) {
  const u64 nl = h->n_local;
  for (int r = 0; r < h->world; ++r) {
    for (u64 c = 0; c < nl; c += h->staging_amps) {
      const u64 len = std::min<u64>(h->staging_amps, nl - c);
      const double2* src = (r == h->rank) ? h->state + c : h->staging;
      NCCL_CHECK(ncclBroadcast(h->state + c, h->staging, len * 2, ncclDouble, r, h->comm, h->stream));
      CUDA_CHECK(cudaMemcpyAsync(out + 2 * (u64(r) * nl + c), src, len * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
      stream_sync(h);
    }
  }
}

void dist_allreduce_sum(sv_handle* h, double* host, size_t n) {
  if (h->world == 1 || n == 0) return;
  ensure_results(h, n);
  CUDA_CHECK(cudaMemcpyAsync(h->d_results, host, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  NCCL_CHECK(ncclAllReduce(h->d_results, h->d_results, n, ncclDouble, ncclSum, h->comm, h->stream));
  d2h(h, host, h->d_results, n * sizeof(double));
}

void dist_probs(sv_handle* h, const std::vector<int>& wires, double* out) {
  const int w = int(wires.size());
  std::vector<int> lpos;   // physical positions of local wires, MSB-first order
  std::vector<int> lidx;   // index j of those wires in `wires`
  u64 need_mask = 0, need_val = 0;   // bin bits fixed by this rank's global bits
  for (int j = 0; j < w; ++j) {
    int p = h->phys[h->n - 1 - wires[j]];
    if (p < h->nl) {
      lpos.push_back(p);
      lidx.push_back(j);
    } else {
      u64 bit = 1ull << (w - 1 - j);
      need_mask |= bit;
      if ((h->rank >> (p - h->nl)) & 1) need_val |= bit;
    }
  }
  const u64 lbins = 1ull << lpos.size();
  ensure_results(h, lbins);
  probs_async(h, h->state, lpos, h->d_results);
  std::vector<double> local(lbins);
  d2h(h, local.data(), h->d_results, lbins * sizeof(double));
  const u64 bins = 1ull << w;
  if (h->world == 1) {
    std::memcpy(out, local.data(), bins * sizeof(double));
    return;
  }
  std::vector<double> full(bins, 0.0);
  const int nlw = int(lpos.size());
  for (u64 lb = 0; lb < lbins; ++lb) {
    u64 b = need_val;
    for (int i = 0; i < nlw; ++i)
      if ((lb >> (nlw - 1 - i)) & 1) b |= 1ull << (w - 1 - lidx[i]);
    full[b] = local[lb];
  }
  dist_allreduce_sum(h, full.data(), bins);
  std::memcpy(out, full.data(), bins * sizeof(double));
}

SwapStats dist_swap_stats(const sv_handle* h) {
  SwapStats s;
  s.swaps = int64_t(h->kc_launches[KC_SWAP]);
  s.bytes_sent = h->kc_bytes[KC_SWAP];
  return s;
}
