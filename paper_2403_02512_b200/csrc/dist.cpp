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

// Collective: export `buf` (a cudaMalloc base) with CUDA IPC, all-gather the handles and map the
// log2 P partners' copies.  Returns 1 when every rank mapped all its partners (else nothing
// stays mapped on any rank).
int register_peers(sv_handle* h, double2* buf) {
  int ok = 1;
  cudaIpcMemHandle_t mine;
  std::memset(&mine, 0, sizeof(mine));
  if (cudaIpcGetMemHandle(&mine, buf) != cudaSuccess) {
    cudaGetLastError();
    ok = 0;
  }
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  char* d_handles = nullptr;
  CUDA_CHECK(cudaMalloc(&d_handles, hb * (h->world + 1)));
  CUDA_CHECK(cudaMemcpyAsync(d_handles + hb * h->world, &mine, hb, cudaMemcpyHostToDevice, h->stream));
  NCCL_CHECK(ncclAllGather(d_handles + hb * h->world, d_handles, hb, ncclChar, h->comm, h->stream));
  std::vector<cudaIpcMemHandle_t> all(h->world);
  CUDA_CHECK(cudaMemcpyAsync(all.data(), d_handles, hb * h->world, cudaMemcpyDeviceToHost, h->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->stream));
  CUDA_CHECK(cudaFree(d_handles));
  sv_handle::PeerMap pm;
  pm.local = buf;
  for (int j = 0; j < 8; ++j) pm.peer[j] = nullptr;
  for (int j = 0; ok && j < h->g && j < 8; ++j) {
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, all[h->rank ^ (1 << j)], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    pm.peer[j] = static_cast<double2*>(p);
  }
  int* d_ok = h->d_barrier + 1;
  CUDA_CHECK(cudaMemcpyAsync(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  NCCL_CHECK(ncclAllReduce(d_ok, d_ok, 1, ncclInt, ncclMin, h->comm, h->stream));
  CUDA_CHECK(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->stream));
  if (ok) {
    h->peers.push_back(pm);
  } else {
    for (int j = 0; j < 8; ++j)
      if (pm.peer[j]) cudaIpcCloseMemHandle(pm.peer[j]);
  }
  return ok;
}

// partner copy of `buf` for global bit j (registering it on first use), or nullptr
double2* peer_of(sv_handle* h, double2* buf, int j) {
  if (!h->p2p || j >= 8) return nullptr;
  for (const auto& pm : h->peers)
    if (pm.local == buf) return pm.peer[j];
  if (!register_peers(h, buf)) return nullptr;
  return h->peers.back().peer[j];
}

// exchange the top local bit (nl-1) with global position G = nl + j
void global_swap_top(sv_handle* h, const std::vector<double2*>& states, int G) {
  if (h->recording) {
    h->rec.push_back({REC_GSWAP, Prim(), G});
    int ot = logical_at(h, h->nl - 1), og = logical_at(h, G);
    h->phys[ot] = G;
    h->phys[og] = h->nl - 1;
    return;
  }
  const int j = G - h->nl;
  const int partner = h->rank ^ (1 << j);
  const int b = (h->rank >> j) & 1;
  const u64 half = h->n_local >> 1;
  // we send our (top bit = 1-b) half and receive the partner's (top bit = b) half into it
  const u64 my_off = (1 - b) ? half : 0;
  // Chunk k: send our chunk k and receive the partner's into staging slot k&1 (main stream), then
  // copy the slot over our chunk k on the copy stream -- so the copy of chunk k overlaps the
  // transfer of chunk k+1.  A slot is reused only after its previous copy finished; chunk k+1's
  // send reads a region no copy has touched yet.
  const u64 chunk = h->staging_amps / 2;
  cudaEvent_t ev[2];
  for (double2* st : states) {
    stat_begin(h, KC_SWAP, 32.0 * double(half), ev);
    double2* peer = peer_of(h, st, j);
    if (peer) {
      // Peer-memory swap: our (top = 1-b) half and the partner's (top = b) half exchange
      // element by element, in place, through the partner's state mapped over NVLink.  The two
      // ranks split the range (b = 0 the first half, b = 1 the second); barriers before (the
      // partner's earlier kernels on its state are done) and after (its stores into ours are).
      const u64 share = half >> 1, lo = b ? share : 0;
      const u64 peer_off = b ? half : 0;
      device_barrier(h);
      launch_exchange(h, st + my_off + lo, peer + peer_off + lo, b ? half - share : share);
      device_barrier(h);
      stat_end(h, KC_SWAP, 32.0 * double(half), ev);
      continue;
    }
    int k = 0;
    for (u64 c = 0; c < half; c += chunk, ++k) {
      const u64 len = std::min<u64>(chunk, half - c);
      double2* slot = h->staging + (k & 1) * chunk;
      if (k >= 2) CUDA_CHECK(cudaStreamWaitEvent(h->stream, h->ev_copy[k & 1], 0));
      NCCL_CHECK(ncclGroupStart());
      NCCL_CHECK(ncclSend(st + my_off + c, len * 2, ncclDouble, partner, h->comm, h->stream));
      NCCL_CHECK(ncclRecv(slot, len * 2, ncclDouble, partner, h->comm, h->stream));
      NCCL_CHECK(ncclGroupEnd());
      CUDA_CHECK(cudaEventRecord(h->ev_recv[k & 1], h->stream));
      CUDA_CHECK(cudaStreamWaitEvent(h->copy_stream, h->ev_recv[k & 1], 0));
      CUDA_CHECK(cudaMemcpyAsync(st + my_off + c, slot, len * sizeof(double2), cudaMemcpyDeviceToDevice,
                                 h->copy_stream));
      CUDA_CHECK(cudaEventRecord(h->ev_copy[k & 1], h->copy_stream));
    }
    for (int s = 0; s < std::min(k, 2); ++s) CUDA_CHECK(cudaStreamWaitEvent(h->stream, h->ev_copy[s], 0));
    stat_end(h, KC_SWAP, 32.0 * double(half), ev);
  }
  int ot = logical_at(h, h->nl - 1), og = logical_at(h, G);
  h->phys[ot] = G;
  h->phys[og] = h->nl - 1;
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
  local_bit_swap(h, states, victim, h->nl - 1);
  global_swap_top(h, states, G);
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
  CUDA_CHECK(cudaMemcpyAsync(&want, d_ok, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->stream));
  h->p2p = want && register_peers(h, h->state);
}

void dist_forget(sv_handle* h, double2* buf) {
  if (!h->p2p || !h->comm) return;
  for (size_t i = 0; i < h->peers.size(); ++i)
    if (h->peers[i].local == buf) {
      // every rank is done with every mapping of this buffer before any rank unmaps or frees it
      if (ncclAllReduce(h->d_barrier, h->d_barrier, 1, ncclInt, ncclSum, h->comm, h->stream) == ncclSuccess)
        cudaStreamSynchronize(h->stream);
      for (int j = 0; j < 8; ++j)
        if (h->peers[i].peer[j]) cudaIpcCloseMemHandle(h->peers[i].peer[j]);
      h->peers.erase(h->peers.begin() + long(i));
      return;
    }
}

void dist_destroy(sv_handle* h) {
  if (h->p2p && h->comm) {
    // no rank unmaps (or frees) a state its partner may still be exchanging with
    if (ncclAllReduce(h->d_barrier, h->d_barrier, 1, ncclInt, ncclSum, h->comm, h->stream) == ncclSuccess)
      cudaStreamSynchronize(h->stream);
  }
  for (auto& pm : h->peers)
    for (int j = 0; j < 8; ++j)
      if (pm.peer[j]) cudaIpcCloseMemHandle(pm.peer[j]);
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
  local_bit_swap(h, states, victim, h->nl - 1);
  global_swap_top(h, states, G);
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
      CUDA_CHECK(cudaStreamSynchronize(h->stream));
    }
  }
}

void dist_allreduce_sum(sv_handle* h, double* host, size_t n) {
  if (h->world == 1 || n == 0) return;
  ensure_results(h, n);
  CUDA_CHECK(cudaMemcpyAsync(h->d_results, host, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  NCCL_CHECK(ncclAllReduce(h->d_results, h->d_results, n, ncclDouble, ncclSum, h->comm, h->stream));
  CUDA_CHECK(cudaMemcpyAsync(host, h->d_results, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->stream));
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
  CUDA_CHECK(cudaMemcpyAsync(local.data(), h->d_results, lbins * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_CHECK(cudaStreamSynchronize(h->stream));
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
