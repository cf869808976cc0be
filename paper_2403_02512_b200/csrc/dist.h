// Sharded state vector over NCCL (one process per GPU): SURVEY.md §8(e) / SPEC.md:424-486.
//
// Shard r holds amplitudes whose global (top log2 P) physical bits spell r.
// h->phys maps each logical bit offset to a physical position; a gate whose dense target
// sits on a global position first swaps that qubit with a local one (a half-shard NCCL
// send/recv with partner r ^ bit), so the layout drifts and is canonicalised only for I/O.
#pragma once

#include "sv_internal.h"

void dist_init(sv_handle* h, const void* nccl_id);
void dist_destroy(sv_handle* h);
// collective: unmap a buffer's peer copies before it is freed (no-op if it was never swapped)
void dist_forget(sv_handle* h, double2* buf);
bool prim_needs_swap(const Prim& p, int nl);
// make the given wires local (dense targets of one op), choosing victims outside `wires`
void dist_make_local(sv_handle* h, const std::vector<double2*>& states, const std::vector<int>& wires);
void dist_make_local_set(sv_handle* h, const std::vector<double2*>& states, const std::vector<int>& wires);
// bring logical offset o local; victim = local qubit (offset not in keep) with the furthest next_use[offset]
void dist_swap_in(sv_handle* h, const std::vector<double2*>& states, int o, const std::vector<int>& keep,
                  const std::vector<int>& next_use);
// bring every global offset in keep local in one multi-bit exchange (plus Belady prefetch of the
// other global qubits needed before the victims are)
void dist_bring_local(sv_handle* h, const std::vector<double2*>& states, const std::vector<int>& keep,
                      const std::vector<int>& next_use);
void dist_canonicalize(sv_handle* h, const std::vector<double2*>& states);
void dist_reset_layout(sv_handle* h);
void dist_gather_state(sv_handle* h, double* out);
void dist_allreduce_sum(sv_handle* h, double* host, size_t n);
void dist_probs(sv_handle* h, const std::vector<int>& wires, double* out);
void adjoint_sweep(sv_handle* h, const sv_op* ops, int n_ops, const std::vector<double2*>& lams, int ncols, int fuse,
                   double* jac);
// swap counters (for the message-trace log of SPEC.md:479)
struct SwapStats {
  int64_t swaps = 0;
  double bytes_sent = 0;
};
SwapStats dist_swap_stats(const sv_handle* h);
