// Gate fusion engine (K7).  First slice: every primitive is its own HBM pass; the
// shared-memory / register tile engine replaces this file's body.
#include "sv_internal.h"

void apply_prims_fused(sv_handle* h, double2* state, const std::vector<Prim>& prims) {
  for (const Prim& p : prims) launch_prim(h, state, p);
}

PlanStats plan_stats(int nl, const std::vector<Prim>& prims) {
  PlanStats s;
  (void)nl;
  s.passes = int64_t(prims.size());
  s.ops = int64_t(prims.size());
  return s;
}
