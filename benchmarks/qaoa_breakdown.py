"""Per-kernel-class breakdown of the 33q QAOA forward + <C> (BASELINE config 3, 1 GPU):
reset, fused passes, expval, timed with the handle's CUDA-event stats."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_02512_b200 import workloads  # noqa: E402
from paper_2403_02512_b200.device import Device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
ops, ham, edges = workloads.qaoa_maxcut(n, p=2, seed=0)
with Device(n) as d:
    d.apply(ops)
    d.expval(ham)
    out = {}
    for stage in ("reset", "apply", "expval"):
        d.synchronize()
        d.set_profiling(True)
        d.reset_stats()
        t0 = time.perf_counter()
        if stage == "reset":
            d.reset()
        elif stage == "apply":
            d.apply(ops)
        else:
            d.expval(ham)
        d.synchronize()
        dt = time.perf_counter() - t0
        st = {k: v for k, v in d.kernel_stats().items() if v["launches"]}
        d.set_profiling(False)
        out[stage] = {"s": dt, "kernels": st}
print(json.dumps({"n": n, "breakdown": out}))
