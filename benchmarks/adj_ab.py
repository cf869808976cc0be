"""A/B of the config-3 adjoint wall time (31-qubit QAOA p=2) under the current env: prints one line
with the min of 3 timed Jacobians after a warm-up, and the host-side share."""
import sys
import time

sys.path.insert(0, ".")
from paper_2403_02512_b200 import workloads  # noqa: E402
from paper_2403_02512_b200.device import Device, jit_stats  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
ops, ham, _ = workloads.qaoa_maxcut(n, p=2, seed=0)
with Device(n) as d:
    d.adjoint_jacobian(ops, [ham])
    ts, dev = [], []
    for _ in range(3):
        d.reset()
        d.synchronize()
        d.reset_stats()
        d.set_profiling(True)
        j0 = jit_stats()
        t0 = time.perf_counter()
        d.adjoint_jacobian(ops, [ham])
        d.synchronize()
        ts.append(time.perf_counter() - t0)
        st = d.kernel_stats()
        dev.append(sum(v["ms"] for v in st.values()) / 1e3)
        j1 = jit_stats()
        print(f"  call: wall {ts[-1]:.4f} device {dev[-1]:.4f} compiled {j1['compiled'] - j0['compiled']} kernels {j1['kernels']}")
        d.set_profiling(False)
    i = min(range(3), key=lambda k: ts[k])
    print(f"wall {ts[i]:.4f} s  device {dev[i]:.4f} s  classes {sorted((k, round(v['ms'], 1), v['launches']) for k, v in st.items())}")
