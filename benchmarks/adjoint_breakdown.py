"""Per-kernel-class device time of one adjoint Jacobian (configs 3 / 5 of BASELINE.json).

    python benchmarks/adjoint_breakdown.py [--config 5] [--qubits N]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from benchmarks.adjoint_bench import config  # noqa: E402
from paper_2403_02512_b200.device import Device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--qubits", type=int, default=0)
    a = ap.parse_args()
    n, ops, obs, desc = config(a.config, a.qubits)
    with Device(n) as d:
        d.adjoint_jacobian(ops, obs)   # warm-up: plans, kernels, buffers
        d.reset()
        d.synchronize()
        d.reset_stats()
        d.set_profiling(True)
        t0 = time.perf_counter()
        d.adjoint_jacobian(ops, obs)
        d.synchronize()
        t = time.perf_counter() - t0
        st = d.kernel_stats()
        d.set_profiling(False)
    rows = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                "GBps": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 else None}
            for k, v in st.items() if v["launches"]}
    print(json.dumps({"workload": desc, "s_wall": t, "device_ms_total": round(sum(v["ms"] for v in st.values()), 2),
                      "classes": rows}))


if __name__ == "__main__":
    main()
