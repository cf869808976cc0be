"""Micro-benchmark of the K7 fused tile kernel: base pass cost, per-phase cost, per-op cost.

    python benchmarks/fused_micro.py [--n 28]

Each case is an op list that plans into exactly one fused pass; prints device ms per pass
(CUDA events on the library stream) and the implied cost per op / per phase.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2403_02512_b200.device import Device, plan_summary  # noqa: E402
from paper_2403_02512_b200.ops import Op  # noqa: E402


def timeit(dev, ops, reps=5):
    # reset before every apply: the canonical layout plans (and compiles) one program for all reps
    dev.reset()
    dev.apply(ops)
    dev.reset_stats()
    dev.set_profiling(True)
    for _ in range(reps):
        dev.reset()
        dev.apply(ops)
    st = dev.kernel_stats()
    dev.set_profiling(False)
    f = st["fused_tile"]
    return f["ms"] / max(f["launches"], 1), f["launches"] / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--case", default="")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    n = a.n
    low = [n - 1, n - 2, n - 3]           # physical bits 0..2
    mid = [n - 4, n - 5, n - 6]
    rng = np.random.default_rng(0)
    cases = {
        "1 phase, 1 RZ (phase1)": [Op("RZ", (low[0],), (0.3,))],
        "1 phase, 8 RX low bits": [Op("RX", (low[i % 3],), (0.1 * i,)) for i in range(8)],
        "1 phase, 32 RX low bits": [Op("RX", (low[i % 3],), (0.1 * i,)) for i in range(32)],
        "1 phase, 32 RY low bits": [Op("RY", (low[i % 3],), (0.1 * i,)) for i in range(32)],
        "1 phase, 32 general U": [Op("Rot", (low[i % 3],), (0.1 * i, 0.2, 0.3)) for i in range(11)],
        "1 phase, 32 RZ": [Op("RZ", (low[i % 3],), (0.1 * i,)) for i in range(32)],
        "1 phase, 32 CNOT (reg ctrl)": [Op("CNOT", (low[i % 3], low[(i + 1) % 3])) for i in range(32)],
        "1 phase, 32 X": [Op("X", (low[i % 3],)) for i in range(32)],
        "2 phases, 32 RX": [Op("RX", ((low + mid)[i % 6],), (0.1 * i,)) for i in range(32)],
        "3 phases, 32 RX": [Op("RX", ((low + mid + [n - 7, n - 8, n - 9])[i % 9],), (0.1 * i,)) for i in range(32)],
    }
    # unmergeable rotation streams: RX on 4 low qubits, then CZs (diagonal) between them, so no two
    # rotations on a qubit are adjacent (no merging); k rounds -> 4k shears + 4k parity phases, 1 phase
    def stream(rounds, qs):
        ops = []
        for r in range(rounds):
            for i, q in enumerate(qs):
                ops.append(Op("RX" if (r + i) % 2 else "RY", (q,), (0.1 + 0.01 * r + 0.001 * i,)))
            for i in range(len(qs)):
                ops.append(Op("CZ", (qs[i], qs[(i + 1) % len(qs)])))
        return ops
    four = [n - 1, n - 2, n - 3, n - 4]
    cases["stream 8 rounds (32 shears + 32 CZ), 1 phase"] = stream(8, four)
    cases["stream 16 rounds (64 shears + 64 CZ), 1 phase"] = stream(16, four)
    cases["stream 32 rounds (128 shears + 128 CZ), 1 phase"] = stream(32, four)
    cases["stream 16 rounds on 8 qubits (2+ phases)"] = stream(8, four + [n - 5, n - 6, n - 7, n - 8])
    out = {}
    with Device(n) as d:
        for name, ops in cases.items():
            if a.case and a.case not in name:
                continue
            ps = plan_summary(n, ops)
            ms, launches = timeit(d, ops, a.reps)
            out[name] = {"ms_per_pass": ms, "passes": ps["passes"], "phases": ps["phases"], "ops": len(ops)}
            print(f"{name:32s} passes={ps['passes']} phases={ps['phases']:3d} ops={len(ops):3d} "
                  f"ms/pass={ms:.3f} GB/s={32 * 2**n / ms / 1e6:.0f}", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
