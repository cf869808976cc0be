"""DRAM locality of fused-pass tiles: one fused pass whose tile holds physical bits 0..2 plus nine
chosen high bits (one RX per chosen qubit), timed per pass; GB/s vs the bit positions.

    python benchmarks/tile_locality.py [--n 30]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_02512_b200.device import Device, plan_summary  # noqa: E402
from paper_2403_02512_b200.ops import Op  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    a = ap.parse_args()
    n = a.n
    sets = {"bits 3-11 (contiguous tile)": list(range(3, 12)), "bits 12-20": list(range(12, 21)),
            f"bits {n - 9}-{n - 1} (top)": list(range(n - 9, n)), "spread 3,6,..,27": list(range(3, 30, 3)),
            "bits 3-6 + 26-29": [3, 4, 5, 6, 26, 27, 28, 29, 15],
            "bits 17-25": list(range(17, 26)), "bits 3-7 + top 4": [3, 4, 5, 6, 7] + list(range(n - 4, n)),
            "bits 21-26 + top 3": list(range(21, 27)) + list(range(n - 3, n)),
            "bits 21-26 + 27-29": list(range(21, 30)),
            "bits 15-20 + top 3": list(range(15, 21)) + list(range(n - 3, n)),
            "bits 21-23 + 27-29 + top 3": [21, 22, 23, 27, 28, 29] + list(range(n - 3, n)),
            "bits 24-26 + top 3 + 3-5": [3, 4, 5, 24, 25, 26] + list(range(n - 3, n)),
            "bits 18-23 + top 3": list(range(18, 24)) + list(range(n - 3, n)),
            "bits 3-8 + top 3": list(range(3, 9)) + list(range(n - 3, n))}
    out = {}
    with Device(n) as d:
        for name, bits in sets.items():
            ops = [Op("RX", (n - 1 - b,), (0.1 + 0.01 * b,)) for b in bits]
            ps = plan_summary(n, ops)
            d.reset()
            d.apply(ops)
            d.reset_stats()
            d.set_profiling(True)
            for _ in range(5):
                d.reset()
                d.apply(ops)
            st = d.kernel_stats()["fused_tile"]
            d.set_profiling(False)
            ms = st["ms"] / st["launches"]
            out[name] = {"passes_planned": ps["passes"], "ms_per_pass": ms, "GBps": 32 * 2 ** n / ms / 1e6}
            print(f"{name:32s} passes={ps['passes']} ms/pass={ms:.3f} GB/s={32 * 2 ** n / ms / 1e6:.0f}", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
