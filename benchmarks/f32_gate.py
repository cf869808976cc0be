"""One complex64 RX / CNOT / RZ on a 31-qubit (16 GiB) state: the target of the f32 ncu capture.

    ncu --set full -k regex:k_pair_v2 -c 1 python benchmarks/f32_gate.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_02512_b200.device import Device  # noqa: E402
from paper_2403_02512_b200.ops import Op  # noqa: E402

with Device(31, precision="f32", fuse=False) as d:
    for op in (Op("RX", (5,), (0.3,)), Op("CNOT", (3, 17)), Op("RZ", (9,), (0.7,))):
        d.apply([op])
    d.synchronize()
    print("ok", d.launch_count)
