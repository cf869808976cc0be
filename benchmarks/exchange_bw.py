"""Qubit-index exchange bandwidth through the library (dist.cpp exchange_bits), under torchrun.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 benchmarks/exchange_bw.py --qubits 32

Each repetition: reset (canonical layout: the top log2 P qubits are global), then one op list
touching every global qubit with a dense gate -> ONE exchange of all global bits (P = 2: one
partner; P = 4: three partners).  Reports the swap kernel-class time and GB/s per direction
(bytes leaving each rank / device time, the barriers included), max over ranks.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_02512_b200.device import Device  # noqa: E402
from paper_2403_02512_b200.ops import Op  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch.distributed as tdist
    tdist.init_process_group("gloo", init_method="env://")
    rank, world = tdist.get_rank(), tdist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    g = world.bit_length() - 1
    nid = [Device.nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(nid, src=0)
    d = Device.sharded(a.qubits, rank, world, nid[0], device=local)
    ops = [Op("H", (q,)) for q in range(g)]
    d.reset()
    d.apply(ops)
    d.reset_stats()
    d.set_profiling(True)
    for _ in range(a.reps):
        d.reset()
        d.apply(ops)
    st = d.kernel_stats()
    d.set_profiling(False)
    sw = st["swap"]
    ms = sw["ms"] / a.reps
    sent = sw["bytes"] / 2.0 / a.reps
    out = [None] * world
    tdist.all_gather_object(out, ms)
    if rank == 0:
        msx = max(out)
        print(json.dumps({"n_qubits": a.qubits, "n_gpus": world, "global_bits": g, "exchanges_per_rep": sw["launches"] / a.reps,
                          "ms_per_exchange_set": msx, "GB_out_per_rank": sent / 1e9,
                          "GBps_per_direction": sent / (msx / 1e3) / 1e9, "xchg_top": os.environ.get("SVB200_XCHG_TOP", "0")}))
    d.release()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
