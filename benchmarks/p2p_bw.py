"""NVLink exchange bandwidth between rank pairs (the global-qubit swap's transport).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 benchmarks/p2p_bw.py

Times a symmetric exchange (each rank sends S bytes to its partner and receives S bytes) with
NCCL send/recv (batch_isend_irecv), and with a CUDA-IPC peer copy (cudaMemcpyPeerAsync of the
partner's buffer into a local one), for a few sizes; prints GB/s per direction per rank.
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
    partner = rank ^ 1
    out = {}
    for mib in (128, 512, 2048):
        n = mib << 20
        a = torch.empty(n, dtype=torch.uint8, device="cuda")
        b = torch.empty(n, dtype=torch.uint8, device="cuda")
        for it in range(4):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, a, partner), dist.P2POp(dist.irecv, b, partner)])
            for r in reqs:
                r.wait()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        out[f"nccl_{mib}MiB_GBps"] = n / (ms / 1e3) / 1e9
    if rank == 0:
        print(json.dumps({"world": world, **out, "env": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
