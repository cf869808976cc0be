"""Sharded (2 GPUs) fused apply vs the oracle on multi-tile shards (n_local >= 13), small
structured cases and random circuits; one JSON list of [case, n, P, max |delta|]."""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch.multiprocessing as mp
from oracle import svoracle as O
from paper_2403_02512_b200 import workloads
from paper_2403_02512_b200.ops import Op

def make(case, n):
    rng = np.random.default_rng(1)
    pre = [Op("H", (q,)) for q in range(1, n)]
    if case == "rz_all":
        return pre + [Op("RZ", (q,), (float(rng.uniform(0, 6)),)) for q in range(n)]
    if case == "rx_local":
        return pre + [Op("RX", (q,), (float(rng.uniform(0, 6)),)) for q in range(1, n)]
    if case == "cnot_local":
        return pre + [Op("RY", (q,), (0.3 * q,)) for q in range(1, n)] + [Op("CNOT", (q, q + 1)) for q in range(1, n - 1)]
    if case == "h0":
        return pre + [Op("RY", (q,), (0.3 * q,)) for q in range(1, n)] + [Op("H", (0,))]
    if case == "cnot_g":
        return pre + [Op("RY", (q,), (0.3 * q,)) for q in range(1, n)] + [Op("CNOT", (0, 5))]
    if case == "cnot_t0":
        return pre + [Op("RY", (q,), (0.3 * q,)) for q in range(1, n)] + [Op("CNOT", (5, 0))]
    if case == "rot_then_cnot01":
        return pre + [Op("RX", (q,), (0.2 + 0.3 * q,)) for q in range(n)] + [Op("CNOT", (0, 1))]
    if case == "rand":
        return workloads.random_circuit(n, 12, seed=8)
    if case == "rand2":
        return workloads.random_circuit(n, 2, seed=8)

def worker(rank, world, ids, q, cases):
    from paper_2403_02512_b200.device import Device
    out = []
    for i, (case, n, P) in enumerate(cases):
        if rank >= P:
            continue
        ops = make(case, n)
        d = Device.sharded(n, rank, P, ids[i], device=rank, fuse=True)
        d.apply(ops)
        st = d.get_state()
        d.release()
        if rank == 0:
            out.append([case, n, P, float(np.abs(st - O.run_circuit(n, ops)).max())])
    if rank == 0:
        q.put(out)

if __name__ == "__main__":
    from paper_2403_02512_b200.device import Device
    cases = [(c, 14, 2) for c in ("rz_all", "rx_local", "cnot_local", "h0", "cnot_g", "cnot_t0", "rot_then_cnot01",
                                  "rand2")] + [("rand", 16, 2), ("rand", 17, 2)]
    ids = [Device.nccl_unique_id() for _ in cases]
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, ids, q, cases)) for r in range(2)]
    [p.start() for p in ps]
    print(json.dumps(q.get(timeout=600)))
    [p.join() for p in ps]
