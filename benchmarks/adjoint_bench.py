"""Adjoint-Jacobian timings for BASELINE.json configs 1, 3 and 5.

    python benchmarks/adjoint_bench.py [--config 1|3|5|all] [--qubits N] [--cpu]
    torchrun --nproc-per-node P --master-addr 127.0.0.1 benchmarks/adjoint_bench.py --config 3 --qubits 33

Under torchrun the state is sharded over P GPUs (global qubits = top log2 P; the NCCL id is
broadcast over a gloo group) and rank 0 prints the max-over-ranks time.

config 1: 20-qubit StronglyEntanglingLayers L=4, observables Z_0..Z_19 (20 x 240 Jacobian)
config 3: QAOA MaxCut p=2 on a 4-regular graph, C = sum 1/2 (1 - Z_i Z_j) (default n=31 on one
          GPU: psi + lambda = 64 GiB; the 33-qubit config needs two GPUs)
config 5: 28-qubit hardware-efficient ansatz, 18 layers, 1000 trainable, 1000-term random Pauli H
Each line: seconds per Jacobian (device time incl. forward pass), fused and per-gate sweeps, and
for config 1 the CPU oracle (numpy restatement of the reference) on one observable, scaled.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2403_02512_b200 import workloads  # noqa: E402
from paper_2403_02512_b200.device import Device  # noqa: E402


def make_device(n, dist):
    if dist is None:
        return Device(n)
    tdist, rank, world, local = dist
    nid = [Device.nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(nid, src=0)
    return Device.sharded(n, rank, world, nid[0], device=local)


def gpu_time(n, ops, obs, fuse, reps=3, dist=None):
    with make_device(n, dist) as d:
        d.adjoint_jacobian(ops, obs, fuse=fuse)      # warm-up (plans, allocations)
        ts = []
        for _ in range(reps):
            d.reset()
            d.synchronize()
            if dist:
                dist[0].barrier()
            t0 = time.perf_counter()
            jac = d.adjoint_jacobian(ops, obs, fuse=fuse)
            d.synchronize()
            t = time.perf_counter() - t0
            if dist:   # max over ranks
                tt = [None] * dist[2]
                dist[0].all_gather_object(tt, t)
                t = max(tt)
            ts.append(t)
            launches = d.launch_count
    return min(ts), jac, launches


def config(c, n):
    if c == 1:
        n = n or 20
        ops, obs = workloads.sel_config(n, 4, seed=0)
        return n, ops, obs, f"{n}q SEL L=4, {len(obs)} observables"
    if c == 3:
        n = n or 31
        ops, ham, edges = workloads.qaoa_maxcut(n, p=2, seed=0)
        return n, ops, [ham], f"{n}q QAOA MaxCut p=2 ({len(edges)} edges)"
    n = n or 28
    ops = workloads.hardware_efficient_ansatz(n, layers=18, n_trainable=1000, seed=0)
    ham = workloads.random_pauli_hamiltonian(n, 1000, seed=0)
    return n, ops, [ham], f"{n}q HEA 18 layers, 1000 trainable, 1000-term H"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="all")
    ap.add_argument("--qubits", type=int, default=0)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--skip-unfused", action="store_true")
    a = ap.parse_args()
    dist = None
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as tdist
        tdist.init_process_group("gloo", init_method="env://")
        dist = (tdist, tdist.get_rank(), tdist.get_world_size(), int(os.environ.get("LOCAL_RANK", "0")))
    cfgs = [1, 3, 5] if a.config == "all" else [int(a.config)]
    for c in cfgs:
        n, ops, obs, desc = config(c, a.qubits)
        ncols = sum(op.n_trainable for op in ops)
        t_f, jac_f, l_f = gpu_time(n, ops, obs, True, dist=dist)
        rec = {"config": c, "workload": desc, "n_qubits": n, "n_gpus": dist[2] if dist else 1,
               "jacobian_shape": [len(obs), ncols], "s_per_jacobian_fused": t_f}
        if not a.skip_unfused:
            t_u, jac_u, _ = gpu_time(n, ops, obs, False, reps=1, dist=dist)
            rec["s_per_jacobian_per_gate_sweep"] = t_u
            rec["fused_vs_per_gate_max_abs_diff"] = float(np.abs(jac_f - jac_u).max())
        if a.cpu and c == 1:
            from oracle import svoracle as O
            t0 = time.perf_counter()
            O.adjoint_jacobian(n, ops, obs[:1])
            t1 = time.perf_counter() - t0
            rec["cpu_oracle_s_one_observable"] = t1
            rec["cpu_oracle_s_estimated_all"] = t1 * len(obs)
            rec["cpu_cores"] = 1
        if dist is None or dist[1] == 0:
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
