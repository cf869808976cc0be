"""Parity and timing at the north star's scale: sharded runs at 30-35 qubits
checked through size-independent properties, one JSON line per check.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 benchmarks/scale_parity.py --check agree --qubits 30
    torchrun ... --check roundtrip --qubits 35 --depth 20
    torchrun ... --check qaoa --qubits 33 [--adjoint]

agree     : the sharded state (P ranks) vs a single-GPU state of the same circuit built on rank 0's
            GPU: norm, <Z_q> for every q, <Z_q Z_q+1> for every q, and a p=1 QAOA Jacobian
            ("sharded vs 1-GPU at n <= 30, |delta| <= 1e-12").
roundtrip : U then U^dagger of a random RX/RY/RZ/CNOT circuit returns |0...0>: norm within 1e-12
            and <Z_q> = 1 within 1e-12 for every q (SPEC.md:466 sharded equivalence, at 34-35 qubits).
qaoa      : p = 1 QAOA MaxCut <C> vs the closed form (oracle/qaoa_closed_form.py), and with
            --adjoint the full 1 x (edges + n) Jacobian's expectation value and timing.
Times are device time, max over ranks.
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
from paper_2403_02512_b200.observables import PauliWord  # noqa: E402
from paper_2403_02512_b200.ops import Op  # noqa: E402


def setup():
    import torch.distributed as tdist
    tdist.init_process_group("gloo", init_method="env://")
    rank, world = tdist.get_rank(), tdist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return tdist, rank, world, local


def sharded(tdist, n, rank, world, local):
    nid = [Device.nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(nid, src=0)
    return Device.sharded(n, rank, world, nid[0], device=local)


def timed(tdist, world, dev, fn):
    dev.synchronize()
    tdist.barrier()
    t0 = time.perf_counter()
    out = fn()
    dev.synchronize()
    t = time.perf_counter() - t0
    ts = [None] * world
    tdist.all_gather_object(ts, t)
    return out, max(ts)


def z_profile(d, n):
    zs = [d.expval(PauliWord(((q, "Z"),))) for q in range(n)]
    zz = [d.expval(PauliWord(((q, "Z"), (q + 1, "Z")))) for q in range(n - 1)]
    return np.array(zs), np.array(zz)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", choices=["agree", "roundtrip", "qaoa"], required=True)
    ap.add_argument("--qubits", type=int, required=True)
    ap.add_argument("--depth", type=int, default=20)
    ap.add_argument("--adjoint", action="store_true")
    a = ap.parse_args()
    tdist, rank, world, local = setup()
    n = a.qubits
    rec = {"check": a.check, "n_qubits": n, "n_gpus": world}
    if a.check == "agree":
        ops = workloads.random_circuit(n, a.depth, seed=0)
        qops, qham, _ = workloads.qaoa_maxcut(n, p=1, seed=0)
        d = sharded(tdist, n, rank, world, local)
        d.apply(ops)   # warm-up
        d.reset()
        _, t = timed(tdist, world, d, lambda: d.apply(ops))
        norm = d.norm()
        zs, zz = z_profile(d, n)
        d.reset()
        jac, t_adj = timed(tdist, world, d, lambda: d.adjoint_jacobian(qops, [qham], return_expvals=True))
        d.release()
        if rank == 0:
            with Device(n, device=local) as s:
                s.apply(ops)
                norm1 = s.norm()
                zs1, zz1 = z_profile(s, n)
                s.reset()
                jac1 = s.adjoint_jacobian(qops, [qham], return_expvals=True)
            scale = float(np.abs(jac1[0]).max())
            rec.update({
                "workload": f"random circuit depth {a.depth} ({len(ops)} gates) + p=1 QAOA Jacobian 1x{jac1[0].shape[1]}",
                "s_per_circuit_sharded": t, "s_per_jacobian_sharded": t_adj,
                "norm_diff": abs(norm - norm1), "z_max_diff": float(np.abs(zs - zs1).max()),
                "zz_max_diff": float(np.abs(zz - zz1).max()),
                "jac_max_rel_diff": float(np.abs(jac[0] - jac1[0]).max()) / max(1.0, scale),
                "expval_diff": abs(float(jac[1][0]) - float(jac1[1][0])),
            })
            rec["pass"] = bool(rec["norm_diff"] < 1e-12 and rec["z_max_diff"] < 1e-12 and rec["zz_max_diff"] < 1e-12
                               and rec["jac_max_rel_diff"] < 1e-10 and rec["expval_diff"] < 1e-10 * max(1.0, abs(jac1[1][0])))
    elif a.check == "roundtrip":
        ops = workloads.random_circuit(n, a.depth, seed=0)
        inv = [Op(o.name, o.wires, o.params, o.ctrls, o.ctrl_values, (), not o.inverse) for o in reversed(ops)]
        d = sharded(tdist, n, rank, world, local)
        d.apply(ops)   # warm-up: plans and pass kernels compiled outside the timed region
        d.apply(inv)
        d.reset()
        _, t_fwd = timed(tdist, world, d, lambda: d.apply(ops))
        _, t_inv = timed(tdist, world, d, lambda: d.apply(inv))
        norm = d.norm()
        zs, _ = z_profile(d, n)
        d.release()
        rec.update({"workload": f"random circuit depth {a.depth} ({len(ops)} gates), then its inverse",
                    "s_per_circuit": t_fwd, "s_per_inverse": t_inv, "norm_diff": abs(norm - 1.0),
                    "z_min": float(zs.min()), "one_minus_z_max": float((1.0 - zs).max())})
        rec["pass"] = bool(rec["norm_diff"] < 1e-12 and rec["one_minus_z_max"] < 1e-12)
    else:
        from oracle.qaoa_closed_form import maxcut_p1_expectation
        ops, ham, edges = workloads.qaoa_maxcut(n, p=1, seed=0)
        g, b = ops[n].params[0] / 2, ops[-1].params[0] / 2
        ref = maxcut_p1_expectation(n, edges, g, b)
        d = sharded(tdist, n, rank, world, local)
        _, t_fwd = timed(tdist, world, d, lambda: d.apply(ops))
        ev = d.expval(ham)
        rec.update({"workload": f"p=1 QAOA MaxCut, 4-regular graph, {len(edges)} edges",
                    "s_forward": t_fwd, "expval": ev, "closed_form": ref, "abs_diff": abs(ev - ref)})
        ok = abs(ev - ref) < 1e-10 * max(1.0, abs(ref))
        if a.adjoint:
            d.reset()
            d.adjoint_jacobian(ops, [ham])   # warm-up (sweep plans, kernels, lambda buffer)
            d.reset()
            (jac, evs), t_adj = timed(tdist, world, d, lambda: d.adjoint_jacobian(ops, [ham], return_expvals=True))
            rec.update({"s_per_jacobian": t_adj, "jacobian_shape": list(jac.shape), "adjoint_expval_diff": abs(evs[0] - ref),
                        "jac_checksum": float(np.abs(jac).sum())})
            ok = ok and abs(evs[0] - ref) < 1e-10 * max(1.0, abs(ref))
        d.release()
        rec["pass"] = bool(ok)
    if rank == 0:
        print(json.dumps(rec), flush=True)
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
