"""Single-GPU numbers for BASELINE.md §5 (one JSON line per row).

    python benchmarks/results.py [--rows 1,2,3,5] [--cpu-seconds 20]

row 1: 20q SEL L=4 Jacobian (20 x 240): device s/Jacobian, max |d| vs the reference-backed golden
       (tests/golden/sel20_golden.npz), and the numpy oracle on one observable x 20 (labelled estimate)
row 2: unfused gate kernels at 30 qubits on every target (RX, H, CNOT(q, q+1)): GB/s min/mean
row 2c: CNOT on every ordered (control, target) pair at 30 qubits
row 2f: the same for a complex64 ("f32") state at 31 qubits (also 16 GiB)
row 3: 33q QAOA p=2 forward + <C> on one GPU (the 33q adjoint needs psi + lambda = 256 GiB: 2 GPUs,
       benchmarks/adjoint_bench.py under torchrun)
row 5: 28q HEA (1000 trainable, 1000-term H): s per expval + gradient
row 5s: the same with a 9000-term H (SURVEY §8(d) stress variant)
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
from paper_2403_02512_b200.ops import Op  # noqa: E402

PEAK = 6551.0


def row1(cpu_seconds):
    from tests.golden_io import load
    from oracle import svoracle as O
    ops, obs = workloads.sel_config(20, 4, seed=0)
    with Device(20) as d:
        d.adjoint_jacobian(ops, obs)
        ts = []
        for _ in range(3):
            d.reset()
            d.synchronize()
            t0 = time.perf_counter()
            jac, ev = d.adjoint_jacobian(ops, obs, return_expvals=True)
            d.synchronize()
            ts.append(time.perf_counter() - t0)
    g = load("sel20_golden.npz")
    rec = {"row": 1, "workload": "20q SEL L=4, Z_0..Z_19, Jacobian 20x240", "s_per_jacobian": min(ts),
           "parity_max_abs_jac": float(np.abs(jac - g["jac"]).max()),
           "parity_max_abs_expval": float(np.abs(ev - g["expvals"]).max())}
    t0 = time.perf_counter()
    O.adjoint_jacobian(20, ops, obs[:1])
    t1 = time.perf_counter() - t0
    rec.update({"cpu_oracle_s_one_observable": t1, "cpu_oracle_s_20_observables_estimate": 20 * t1,
                "cpu_kind": "numpy oracle (restatement of svkit on apply_matrix), default BLAS threads",
                "cpu_cores": len(os.sched_getaffinity(0))})
    return rec


def row2(precision="f64"):
    n = 30 if precision == "f64" else 31
    out = {}
    with Device(n, precision=precision, fuse=False) as d:
        for name, mk in (("RX", lambda q: Op("RX", (q,), (0.3,))), ("H", lambda q: Op("H", (q,))),
                         ("CNOT", lambda q: Op("CNOT", (q, (q + 1) % n)))):
            gbs = []
            for q in range(n):
                op = [mk(q)]
                d.apply(op)
                d.reset_stats()
                d.set_profiling(True)
                for _ in range(3):
                    d.apply(op)
                st = d.kernel_stats()
                d.set_profiling(False)
                ms = sum(v["ms"] for v in st.values())
                by = sum(v["bytes"] for v in st.values())
                gbs.append(by / (ms / 1e3) / 1e9)
            out[name] = {"min_GBps": min(gbs), "mean_GBps": float(np.mean(gbs)), "max_GBps": max(gbs),
                         "mean_frac_of_6551": float(np.mean(gbs)) / PEAK, "mean_frac_of_8000": float(np.mean(gbs)) / 8000}
    if precision == "f32":
        return {"row": "2f", "workload": "unfused single-gate kernels, complex64 at 31 qubits, every target", **out}
    return {"row": 2, "workload": "unfused single-gate kernels at 30 qubits, every target", **out}


def row2c():
    """CNOT on every ordered (control, target) pair at 30 qubits (PAPER.md:128 'every gate index
    pairing'): GB/s of algorithmic bytes (the half of the state a CNOT changes).
    A control on physical bit 0 (qubit n-1) changes one amplitude of every 32-byte sector, so
    DRAM moves twice the algorithmic bytes there: those pairs are reported separately."""
    n = 30
    rows = {}
    with Device(n, fuse=False) as d:
        for c in range(n):
            for t in range(n):
                if c == t:
                    continue
                op = [Op("CNOT", (c, t))]
                d.apply(op)
                d.reset_stats()
                d.set_profiling(True)
                for _ in range(2):
                    d.apply(op)
                st = d.kernel_stats()
                d.set_profiling(False)
                ms = sum(v["ms"] for v in st.values())
                by = sum(v["bytes"] for v in st.values())
                rows[(c, t)] = by / (ms / 1e3) / 1e9
    g = np.array(list(rows.values()))
    ctrl0 = np.array([v for (c, t), v in rows.items() if c == n - 1])
    rest = np.array([v for (c, t), v in rows.items() if c != n - 1])
    worst = sorted(rows.items(), key=lambda kv: kv[1])[:5]
    return {"row": "2c", "workload": "unfused CNOT, 30 qubits, all 870 ordered (control, target) pairs",
            "min_GBps": float(g.min()), "mean_GBps": float(g.mean()), "max_GBps": float(g.max()),
            "mean_frac_of_6551": float(g.mean()) / PEAK,
            "control_not_on_bit0": {"min_GBps": float(rest.min()), "mean_GBps": float(rest.mean())},
            "control_on_bit0": {"mean_GBps": float(ctrl0.mean()),
                                "note": "half of every 32 B sector changes: DRAM traffic = 2x algorithmic"},
            "worst5": [[c, t, v] for (c, t), v in worst]}


def row3():
    n = 33
    ops, ham, edges = workloads.qaoa_maxcut(n, p=2, seed=0)
    with Device(n) as d:
        d.apply(ops)
        d.expval(ham)
        ts = []
        for _ in range(2):
            d.reset()
            d.synchronize()
            t0 = time.perf_counter()
            d.apply(ops)
            e = d.expval(ham)
            d.synchronize()
            ts.append(time.perf_counter() - t0)
    return {"row": 3, "workload": f"33q QAOA MaxCut p=2 ({len(edges)} edges): forward + <C>", "s": min(ts),
            "expval": e, "state_GiB": 16 * 2 ** n / 2 ** 30}


def row5():
    n = 28
    ops = workloads.hardware_efficient_ansatz(n, layers=18, n_trainable=1000, seed=0)
    ham = workloads.random_pauli_hamiltonian(n, 1000, seed=0)
    with Device(n) as d:
        d.adjoint_jacobian(ops, [ham])
        ts = []
        for _ in range(2):
            d.reset()
            d.synchronize()
            t0 = time.perf_counter()
            jac, ev = d.adjoint_jacobian(ops, [ham], return_expvals=True)
            d.synchronize()
            ts.append(time.perf_counter() - t0)
    return {"row": 5, "workload": "28q HEA 18 layers, 1000 trainable, 1000-term H: expval + gradient",
            "s": min(ts), "expval": float(ev[0])}


def row5s():
    """Config 5's stress variant (T ~ 9000 terms, C2H4 scale)."""
    n = 28
    ops = workloads.hardware_efficient_ansatz(n, layers=18, n_trainable=1000, seed=0)
    ham = workloads.random_pauli_hamiltonian(n, 9000, seed=1)
    with Device(n) as d:
        d.adjoint_jacobian(ops, [ham])
        d.reset()
        d.synchronize()
        d.reset_stats()
        d.set_profiling(True)
        t0 = time.perf_counter()
        jac, ev = d.adjoint_jacobian(ops, [ham], return_expvals=True)
        d.synchronize()
        t = time.perf_counter() - t0
        st = {k: {"launches": v["launches"], "ms": v["ms"]} for k, v in d.kernel_stats().items() if v["launches"]}
        d.set_profiling(False)
    return {"row": "5s", "workload": "28q HEA 18 layers, 1000 trainable, 9000-term random Pauli H: expval + gradient",
            "s": t, "expval": float(ev[0]), "kernel_classes": st}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="1,2,3,5")
    ap.add_argument("--cpu-seconds", type=float, default=20)
    a = ap.parse_args()
    fns = {"1": lambda: row1(a.cpu_seconds), "2": row2, "2c": row2c, "2f": lambda: row2("f32"), "3": row3, "5": row5, "5s": row5s}
    for r in a.rows.split(","):
        print(json.dumps(fns[r]()), flush=True)


if __name__ == "__main__":
    main()
