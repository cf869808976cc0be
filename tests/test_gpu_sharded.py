"""GPU, world_size 2 (and 4 when available): sharded state over NCCL vs the oracle.

One process per GPU (SPEC.md:429-486 semantics; global qubits = top log2 P): state after
random circuits (global-qubit swaps), expvals with X/Y/Z on global qubits, probabilities over
global wires, and the adjoint Jacobian -- all against the monolithic oracle.
"""

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import svoracle as O
from paper_2403_02512_b200 import workloads
from paper_2403_02512_b200.observables import DenseHermitian, Hamiltonian, PauliWord
from paper_2403_02512_b200.ops import Op

pytestmark = pytest.mark.gpu


def n_gpus():
    from paper_2403_02512_b200 import _lib
    return _lib.device_count()


def _worker(rank, world, nccl_ids, q):
    try:
        from paper_2403_02512_b200.device import Device
        n = 12
        rng = np.random.default_rng(5)
        psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        psi /= np.linalg.norm(psi)
        ops = workloads.random_circuit(n, 10, seed=3)
        ops += [Op("SWAP", (0, 11)), Op("IsingXX", (1, 0), (0.3,)), Op("CNOT", (0, 1), ctrls=(5,)),
                Op("DoubleExcitation", (0, 1, 6, 7), (0.4,)), Op("RZ", (1,), (0.7,), ctrls=(0,))]
        res = {}
        m = rng.normal(size=(32, 32)) + 1j * rng.normal(size=(32, 32))
        dense = DenseHermitian((0, 9, 1, 4, 6), m + m.conj().T)
        for fuse in (False, True):
            d = Device.sharded(n, rank, world, nccl_ids[int(fuse)], device=rank, fuse=fuse)
            d.set_state(psi)
            d.apply(ops)
            res[f"state{int(fuse)}"] = d.get_state()
            ham = Hamiltonian([0.5, -0.3, 0.8], [PauliWord(((0, "X"), (3, "Y"))), PauliWord(((1, "Z"), (0, "Z"))),
                                                  PauliWord(((1, "Y"),))])
            res[f"ev{int(fuse)}"] = d.expval(ham)
            res[f"probs{int(fuse)}"] = d.probs([0, 7, 1])
            res[f"norm{int(fuse)}"] = d.norm()
            res[f"samp{int(fuse)}"] = d.sample_indices(5000, seed=99, wires=[0, 7, 1, 11])
            res[f"var{int(fuse)}"] = d.var(ham)
            res[f"dense{int(fuse)}"] = d.expval(dense)     # 5 wires incl. global qubit 0
            d.release()
        sel_ops, obs = workloads.sel_config(n, 2, seed=2)
        qaoa_ops, qaoa_h, _ = workloads.qaoa_maxcut(n, p=2, seed=1)
        hea_ops = workloads.hardware_efficient_ansatz(n, layers=3, n_trainable=60, seed=2)
        hea_h = workloads.random_pauli_hamiltonian(n, 12, seed=4)
        for fuse in (False, True):
            d = Device.sharded(n, rank, world, nccl_ids[2 + int(fuse)], device=rank, fuse=fuse)
            res[f"jac{int(fuse)}"], res[f"jev{int(fuse)}"] = d.adjoint_jacobian(sel_ops, obs[:3], return_expvals=True)
            res[f"qjac{int(fuse)}"], res[f"qjev{int(fuse)}"] = d.adjoint_jacobian(qaoa_ops, [qaoa_h], return_expvals=True)
            res[f"hjac{int(fuse)}"], res[f"hjev{int(fuse)}"] = d.adjoint_jacobian(hea_ops, [hea_h], return_expvals=True)
            d.release()
        if rank == 0:
            ref = O.run_circuit(n, ops, psi)
            out = {}
            for f in (0, 1):
                out[f"state{f}"] = float(np.abs(res[f"state{f}"] - ref).max())
                out[f"ev{f}"] = abs(res[f"ev{f}"] - O.expval(ref, n, ham))
                out[f"probs{f}"] = float(np.abs(res[f"probs{f}"] - O.probabilities(ref, n, [0, 7, 1])).max())
                out[f"norm{f}"] = abs(res[f"norm{f}"] - 1.0)
                out[f"samp{f}"] = float((res[f"samp{f}"] != O.sample(ref, n, 5000, seed=99, wires=[0, 7, 1, 11])).sum()) * 5e-13
                out[f"var{f}"] = abs(res[f"var{f}"] - O.variance(ref, n, ham))
                out[f"dense{f}"] = abs(res[f"dense{f}"] - O.expval(ref, n, dense)) / max(1.0, np.abs(dense.matrix).sum())
            refs = {"": O.adjoint_jacobian(n, sel_ops, obs[:3]), "q": O.adjoint_jacobian(n, qaoa_ops, [qaoa_h]),
                    "h": O.adjoint_jacobian(n, hea_ops, [hea_h])}
            for key, (jref, evref) in refs.items():
                for f in (0, 1):
                    scale = max(1.0, float(np.abs(jref).max()))
                    out[f"{key}jac{f}"] = float(np.abs(res[f"{key}jac{f}"] - jref).max()) / scale
                    out[f"{key}jev{f}"] = float(np.abs(np.asarray(res[f"{key}jev{f}"]) - evref).max()) / scale
            q.put(("ok", out))
    except Exception as exc:  # surface worker failures to the test
        import traceback
        q.put(("err", f"rank {rank}: {exc}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_nccl_matches_oracle(world):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2403_02512_b200.device import Device
    nccl_ids = [Device.nccl_unique_id() for _ in range(4)]   # one id per communicator
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, nccl_ids, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", out
    for k, v in out.items():
        tol = 1e-10 if "j" in k else 1e-12
        assert v < tol, (k, v)


def _swap_path_worker(rank, world, nccl_ids, q):
    try:
        import os
        from paper_2403_02512_b200.device import Device
        n = 14
        ops = workloads.random_circuit(n, 12, seed=8)
        qaoa_ops, qaoa_h, _ = workloads.qaoa_maxcut(n, p=2, seed=3)
        res = []
        for i, flag in enumerate(("1", "0")):   # peer-memory swaps, then the NCCL send/recv fallback
            os.environ["SVB200_P2P_SWAP"] = flag
            d = Device.sharded(n, rank, world, nccl_ids[2 * i], device=rank)
            d.apply(ops)
            st = d.get_state()
            d.release()
            d = Device.sharded(n, rank, world, nccl_ids[2 * i + 1], device=rank)
            jac = d.adjoint_jacobian(qaoa_ops, [qaoa_h])
            d.reset()
            d.apply(ops)
            ev = d.expval(qaoa_h)   # diagonal group of 28 ZZ terms on 2^13-amplitude shards: WHT kernel
            ev_terms = sum(c * d.expval(t) for c, t in zip(qaoa_h.coeffs, qaoa_h.terms))   # per-term kernel
            st2 = d.get_state()
            d.release()
            res.append((st, jac, (ev, ev_terms), st2))
        if rank == 0:
            same_state = bool(np.array_equal(res[0][0].view(np.uint64), res[1][0].view(np.uint64)))
            same_jac = bool(np.array_equal(res[0][1], res[1][1]))
            jref, _ = O.adjoint_jacobian(n, qaoa_ops, [qaoa_h])
            scale = sum(abs(c) for c in qaoa_h.coeffs)
            jac_ok = bool(np.abs(res[0][1] - jref).max() < 1e-10 * max(1.0, scale, float(np.abs(jref).max())))
            psi = O.run_circuit(n, ops)
            ev_ref = O.expval(psi, n, qaoa_h)
            ev_ok = bool(abs(res[0][2][0] - ev_ref) < 1e-12 * max(1.0, scale))
            if not ev_ok:
                ev_ok = (res[0][2], ev_ref, float(np.abs(res[0][0] - psi).max()), float(np.abs(res[0][3] - psi).max()),
                         O.expval(res[0][0], n, qaoa_h), O.expval(res[0][3], n, qaoa_h))
            q.put(("ok", {"state": same_state, "jac": same_jac, "jac_vs_oracle": jac_ok, "ev_vs_oracle": ev_ok}))
    except Exception as exc:
        import traceback
        q.put(("err", f"rank {rank}: {exc}\n{traceback.format_exc()}"))


def test_peer_memory_swap_bit_identical_to_nccl_swap():
    """The peer-memory exchange kernel and the NCCL send/recv path move the same amplitudes:
    states and Jacobians must agree bit for bit."""
    world = 2
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2403_02512_b200.device import Device
    nccl_ids = [Device.nccl_unique_id() for _ in range(4)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_swap_path_worker, args=(r, world, nccl_ids, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", out
    assert out == {"state": True, "jac": True, "jac_vs_oracle": True, "ev_vs_oracle": True}, out
