"""GPU, world_size 2, 4 and 8 (each skipped without enough GPUs): sharded state over NCCL vs the oracle.

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


def run_world(target, world, n_ids, timeout=900):
    """Spawn one process per GPU, return rank 0's (status, result).  A rank that fails makes its
    peers' NCCL waits time out (SVB200_NCCL_TIMEOUT, communicator aborted) instead of hanging; any
    process still alive at the end is killed."""
    import os
    from paper_2403_02512_b200.device import Device
    os.environ.setdefault("SVB200_NCCL_TIMEOUT", "180")
    nccl_ids = [Device.nccl_unique_id() for _ in range(n_ids)]   # one id per communicator
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, nccl_ids, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        status, out = q.get(timeout=timeout)
    finally:
        for p in procs:
            p.join(timeout=60 if p is procs[0] else 30)
            if p.is_alive():
                p.kill()
    return status, out


# Shards span several 2^12-amplitude tiles (n_local = 14): the sharded fused passes run their
# multi-tile tile loops on every rank (the bug class of round 1 lived exactly there).
N_LOCAL = 14


def sharded_ops(n, world, seed=3):
    """Random circuit plus gates whose targets, controls and partners sit on the global qubits
    0 .. log2(world)-1: globally-controlled gates (no exchange), dense gates across two global bits
    (multi-bit exchange), SWAP / DoubleExcitation spanning global and local bits."""
    g = world.bit_length() - 1
    ops = workloads.random_circuit(n, 10, seed=seed)
    ops += [Op("SWAP", (0, n - 1)), Op("IsingXX", (1 % n, 0), (0.3,)), Op("CNOT", (0, 1), ctrls=(5,)),
            Op("DoubleExcitation", (0, 1, 6, 7), (0.4,)), Op("RZ", (1,), (0.7,), ctrls=(0,)),
            Op("RY", (n - 2,), (0.9,), ctrls=(0,), ctrl_values=(0,)),
            Op("CNOT", (n - 3, n - 4), ctrls=(g - 1,)),
            Op("Rot", (g - 1,), (0.1, 0.2, 0.3)),
            Op("IsingXY", (0, g - 1) if g > 1 else (0, 2), (0.6,)),
            Op("SWAP", (0, g - 1) if g > 1 else (0, 3)),
            Op("RX", (n - 1,), (1.1,), ctrls=(g - 1,)),
            Op("H", (g - 1,)), Op("CZ", (0, g - 1) if g > 1 else (0, 4))]
    ops += workloads.random_circuit(n, 4, seed=seed + 1)
    return ops


def _worker(rank, world, nccl_ids, q):
    try:
        from paper_2403_02512_b200.device import Device
        n = N_LOCAL + world.bit_length() - 1
        rng = np.random.default_rng(5)
        psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        psi /= np.linalg.norm(psi)
        ops = sharded_ops(n, world)
        res = {}
        m = rng.normal(size=(32, 32)) + 1j * rng.normal(size=(32, 32))
        dense = DenseHermitian((0, 9, 1, 4, 6), m + m.conj().T)
        for fuse in (False, True):
            d = Device.sharded(n, rank, world, nccl_ids[int(fuse)], device=rank, fuse=fuse)
            assert d.n_local >= 13, "shards must span several fused tiles"
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


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_nccl_matches_oracle(world):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    status, out = run_world(_worker, world, 4)
    assert status == "ok", out
    for k, v in out.items():
        tol = 1e-10 if "j" in k else 1e-12
        assert v < tol, (k, v)


def _swap_path_worker(rank, world, nccl_ids, q):
    try:
        import os
        from paper_2403_02512_b200.device import Device
        n = N_LOCAL + world.bit_length() - 1
        ops = sharded_ops(n, world, seed=8)
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
            ev_ok = bool(abs(res[0][2][0] - ev_ref) < 1e-12 * max(1.0, scale)
                         and abs(res[0][2][1] - ev_ref) < 1e-12 * max(1.0, scale))
            if not ev_ok:
                ev_ok = (res[0][2], ev_ref, float(np.abs(res[0][0] - psi).max()), float(np.abs(res[0][3] - psi).max()),
                         O.expval(res[0][0], n, qaoa_h), O.expval(res[0][3], n, qaoa_h))
            q.put(("ok", {"state": same_state, "jac": same_jac, "jac_vs_oracle": jac_ok, "ev_vs_oracle": ev_ok}))
    except Exception as exc:
        import traceback
        q.put(("err", f"rank {rank}: {exc}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("world", [2, 4])
def test_peer_memory_swap_bit_identical_to_nccl_swap(world):
    """The peer-memory exchange kernels (single- and multi-bit) and the NCCL send/recv path move
    the same amplitudes: states and Jacobians must agree bit for bit."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    status, out = run_world(_swap_path_worker, world, 4)
    assert status == "ok", out
    assert out == {"state": True, "jac": True, "jac_vs_oracle": True, "ev_vs_oracle": True}, out


def _dead_peer_worker(rank, world, nccl_ids, q):
    import os
    import time
    os.environ["SVB200_NCCL_TIMEOUT"] = "20"
    from paper_2403_02512_b200.device import Device
    from paper_2403_02512_b200.errors import DeviceError
    d = Device.sharded(16, rank, world, nccl_ids[0], device=rank)
    if rank == 1:
        os._exit(0)   # the peer disappears without a word
    t0 = time.time()
    log = os.environ.get("SVB200_TEST_LOG")
    try:
        d.expval(PauliWord(((0, "Z"),)))   # an allreduce no peer will ever join
        q.put(("ok", "collective returned without its peer"))
    except DeviceError as e:
        if log:
            with open(log, "a") as f:
                f.write(f"rank 0 raised after {time.time() - t0:.1f} s: {e}\n")
        q.put(("ok", ("aborted", str(e), time.time() - t0)))
    if log:
        with open(log, "a") as f:
            f.write("rank 0 releasing\n")
    d.release()
    if log:
        with open(log, "a") as f:
            f.write("rank 0 released\n")


def test_dead_peer_aborts_instead_of_hanging():
    """A rank whose peer died does not hang in NCCL: the stream watchdog aborts the communicator
    (ncclCommAbort) after SVB200_NCCL_TIMEOUT seconds and the call raises DeviceError."""
    world = 2
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    status, out = run_world(_dead_peer_worker, world, 1, timeout=300)
    assert status == "ok" and out[0] == "aborted", out
    assert "aborted" in out[1] and out[2] < 120, out
