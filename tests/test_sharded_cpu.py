"""CPU, world_size 2, 4 and 8 over gloo: the sharded driver's own decisions (sv_plan_sharded:
per-rank local primitives, global-qubit swaps, final canonicalisation) replayed on CPU ranks
reproduce the monolithic oracle ("sharded equivalence").

Each rank holds its contiguous shard (global qubits = top log2 P); a recorded swap
of global position G with the top local bit exchanges one half-shard with rank ^ (1 << (G - nl))
through torch.distributed send/recv -- the same data movement dist.cpp does with ncclSend/Recv.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import svoracle as O
from paper_2403_02512_b200 import _lib, workloads
from paper_2403_02512_b200.ops import Op


def plan_sharded(n, rank, world, ops):
    packed = _lib.PackedOps(ops)
    sizes = (ctypes.c_int64 * 2)()
    L = _lib.lib()
    _lib.check(L.sv_plan_sharded(n, rank, world, packed.ptr, packed.n, None, 0, None, 0, sizes))
    ints = np.zeros(sizes[0], dtype=np.int64)
    dbls = np.zeros(max(sizes[1], 1), dtype=np.float64)
    _lib.check(L.sv_plan_sharded(n, rank, world, packed.ptr, packed.n,
                                 ints.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), sizes[0],
                                 dbls.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), sizes[1], sizes))
    return ints, dbls[: sizes[1]]


def replay(rank, world, ints, dbls, shard):
    import torch
    C = dbls[0::2] + 1j * dbls[1::2]
    I = [int(x) for x in ints]
    pos = 0

    def nxt():
        nonlocal pos
        pos += 1
        return I[pos - 1]

    assert nxt() == 1
    n, nl, r, w, nsteps = nxt(), nxt(), nxt(), nxt(), nxt()
    assert (r, w) == (rank, world)
    idx = np.arange(1 << nl, dtype=np.int64)
    swaps = 0
    for _ in range(nsteps):
        kind = nxt()
        if kind == 1:   # global swap: exchange our (top local bit = 1 - b) half with the partner
            G = nxt()
            j = G - nl
            partner = rank ^ (1 << j)
            b = (rank >> j) & 1
            half = 1 << (nl - 1)
            off = half if b == 0 else 0
            send = torch.from_numpy(np.ascontiguousarray(shard[off:off + half]).view(np.float64).copy())
            recv = torch.empty_like(send)
            if rank < partner:
                dist.send(send, partner)
                dist.recv(recv, partner)
            else:
                dist.recv(recv, partner)
                dist.send(send, partner)
            shard[off:off + half] = recv.numpy().view(np.complex128)
            swaps += 1
            continue
        if kind == 2:   # multi-bit exchange (dist.cpp exchange_bits): global Gs[i] <-> local ps[i]
            k = nxt()
            Gs, ps = [], []
            for _ in range(k):
                Gs.append(nxt())
                ps.append(nxt())
            g = sum(((rank >> (G - nl)) & 1) << i for i, G in enumerate(Gs))
            vbits = sum(((idx >> p) & 1) << i for i, p in enumerate(ps))
            for step in range(1, 1 << k):   # XOR schedule, as the NCCL fallback runs it
                c = g ^ step
                partner = rank
                for i, G in enumerate(Gs):
                    partner = (partner & ~(1 << (G - nl))) | (((c >> i) & 1) << (G - nl))
                sel = idx[vbits == c]   # ascending = ordered by the non-victim bits on both ranks
                send = torch.from_numpy(np.ascontiguousarray(shard[sel]).view(np.float64).copy())
                recv = torch.empty_like(send)
                if rank < partner:
                    dist.send(send, partner)
                    dist.recv(recv, partner)
                else:
                    dist.recv(recv, partner)
                    dist.send(send, partner)
                shard[sel] = recv.numpy().view(np.complex128)
            swaps += 1
            continue
        t, fmask, fval, xmask, nb = nxt(), nxt() & 0xFFFFFFFFFFFFFFFF, nxt() & 0xFFFFFFFFFFFFFFFF, \
            nxt() & 0xFFFFFFFFFFFFFFFF, nxt()
        pp = [nxt() for _ in range(nb)]
        moff, mlen = nxt(), nxt()
        m = C[moff:moff + mlen]
        sel = idx[(idx & fmask) == fval]
        if t == 0:
            i0, i1 = sel, sel ^ xmask
            a0, a1 = shard[i0].copy(), shard[i1].copy()
            shard[i0] = m[0] * a0 + m[1] * a1
            shard[i1] = m[2] * a0 + m[3] * a1
        elif t == 1:
            tt = np.zeros_like(sel)
            for j, q in enumerate(pp):
                tt |= ((sel >> q) & 1) << j
            shard[sel] *= m[tt]
        else:
            d = 1 << nb
            offs = np.array([sum(((rr >> j) & 1) << q for j, q in enumerate(pp)) for rr in range(d)])
            grp = sel[:, None] | offs[None, :]
            shard[grp] = shard[grp] @ m.reshape(d, d).T
    phys = [nxt() for _ in range(n)]
    assert phys == list(range(n)), "driver must leave the canonical layout after canonicalisation"
    return swaps


def _worker(rank, world, port, n, seed, ops_kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = make_ops(ops_kind, n, seed)
        rng = np.random.default_rng(seed)
        psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        psi /= np.linalg.norm(psi)
        nl = n - (world.bit_length() - 1)
        shard = psi[rank << nl:(rank + 1) << nl].copy()
        ints, dbls = plan_sharded(n, rank, world, ops)
        swaps = replay(rank, world, ints, dbls, shard)
        import torch
        parts = [torch.empty(2 << nl, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(shard.view(np.float64).copy()))
        if rank == 0:
            got = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            ref = O.run_circuit(n, ops, psi)
            q.put((float(np.abs(got - ref).max()), swaps))
    finally:
        dist.destroy_process_group()


def make_ops(kind, n, seed):
    if kind == "random":
        return workloads.random_circuit(n, 8, seed=seed)
    if kind == "sel":
        return workloads.strongly_entangling_layers(n, np.random.default_rng(seed).uniform(0, 6, size=(2, n, 3)))
    rng = np.random.default_rng(seed)
    ops = []
    for _ in range(60):   # controls / diagonals / dense targets on the global qubits
        a, b, c = (int(x) for x in rng.choice(n, size=3, replace=False))
        pick = int(rng.integers(6))
        if pick == 0:
            ops.append(Op("CNOT", (a, b)))
        elif pick == 1:
            ops.append(Op("RZ", (a,), (float(rng.uniform(0, 6)),)))
        elif pick == 2:
            ops.append(Op("IsingZZ", (a, b), (float(rng.uniform(0, 6)),)))
        elif pick == 3:
            ops.append(Op("RY", (a,), (float(rng.uniform(0, 6)),), ctrls=(b, c), ctrl_values=(1, 0)))
        elif pick == 4:
            ops.append(Op("IsingXX", (a, b), (float(rng.uniform(0, 6)),)))
        else:
            ops.append(Op("SWAP", (a, b)))
    return ops


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,kind", [(2, "random"), (2, "mixed"), (4, "sel"), (4, "mixed"), (8, "random"),
                                        (8, "mixed")])
def test_sharded_replay_matches_monolithic(world, kind):
    n = 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, 11, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    err, swaps = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12
    assert swaps > 0


def test_multi_bit_exchange_is_one_all_to_all():
    """At P = 8 a layer that needs all three global qubits brings them in with one exchange
    (multi-bit swaps via all-to-all), not three sequential pairwise swaps."""
    n = 10
    ops = [Op("RX", (q,), (0.1 * (q + 1),)) for q in range(n)]   # every qubit, globals first
    ints, _ = plan_sharded(n, 0, 8, ops)
    nsteps, pos, xs = int(ints[5]), 6, []
    for _ in range(nsteps):
        k = int(ints[pos])
        if k == 2:
            xs.append(int(ints[pos + 1]))
            pos += 2 + 2 * int(ints[pos + 1])
        elif k == 1:
            pos += 2
        else:
            nb = int(ints[pos + 5])
            pos += 6 + nb + 2
    assert xs and xs[0] == 3, xs


def test_plan_sharded_no_comm_for_diagonal_and_controls_on_global():
    """Diagonal gates and controls on global qubits need no exchange (SURVEY §8(e) no-comm cases)."""
    n = 8
    ops = [Op("RZ", (0,), (0.3,)), Op("CZ", (0, 1)), Op("IsingZZ", (1, 5), (0.2,)),
           Op("CNOT", (0, 4)), Op("RY", (6,), (0.4,), ctrls=(1,))]
    for rank in range(4):
        ints, _ = plan_sharded(n, rank, 4, ops)
        nsteps = int(ints[5])
        kinds, pos = [], 6
        for _ in range(nsteps):
            k = int(ints[pos])
            kinds.append(k)
            if k == 1:
                pos += 2
            elif k == 2:
                pos += 2 + 2 * int(ints[pos + 1])
            else:
                nb = int(ints[pos + 5])
                pos += 6 + nb + 2
        assert 1 not in kinds
