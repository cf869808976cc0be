"""Observable batching across GPUs: ``batched_expval_and_grad``.

The paper's single-producer / multi-consumer pipeline (PAPER §2 Listing 2): the Hamiltonian's
terms are split into chunks, a pool of workers -- one per GPU, each owning a private state in
that GPU's HBM -- computes the energy and gradient of its chunks with ONE adjoint call (forward
pass once, one reverse sweep per chunk), and the results are merged by chunk index in a fixed
order. Workers are host threads (the C-ABI releases the GIL), so the pool scales over the GPUs
of one node without any data-path collective: linearity of the gradient in the observable is
the only "exchange".

Partition rule: without ``batch_size`` the n terms go to g chunks of
ceil/floor(n/g) (9 terms, g=4 -> 3,2,2,2); with ``batch_size`` b, chunks of b terms are dealt to
the workers round-robin (b trades memory -- one lambda per chunk in flight -- for recompute).

Determinism ("bit-identical for g in {1,2,4,8} and b in {1,3,n}"): the unit of
arithmetic is a CANONICAL chunk that depends on the Hamiltonian alone -- the terms split by the
ceil(n/8) rule into at most 8 chunks -- never on g or b.  Each canonical chunk's energy and
gradient come from one reverse sweep with that chunk as the observable; the workers (the SPEC
partition above decides which worker owns which canonical chunk: the owner of its first term)
only change where a chunk is computed, and b only how many canonical chunks share one adjoint
call (one forward pass).  The merge sums canonical chunks in chunk order, so energy and gradient
are bit-identical for every g and b; they equal the unbatched adjoint within 1e-12.

Environment overrides (the paper's PL_FWD_BATCH / PL_BWD_BATCH analogue):
``SVB200_BATCH_WORKERS`` (default: number of visible GPUs), ``SVB200_BATCH_SIZE``.
"""

import os
import threading

import numpy as np

from . import _lib
from .device import Device
from .errors import ValidationError
from .observables import Hamiltonian, PauliWord, as_observable
from .ops import Op


def plan_chunks(n_terms, n_workers, batch_size=None):
    """Chunk plan: list of (worker, [term indices]) in chunk order."""
    if n_workers < 1:
        raise ValidationError("n_workers must be >= 1")
    if batch_size is not None and batch_size < 1:
        raise ValidationError("batch_size must be >= 1")
    if batch_size is None:
        base, extra = divmod(n_terms, n_workers)
        chunks, start = [], 0
        for w in range(n_workers):
            size = base + (1 if w < extra else 0)
            chunks.append((w, list(range(start, start + size))))
            start += size
        return chunks
    return [(k % n_workers, list(range(s, min(s + batch_size, n_terms))))
            for k, s in enumerate(range(0, n_terms, batch_size))]


def batched_expval_and_grad(ops, hamiltonian, n_workers=None, batch_size=None, devices=None, fuse=True,
                            n_qubits=None):
    """(energy, gradient) of <H> for the circuit ``ops`` applied to |0...0>.

    ``devices``: GPU ordinals the workers are placed on (worker w -> devices[w % len]);
    default all visible GPUs. ``n_qubits`` defaults to the highest wire used + 1.
    """
    ops = [o if isinstance(o, Op) else Op(*o) for o in ops]
    h = as_observable(hamiltonian)
    if isinstance(h, PauliWord):
        h = Hamiltonian((1.0,), (h,))
    if not isinstance(h, Hamiltonian):
        raise ValidationError("batched_expval_and_grad takes a Pauli-sum Hamiltonian")
    if n_qubits is None:
        n_qubits = 1 + max([q for o in ops for q in tuple(o.wires) + tuple(o.ctrls)] +
                           [q for t in h.terms for q, _ in t.factors] + [0])
    if devices is None:
        devices = list(range(max(1, _lib.device_count())))
    if n_workers is None:
        n_workers = int(os.environ.get("SVB200_BATCH_WORKERS", len(devices)))
    if batch_size is None and os.environ.get("SVB200_BATCH_SIZE"):
        batch_size = int(os.environ["SVB200_BATCH_SIZE"])
    plan = plan_chunks(len(h.terms), n_workers, batch_size)
    canon = canonical_chunks(len(h.terms))
    owner_of_term = {}
    for w, idx in plan:
        for i in idx:
            owner_of_term[i] = w
    owner = [owner_of_term[idx[0]] for idx in canon]
    per_call = max(1, (batch_size or len(h.terms)) // max(1, len(canon[0]))) if canon else 1
    ncols = sum(op.n_trainable for op in ops)
    energy_c = [0.0] * len(canon)
    grad_c = [np.zeros(ncols) for _ in canon]
    errors = []

    def worker(w):
        mine = [k for k in range(len(canon)) if owner[k] == w]
        if not mine:
            return
        try:
            with Device(n_qubits, device=devices[w % len(devices)], fuse=fuse) as dev:
                for s in range(0, len(mine), per_call):   # b: canonical chunks per adjoint call
                    ks = mine[s:s + per_call]
                    obs = [Hamiltonian(tuple(h.coeffs[i] for i in canon[k]), tuple(h.terms[i] for i in canon[k]))
                           for k in ks]
                    dev.reset()
                    jac, ev = dev.adjoint_jacobian(ops, obs, return_expvals=True)
                    for r, k in enumerate(ks):
                        energy_c[k] = float(ev[r])
                        grad_c[k] = jac[r]
        except Exception as exc:  # surfaced on the calling thread
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(w,)) for w in range(n_workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    energy = 0.0
    grad = np.zeros(ncols)
    for k in range(len(canon)):         # fixed reduction order: canonical chunk index
        energy += energy_c[k]
        grad = grad + grad_c[k]
    return energy, grad


def canonical_chunks(n_terms, max_chunks=8):
    """The arithmetic unit of batching: the ceil(n/8) partition of the terms (at most 8 chunks),
    a function of the Hamiltonian alone (g and b never regroup terms)."""
    if n_terms == 0:
        return []
    return [idx for _, idx in plan_chunks(n_terms, min(max_chunks, n_terms)) if idx]
