"""Helpers to read the committed golden vectors (tests/golden/*.npz)."""

import ast
import os

import numpy as np

from paper_2403_02512_b200.ops import Op

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def unpack_ops(d, prefix):
    ops = []
    for rec in d[f"{prefix}_ops"]:
        name, wires, params, ctrls, vals, trainable, inverse, mi = ast.literal_eval(str(rec))
        m = d[f"{prefix}_mat{mi}"] if mi >= 0 else None
        ops.append(Op(name, wires, params, ctrls, vals, trainable, inverse, m))
    return ops


def unpack_obs(d, prefix):
    from paper_2403_02512_b200.observables import DenseHermitian, Hamiltonian, PauliWord
    out = []
    for rec in d[f"{prefix}_obs"]:
        r = ast.literal_eval(str(rec))
        if r[0] == "pauli":
            out.append(PauliWord(r[1]))
        elif r[0] == "ham":
            out.append(Hamiltonian(r[1], [PauliWord(f) for f in r[2]]))
        else:
            out.append(DenseHermitian(r[1], d[f"{prefix}_omat{r[2]}"]))
    return out


ADJ_JOBS = ("sel6", "rand0", "rand1", "rand2", "qaoa8")
