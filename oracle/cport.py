"""ctypes loader + gcc build for oracle/c/svport.c -- TEST / BASELINE INFRASTRUCTURE ONLY.

The C port restates the reference's Alg. 1 / Alg. 2 (state.py:154-226) with OpenMP over the
disjoint pairs. bench.py times it as the CPU baseline ("kind": "port"); tests check it
against the numpy oracle. Never imported by the product package.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "svport.c")
LIB = os.path.join(HERE, "libsvport.so")

_lib = None


def build(force=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    # x86-64-v3 (AVX2): portable to the GPU box's host CPU, unlike -march=native
    cmd = ["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-shared", "-fPIC", SRC, "-o", LIB + ".tmp"]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        dp, ip = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
        L.svp_apply_1q.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int]
        L.svp_apply_ctrl_1q.argtypes = [dp, ctypes.c_int, ip, ip, ctypes.c_int, ctypes.c_int, dp, ctypes.c_int]
        L.svp_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads():
    return lib().svp_max_threads()


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def apply_1q(amps, n, q, m, threads=0):
    m = np.ascontiguousarray(m, dtype=np.complex128)
    lib().svp_apply_1q(_dp(amps.view(np.float64)), int(n), int(q), _dp(m.view(np.float64)), int(threads or max_threads()))


def apply_ctrl_1q(amps, n, ctrls, vals, q, m, threads=0):
    c = np.ascontiguousarray(ctrls, dtype=np.int32)
    v = np.ascontiguousarray(vals, dtype=np.int32)
    m = np.ascontiguousarray(m, dtype=np.complex128)
    ip = ctypes.POINTER(ctypes.c_int)
    lib().svp_apply_ctrl_1q(_dp(amps.view(np.float64)), int(n), c.ctypes.data_as(ip), v.ctypes.data_as(ip), len(c),
                            int(q), _dp(m.view(np.float64)), int(threads or max_threads()))


def apply_op(amps, n, op, threads=0):
    """Apply one 1q (optionally controlled) op; the random-circuit workload only needs these."""
    from oracle import svoracle
    m = svoracle.base_matrix(op)
    if op.name == "CNOT":
        apply_ctrl_1q(amps, n, [op.wires[0]] + list(op.ctrls), [1] + list(op.ctrl_values or (1,) * len(op.ctrls)),
                      op.wires[1], svoracle.PAULI["X"], threads)
    elif len(op.wires) == 1 and not op.ctrls:
        apply_1q(amps, n, op.wires[0], m, threads)
    elif len(op.wires) == 1:
        apply_ctrl_1q(amps, n, op.ctrls, op.ctrl_values or (1,) * len(op.ctrls), op.wires[0], m, threads)
    else:
        raise NotImplementedError(op.name)
