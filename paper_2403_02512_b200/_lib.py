"""ctypes binding of libsvb200.so (include/svb200.h).

The library is the product: if it is missing this module raises at load time -- there is
no CPU fallback. Build it with ``python -m paper_2403_02512_b200.build``.
"""

import ctypes
import os
from ctypes import POINTER, c_char, c_char_p, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

from .errors import raise_for_status
from .observables import DenseHermitian, Hamiltonian, PauliWord, SparseHermitian, as_observable
from .ops import KIND_CODE, Op

# SVB200_LIB selects another in-tree build of the same library (A/B kernel experiments)
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("SVB200_LIB", "libsvb200.so"))

# Every symbol include/svb200.h declares (checked by tests/test_boundary.py).
EXPORTS = (
    "sv_device_count", "sv_create", "sv_nccl_unique_id", "sv_create_sharded", "sv_destroy", "sv_info",
    "sv_reset", "sv_set_basis_state", "sv_set_state", "sv_get_state", "sv_norm",
    "sv_apply_single_qubit", "sv_apply_controlled_single_qubit", "sv_apply_matrix", "sv_apply_ops",
    "sv_expval", "sv_probs", "sv_var", "sv_sample", "sv_adjoint_jacobian", "sv_last_error", "sv_synchronize", "sv_stream",
    "sv_launch_count", "sv_set_profiling", "sv_kernel_stats", "sv_reset_stats", "sv_plan_summary",
    "sv_plan_program", "sv_plan_sharded", "sv_plan_compile", "sv_plan_fp64", "sv_jit_stats",
    "sv_create_ex", "sv_set_state_c64", "sv_get_state_c64",
)


class SvOp(ctypes.Structure):
    _fields_ = [
        ("kind", c_int32), ("n_wires", c_int32), ("wires", POINTER(c_int32)),
        ("n_ctrls", c_int32), ("ctrls", POINTER(c_int32)), ("ctrl_values", POINTER(c_int32)),
        ("params", c_double * 3), ("inverse", c_int32), ("trainable_mask", c_int32),
        ("matrix", POINTER(c_double)),
    ]


class SvObs(ctypes.Structure):
    _fields_ = [
        ("type", c_int32), ("n_terms", c_int32), ("coeffs", POINTER(c_double)),
        ("term_len", POINTER(c_int32)), ("term_wires", POINTER(c_int32)), ("term_paulis", c_char_p),
        ("n_wires", c_int32), ("wires", POINTER(c_int32)), ("matrix", POINTER(c_double)),
        ("csr_dim", ctypes.c_int64), ("csr_nnz", ctypes.c_int64), ("csr_indptr", POINTER(ctypes.c_int64)),
        ("csr_indices", POINTER(ctypes.c_int64)), ("csr_data", POINTER(c_double)),
    ]


_lib = None


def lib():
    """Load libsvb200.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2403_02512_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        H = c_void_p
        sig = {
            "sv_device_count": [POINTER(c_int)],
            "sv_create": [c_int, c_int, POINTER(H)],
            "sv_create_ex": [c_int, c_int, c_int, POINTER(H)],
            "sv_set_state_c64": [H, POINTER(ctypes.c_float), c_uint64],
            "sv_get_state_c64": [H, POINTER(ctypes.c_float), c_uint64],
            "sv_nccl_unique_id": [c_void_p],
            "sv_create_sharded": [c_int, c_int, c_int, c_int, c_void_p, POINTER(H)],
            "sv_destroy": [H],
            "sv_info": [H, POINTER(c_int64)],
            "sv_reset": [H],
            "sv_set_basis_state": [H, c_uint64],
            "sv_set_state": [H, POINTER(c_double), c_uint64],
            "sv_get_state": [H, POINTER(c_double), c_uint64],
            "sv_norm": [H, POINTER(c_double)],
            "sv_apply_single_qubit": [H, c_int, POINTER(c_double)],
            "sv_apply_controlled_single_qubit": [H, POINTER(c_int32), c_int, c_int, POINTER(c_double), POINTER(c_int32)],
            "sv_apply_matrix": [H, POINTER(c_int32), c_int, POINTER(c_double)],
            "sv_apply_ops": [H, POINTER(SvOp), c_int, c_int],
            "sv_expval": [H, POINTER(SvObs), POINTER(c_double)],
            "sv_probs": [H, POINTER(c_int32), c_int, POINTER(c_double)],
            "sv_var": [H, POINTER(SvObs), POINTER(c_double)],
            "sv_sample": [H, POINTER(c_int32), c_int, ctypes.c_uint64, ctypes.c_uint64, POINTER(ctypes.c_int64)],
            "sv_adjoint_jacobian": [H, POINTER(SvOp), c_int, POINTER(SvObs), c_int, c_int, POINTER(c_double),
                                    POINTER(c_double)],
            "sv_synchronize": [H],
            "sv_set_profiling": [H, c_int],
            "sv_kernel_stats": [H, POINTER(c_double), c_int, POINTER(c_int), POINTER(c_char), c_int],
            "sv_reset_stats": [H],
            "sv_plan_summary": [c_int, POINTER(SvOp), c_int, POINTER(c_int64)],
            "sv_plan_program": [c_int, POINTER(SvOp), c_int, POINTER(c_int64), c_int64, POINTER(c_double), c_int64,
                                POINTER(c_int64)],
            "sv_plan_sharded": [c_int, c_int, c_int, POINTER(SvOp), c_int, POINTER(c_int64), c_int64,
                                POINTER(c_double), c_int64, POINTER(c_int64)],
            "sv_plan_compile": [c_int, POINTER(SvOp), c_int, c_int, POINTER(c_int64)],
            "sv_jit_stats": [POINTER(c_int64)],
            "sv_plan_fp64": [c_int, POINTER(SvOp), c_int, POINTER(c_double)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = c_int
        L.sv_last_error.argtypes = []
        L.sv_last_error.restype = c_char_p
        L.sv_stream.argtypes = [H]
        L.sv_stream.restype = c_void_p
        L.sv_launch_count.argtypes = [H]
        L.sv_launch_count.restype = c_int64
        _lib = L
    return _lib


def check(status):
    if status != 0:
        raise_for_status(status, lib().sv_last_error().decode(errors="replace"))


def device_count():
    n = c_int(0)
    check(lib().sv_device_count(ctypes.byref(n)))
    return n.value


def _iptr(a):
    return a.ctypes.data_as(POINTER(c_int32))


def _dptr(a):
    return a.ctypes.data_as(POINTER(c_double))


def _svop_dtype():
    f = SvOp
    names = ["kind", "n_wires", "wires", "n_ctrls", "ctrls", "ctrl_values", "params", "inverse", "trainable_mask",
             "matrix"]
    formats = [np.int32, np.int32, np.uint64, np.int32, np.uint64, np.uint64, (np.float64, 3), np.int32, np.int32,
               np.uint64]
    return np.dtype({"names": names, "formats": formats, "offsets": [getattr(f, k).offset for k in names],
                     "itemsize": ctypes.sizeof(SvOp)})


_SVOP_DTYPE = None


class PackedOps:
    """Op records marshalled into C structs; owns every buffer the structs point to.

    Vectorised: one numpy record array laid out as `sv_op` (include/svb200.h) plus one int32
    buffer holding every op's wires, controls and control values (the structs point into it),
    so marshalling a 2225-op circuit costs ~1 ms instead of ~8 ms of per-field ctypes writes.
    """

    def __init__(self, ops):
        global _SVOP_DTYPE
        if _SVOP_DTYPE is None:
            _SVOP_DTYPE = _svop_dtype()
        ops = list(ops)
        for op in ops:
            if not isinstance(op, Op):
                raise TypeError(f"expected Op, got {type(op).__name__}")
        self.n = n = len(ops)
        rec = np.zeros(max(n, 1), dtype=_SVOP_DTYPE)
        ints, starts = [], []
        for op in ops:
            starts.append(len(ints))
            ints.extend(op.wires)
            ints.extend(op.ctrls)
            ints.extend(op.ctrl_values)
        buf = np.asarray(ints if ints else [0], dtype=np.int32)
        base = buf.ctypes.data
        self._keep = [rec, buf]
        if n:
            rec["kind"][:n] = [KIND_CODE[op.name] for op in ops]
            nw = np.fromiter((len(op.wires) for op in ops), np.int64, n)
            nc = np.fromiter((len(op.ctrls) for op in ops), np.int64, n)
            st = np.asarray(starts, dtype=np.int64)
            rec["n_wires"][:n] = nw
            rec["wires"][:n] = (base + 4 * st).astype(np.uint64)
            rec["n_ctrls"][:n] = nc
            has_c = nc > 0
            rec["ctrls"][:n] = np.where(has_c, base + 4 * (st + nw), 0).astype(np.uint64)
            rec["ctrl_values"][:n] = np.where(has_c, base + 4 * (st + nw + nc), 0).astype(np.uint64)
            params = np.zeros((n, 3))
            for i, op in enumerate(ops):
                if op.params:
                    p = op.params[:3]
                    params[i, :len(p)] = p
            rec["params"][:n] = params
            rec["inverse"][:n] = [1 if op.inverse else 0 for op in ops]
            rec["trainable_mask"][:n] = [sum(1 << j for j, t in enumerate(op.trainable) if t) if op.trainable else 0
                                         for op in ops]
            for i, op in enumerate(ops):
                if op.matrix is not None:
                    m = np.ascontiguousarray(op.matrix, dtype=np.complex128).view(np.float64)
                    rec["matrix"][i] = m.ctypes.data
                    self._keep.append(m)
        self.arr = (SvOp * max(n, 1)).from_buffer(rec)

    @property
    def ptr(self):
        return self.arr


class PackedObs:
    """Observable records marshalled into C structs."""

    def __init__(self, observables):
        obs = [as_observable(o) for o in observables]
        self.n = len(obs)
        self.arr = (SvObs * max(self.n, 1))()
        self._keep = []
        for i, o in enumerate(obs):
            rec = self.arr[i]
            if isinstance(o, SparseHermitian):
                rec.type = 3
                ip, ix = o.indptr, o.indices
                dv = o.data.view(np.float64)
                rec.csr_dim, rec.csr_nnz = o.dim, len(ix)
                rec.csr_indptr = ip.ctypes.data_as(POINTER(ctypes.c_int64))
                rec.csr_indices = ix.ctypes.data_as(POINTER(ctypes.c_int64))
                rec.csr_data = _dptr(dv)
                self._keep += [ip, ix, dv]
                continue
            if isinstance(o, DenseHermitian):
                rec.type = 2
                w = np.ascontiguousarray(o.wires, dtype=np.int32)
                m = np.ascontiguousarray(o.matrix, dtype=np.complex128).view(np.float64)
                rec.n_wires = len(w)
                rec.wires = _iptr(w)
                rec.matrix = _dptr(m)
                self._keep += [w, m]
                continue
            if isinstance(o, PauliWord):
                rec.type = 0
                terms, coeffs = [o], None
            elif isinstance(o, Hamiltonian):
                rec.type = 1
                terms = list(o.terms)
                coeffs = np.ascontiguousarray(o.coeffs, dtype=np.float64)
            else:
                raise TypeError(f"unsupported observable {type(o).__name__}")
            lens = np.array([len(t.factors) for t in terms], dtype=np.int32)
            wires = np.array([w for t in terms for w, _ in t.factors], dtype=np.int32)
            paulis = "".join(p for t in terms for _, p in t.factors).encode() + b"\0"
            rec.n_terms = len(terms)
            rec.term_len = _iptr(lens)
            rec.term_wires = _iptr(wires)
            rec.term_paulis = paulis
            self._keep += [lens, wires, paulis]
            if coeffs is not None:
                rec.coeffs = _dptr(coeffs)
                self._keep.append(coeffs)

    @property
    def ptr(self):
        return self.arr
