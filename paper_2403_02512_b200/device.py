"""``Device``: the py-bindings device handle of the reference on a B200.

``bind_device(n_qubits, precision, tier)`` returns a handle that owns a complex128 ("f64") or
complex64 ("f32", single GPU, one kernel per op) state in HBM; ``apply`` / ``expval`` / ``var`` / ``probs`` / ``sample`` / ``adjoint_jacobian`` forward 1:1 to the C-ABI
(include/svb200.h) with copy-out marshalling. One mutator per handle
 is enforced by a per-handle mutex inside the library.
"""

import ctypes
from ctypes import byref, c_double, c_int64, c_void_p

import numpy as np

from . import _lib
from .errors import UnsupportedOperationError, ValidationError
from .observables import as_observable
from .ops import Op


class Device:
    """Handle to a state vector on one GPU, or one shard of a state sharded over NCCL ranks."""

    def __init__(self, n_qubits, precision="f64", device=0, fuse=True, _sharded=None):
        if precision not in ("f64", "f32"):
            raise ValidationError(f"unknown precision {precision!r}; expected 'f64' or 'f32'")
        if precision == "f32" and _sharded is not None:
            raise UnsupportedOperationError("complex64 (f32) states are single-GPU only; shard a complex128 state")
        if not isinstance(n_qubits, (int, np.integer)):
            raise ValidationError(f"n_qubits must be a positive integer, got {n_qubits!r}")
        L = _lib.lib()
        self._h = c_void_p()
        self.fuse = bool(fuse)
        if _sharded is None:
            bits = 64 if precision == "f64" else 32
            _lib.check(L.sv_create_ex(int(n_qubits), int(device), bits, byref(self._h)))
        else:
            rank, world, nccl_id = _sharded
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            _lib.check(L.sv_create_sharded(int(n_qubits), int(rank), int(world), int(device), buf, byref(self._h)))
        info = (c_int64 * 6)()
        _lib.check(L.sv_info(self._h, info))
        self.n_qubits, self.n_local, self.rank, self.world, self.device = (int(info[i]) for i in range(5))
        self.precision = precision
        self.dtype = np.complex128 if precision == "f64" else np.complex64

    # ---- lifecycle ---------------------------------------------------------------------
    @classmethod
    def sharded(cls, n_qubits, rank, world, nccl_id, device=None, fuse=True):
        """One shard of an n-qubit state over ``world`` ranks."""
        return cls(n_qubits, device=rank if device is None else device, fuse=fuse, _sharded=(rank, world, nccl_id))

    @staticmethod
    def nccl_unique_id():
        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.lib().sv_nccl_unique_id(buf))
        return buf.raw

    def release(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.check(_lib.lib().sv_destroy(self._h))
            self._h = c_void_p()

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.release()

    @property
    def handle(self):
        if not self._h.value:
            raise ValidationError("device handle used after release")
        return self._h

    # ---- state I/O ---------------------------------------------------------------------
    def reset(self):
        _lib.check(_lib.lib().sv_reset(self.handle))

    def set_basis_state(self, index):
        _lib.check(_lib.lib().sv_set_basis_state(self.handle, int(index)))

    def set_state(self, amplitudes):
        a = np.ascontiguousarray(amplitudes, dtype=self.dtype)
        if a.ndim != 1:
            raise ValidationError("amplitude array must be 1-D")
        if self.precision == "f32":
            _lib.check(_lib.lib().sv_set_state_c64(
                self.handle, a.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float)), a.size))
            return
        _lib.check(_lib.lib().sv_set_state(self.handle, a.view(np.float64).ctypes.data_as(ctypes.POINTER(c_double)),
                                           a.size))

    def get_state(self):
        out = np.empty(1 << self.n_qubits, dtype=self.dtype)
        if self.precision == "f32":
            _lib.check(_lib.lib().sv_get_state_c64(
                self.handle, out.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float)), out.size))
            return out
        _lib.check(_lib.lib().sv_get_state(self.handle, out.view(np.float64).ctypes.data_as(ctypes.POINTER(c_double)),
                                           out.size))
        return out

    def norm(self):
        v = c_double()
        _lib.check(_lib.lib().sv_norm(self.handle, byref(v)))
        return v.value

    # ---- gates -------------------------------------------------------------------------
    def apply(self, ops, fuse=None):
        """Apply an op list (or a circuit_ir.Circuit) in order (Device.apply)."""
        ops = getattr(ops, "ops", ops)
        ops = [o if isinstance(o, Op) else Op(*o) for o in ops]
        packed = _lib.PackedOps(ops)
        f = self.fuse if fuse is None else fuse
        _lib.check(_lib.lib().sv_apply_ops(self.handle, packed.ptr, packed.n, int(bool(f))))

    def apply_matrix(self, wires, matrix):
        wires = np.ascontiguousarray(wires, dtype=np.int32)
        m = np.ascontiguousarray(matrix, dtype=np.complex128)
        if m.shape != (1 << len(wires),) * 2:
            raise ValidationError(f"matrix shape {m.shape} does not match {len(wires)} wires")
        _lib.check(_lib.lib().sv_apply_matrix(self.handle, wires.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                              len(wires), m.view(np.float64).ctypes.data_as(ctypes.POINTER(c_double))))

    # ---- measurements ------------------------------------------------------------------
    def expval(self, obs):
        packed = _lib.PackedObs([as_observable(obs)])
        v = c_double()
        _lib.check(_lib.lib().sv_expval(self.handle, packed.ptr, byref(v)))
        return v.value

    def expvals(self, observables):
        return np.array([self.expval(o) for o in observables])

    def probs(self, wires=None):
        if wires is None:
            w = np.zeros(0, dtype=np.int32)
            size = 1 << self.n_qubits
        else:
            w = np.ascontiguousarray(wires, dtype=np.int32)
            size = 1 << len(w)
        out = np.empty(size, dtype=np.float64)
        _lib.check(_lib.lib().sv_probs(self.handle, w.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(w),
                                       out.ctypes.data_as(ctypes.POINTER(c_double))))
        return out

    def var(self, obs):
        """Variance <O^2> - <O>^2."""
        pb = _lib.PackedObs([as_observable(obs)])
        v = c_double()
        _lib.check(_lib.lib().sv_var(self.handle, pb.ptr, ctypes.byref(v)))
        return v.value

    def sample_indices(self, shots, seed=0, wires=None):
        """``shots`` outcome indices over ``wires`` (all if None; wires[0] = MSB), deterministic
        per seed; the draw procedure is documented at sv_sample in include/svb200.h."""
        w = np.zeros(0, dtype=np.int32) if wires is None else np.ascontiguousarray(wires, dtype=np.int32)
        out = np.empty(int(shots), dtype=np.int64)
        _lib.check(_lib.lib().sv_sample(self.handle, w.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(w),
                                        int(shots), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out

    def sample(self, shots, seed=0, wires=None):
        """SampleSet: ``shots`` rows of 0/1 bits, one column per measured wire."""
        width = self.n_qubits if wires is None else len(wires)
        idx = self.sample_indices(shots, seed, wires)
        return ((idx[:, None] >> np.arange(width - 1, -1, -1)) & 1).astype(np.int8)

    # ---- adjoint Jacobian ----------------------------------------------------------------
    def adjoint_jacobian(self, ops, observables, return_expvals=False, fuse=None):
        """n_obs x n_trainable Jacobian of <O_k> by one forward pass + reverse sweep.

        Starts from the handle's current state; on return the handle holds the state swept back
        to the input (fp64 round-off).
        """
        ops = [o if isinstance(o, Op) else Op(*o) for o in getattr(ops, "ops", ops)]
        obs = [as_observable(o) for o in observables]
        ncols = sum(op.n_trainable for op in ops)
        po, pb = _lib.PackedOps(ops), _lib.PackedObs(obs)
        jac = np.zeros((len(obs), ncols), dtype=np.float64)
        ev = np.zeros(len(obs), dtype=np.float64)
        f = self.fuse if fuse is None else fuse
        _lib.check(_lib.lib().sv_adjoint_jacobian(self.handle, po.ptr, po.n, pb.ptr, pb.n, int(bool(f)),
                                                  jac.ctypes.data_as(ctypes.POINTER(c_double)),
                                                  ev.ctypes.data_as(ctypes.POINTER(c_double))))
        return (jac, ev) if return_expvals else jac

    # ---- diagnostics -------------------------------------------------------------------
    def synchronize(self):
        _lib.check(_lib.lib().sv_synchronize(self.handle))

    @property
    def stream(self):
        return _lib.lib().sv_stream(self.handle)

    @property
    def launch_count(self):
        return int(_lib.lib().sv_launch_count(self.handle))

    def set_profiling(self, enabled=True):
        _lib.check(_lib.lib().sv_set_profiling(self.handle, int(bool(enabled))))

    def kernel_stats(self):
        out = (c_double * 64)()
        n = ctypes.c_int()
        names = ctypes.create_string_buffer(512)
        _lib.check(_lib.lib().sv_kernel_stats(self.handle, out, 20, byref(n), names, 512))
        keys = names.value.decode().split(",")
        return {keys[k]: {"launches": out[3 * k], "ms": out[3 * k + 1], "bytes": out[3 * k + 2]}
                for k in range(n.value)}

    def reset_stats(self):
        _lib.check(_lib.lib().sv_reset_stats(self.handle))


def bind_device(n_qubits, precision="f64", tier=None, device=0, fuse=True):
    """Reference-named constructor. ``tier`` is accepted for API parity;
    the GPU path has exactly one tier."""
    if tier not in (None, "cuda", "sm_100a"):
        raise ValidationError(f"unknown tier {tier!r}; the B200 build has the single tier 'sm_100a'")
    return Device(n_qubits, precision=precision, device=device, fuse=fuse)


def plan_summary(n_qubits, ops):
    """Host-only fusion plan summary {passes, ops, tile_bits, phases} (no GPU needed)."""
    packed = _lib.PackedOps(ops)
    out = (c_int64 * 4)()
    _lib.check(_lib.lib().sv_plan_summary(int(n_qubits), packed.ptr, packed.n, out))
    return {"passes": out[0], "ops": out[1], "tile_bits": out[2], "phases": out[3]}


def plan_compile(n_qubits, ops, two_array=False):
    """Host-only: plan the op list and compile every fused pass into its own sm_100a kernel with
    the runtime pass compiler (NVRTC; no GPU needed).  Returns {passes, compiled_passes,
    kernels_compiled_total, compile_s_total} (the last two are process-wide counters)."""
    packed = _lib.PackedOps(ops)
    out = (c_int64 * 4)()
    _lib.check(_lib.lib().sv_plan_compile(int(n_qubits), packed.ptr, packed.n, int(bool(two_array)), out))
    return {"passes": out[0], "compiled_passes": out[1], "kernels_compiled_total": out[2],
            "compile_s_total": out[3] * 1e-6}


def jit_stats():
    """Process-wide pass-compiler counters: {compiled, compile_s, kernels} (NVRTC runs; disk-cache
    hits are not compiles)."""
    out = (c_int64 * 3)()
    _lib.check(_lib.lib().sv_jit_stats(out))
    return {"compiled": int(out[0]), "compile_s": out[1] * 1e-6, "kernels": int(out[2])}


def plan_fp64_flops_per_amp(n_qubits, ops):
    """Host-only: FP64 flops per amplitude the fused program of this op list performs."""
    packed = _lib.PackedOps(ops)
    out = ctypes.c_double()
    _lib.check(_lib.lib().sv_plan_fp64(int(n_qubits), packed.ptr, packed.n, ctypes.byref(out)))
    return out.value


B200_HBM_BYTES = 179 * 10**9   # usable HBM3e per B200 (cudaMemGetInfo total on this pool's boxes, ~179 GB)


def memory_plan(n_qubits, world=1, n_observables=1, fused=True, precision="f64"):
    """Per-GPU device memory of a state-vector job (the buffers libsvb200 allocates): the shard, the
    adjoint sweep's lambda (one kept buffer for the fused sweep, plus one saved final state when
    several observables share the forward pass; the per-gate sweep keeps one lambda per
    observable), and the sharded swap staging (two slots of up to 1 GiB each).  Returns a dict of
    byte counts and whether it fits one B200 (SPEC.md:643 capacity errors surface as
    CapacityError at run time; this is the plan the north star's 35-qubit / 8-GPU adjoint rests on)."""
    amp = 16 if precision == "f64" else 8
    g = world.bit_length() - 1
    if world < 1 or (world & (world - 1)):
        raise ValidationError("n_shards must be a power of two")
    shard = amp * (1 << (n_qubits - g))
    if fused:
        lam = shard * (1 + (1 if n_observables > 1 else 0))
    else:
        lam = shard * n_observables
    staging = 0 if world == 1 else min(2 * 2**30, 16 * (1 << (n_qubits - g - 1)))
    total = shard + lam + staging
    return {"n_qubits": n_qubits, "world": world, "state_bytes": shard, "adjoint_bytes": lam,
            "staging_bytes": staging, "total_bytes": total, "fits_b200": total < B200_HBM_BYTES}
