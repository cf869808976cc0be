"""CPU: the runtime pass compiler (csrc/fused_jit.cpp) turns every planned pass into an sm_100a
kernel with NVRTC -- no GPU needed to check that every op case generates code that compiles.
(The kernels' results are checked on the GPU by tests/test_gpu_parity.py, which runs through them.)"""

import numpy as np

from paper_2403_02512_b200 import workloads
from paper_2403_02512_b200.device import jit_stats, plan_compile
from tests.test_planner import random_op


def _all_compiled(info):
    assert info["passes"] > 0
    assert info["compiled_passes"] == info["passes"], info


def test_compile_random_rotation_circuit():
    # shears (RX / RY types), phases, controlled X with thread / register controls
    _all_compiled(plan_compile(14, workloads.random_circuit(14, 8, seed=1)))


def test_compile_every_gate_kind():
    # PAIRG / DENSE2 / DIAGG / parity cases, controls with values, inverses, matrices
    rng = np.random.default_rng(3)
    ops = [random_op(rng, 13) for _ in range(120)]
    _all_compiled(plan_compile(13, ops))


def test_compile_qaoa_parity_phases():
    ops, _, _ = workloads.qaoa_maxcut(12, p=1, seed=0)
    _all_compiled(plan_compile(12, ops))


def test_compile_two_array_layout():
    # the adjoint sweep's psi | lambda state (top bit pinned, split pointers)
    _all_compiled(plan_compile(12, workloads.random_circuit(11, 4, seed=2), two_array=True))


def test_structure_cache_reuses_kernels():
    # new parameters, same structure: no new kernels (coefficients travel as kernel parameters; the
    # TAN/COT form of each scaled rotation is remembered per circuit structure, with hysteresis).
    # Counted as distinct kernels in the process (NVRTC runs would miss on-disk cache hits).
    a = workloads.random_circuit(12, 6, seed=5)
    plan_compile(12, a)
    k0 = jit_stats()["kernels"]
    b = [op.__class__(op.name, op.wires, tuple(p + 0.25 for p in op.params), op.ctrls, op.ctrl_values)
         for op in a]
    _all_compiled(plan_compile(12, b))
    assert jit_stats()["kernels"] == k0


def test_scaled_rotation_form_switches_only_beyond_band():
    # a large parameter change moves some rotations out of their remembered form's band: a few
    # passes get new kernels once; planning the new angles again reuses them
    a = workloads.random_circuit(12, 6, seed=7)
    plan_compile(12, a)
    k0 = jit_stats()["kernels"]
    b = [op.__class__(op.name, op.wires, tuple(p + 1.6 for p in op.params), op.ctrls, op.ctrl_values)
         for op in a]
    _all_compiled(plan_compile(12, b))
    k1 = jit_stats()["kernels"]
    assert k1 > k0
    plan_compile(12, b)
    assert jit_stats()["kernels"] == k1
