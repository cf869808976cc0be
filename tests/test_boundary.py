"""CPU: the C-ABI library builds, loads, exports every symbol of include/svb200.h, and its
host-side logic (validation -> error classes, op lowering / fusion planning) works without a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2403_02512_b200 import _lib, errors, workloads
from paper_2403_02512_b200.device import plan_summary
from paper_2403_02512_b200.ops import GATE_KINDS, Op

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2403_02512_b200 import build
    build.build()
    return _lib.lib()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "svb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_kind_enum_matches_header():
    text = open(os.path.join(ROOT, "include", "svb200.h")).read()
    body = re.search(r"enum sv_gate_kind \{(.*?)\};", text, re.S).group(1)
    names = re.findall(r"SV_GATE_([A-Z_]+)", body)
    assert len(names) == len(GATE_KINDS) + 1          # + SV_GATE_COUNT
    norm = [k.upper().replace("EXCITATION", "_EXCITATION").replace("CONTROLLEDMATRIX", "CONTROLLED_MATRIX")
            for k in GATE_KINDS]
    assert names[:-1] == norm


def test_device_count_without_gpu_is_zero_or_more(lib):
    assert _lib.device_count() >= 0


def test_status_maps_to_reference_classes(lib):
    ops = [Op("RX", (5,), (0.1,))]                    # wire out of range
    with pytest.raises(errors.ValidationError, match="out of range"):
        plan_summary(3, ops)
    with pytest.raises(errors.ValidationError, match="duplicate wires"):
        plan_summary(3, [Op("CNOT", (1, 1))])
    with pytest.raises(errors.ValidationError, match="overlaps controls"):
        plan_summary(3, [Op("RX", (1,), (0.1,), ctrls=(1,))])
    with pytest.raises(errors.ValidationError):
        plan_summary(0, [])
    assert issubclass(errors.ValidationError, ValueError)
    assert issubclass(errors.CapacityError, errors.SvkitError)


def test_unsupported_trainable_kind(lib):
    op = Op("H", (0,))
    op.trainable = (True,)        # forged flag on a parameterless gate
    with pytest.raises(errors.UnsupportedOperationError):
        plan_summary(2, [op])


def test_plan_summary_counts_ops(lib):
    ops = workloads.random_circuit(12, 6, seed=3)
    s = plan_summary(12, ops)
    assert s["ops"] == len(ops)
    assert 1 <= s["passes"] <= s["ops"]


def test_op_and_observable_packing():
    ops = [Op("Rot", (0,), (0.1, 0.2, 0.3), trainable=(True, False, True)),
           Op("CNOT", (0, 1), ctrls=(2,), ctrl_values="0"),
           Op("Matrix", (1, 2), matrix=np.eye(4))]
    p = _lib.PackedOps(ops)
    assert p.n == 3
    assert p.arr[0].trainable_mask == 0b101
    assert p.arr[1].n_ctrls == 1 and p.arr[1].ctrl_values[0] == 0
    assert p.arr[2].matrix[0] == 1.0 and p.arr[2].matrix[1] == 0.0
    from paper_2403_02512_b200.observables import Hamiltonian, PauliWord
    o = _lib.PackedObs([Hamiltonian([0.5, -1.0], [PauliWord(((0, "X"), (2, "Y"))), PauliWord(())])])
    assert o.arr[0].type == 1 and o.arr[0].n_terms == 2
    assert o.arr[0].term_paulis == b"XY"


def test_ctypes_signatures_cover_exports(lib):
    for s in _lib.EXPORTS:
        f = getattr(lib, s)
        assert isinstance(f, ctypes._CFuncPtr)


def test_memory_plan_of_the_north_star_configs():
    """33q adjoint needs 2 GPUs (psi + lambda = 275 GB); 34q fits 4, 35q fits 8 with
    psi + lambda = 137.4 GB per GPU (document and assert the 35q / P=8 plan)."""
    from paper_2403_02512_b200.device import memory_plan
    assert memory_plan(30)["state_bytes"] == 16 * 2**30
    assert not memory_plan(33, 1)["fits_b200"] and memory_plan(33, 2)["fits_b200"]
    p35 = memory_plan(35, 8)
    assert p35["state_bytes"] + p35["adjoint_bytes"] == 2 * 16 * 2**32   # 137.4 GB
    assert p35["fits_b200"] and memory_plan(34, 4)["fits_b200"]
    assert not memory_plan(35, 4)["fits_b200"]                          # 35q adjoint needs 8 GPUs
    assert memory_plan(35, 4, n_observables=0)["state_bytes"] < 179e9   # the 35q forward fits 4
