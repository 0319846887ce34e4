"""CPU-only checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/lancelot_b200.h declares, there is no CPU
fallback, and the host-side planning logic matches the reference's own unit
tests (test_distance.cpp)."""
import ctypes
import math
import os

import pytest

import paper_2408_06197_b200.lancelot as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(L.LIB_PATH)
    names = L.exported_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python mirror binds every one of them
    bound = L.lib()
    for n in names:
        assert hasattr(bound, n)


def test_cpp_mirror_header_names_match_reference_api():
    with open(os.path.join(ROOT, "include", "lancelot_b200.hpp")) as f:
        hpp = f.read()
    for sym in ("build_distance_matrix", "masked_aggregate", "slot_reduce_steps", "HoistPlan",
                "WidthError", "KeyError", "ShapeError", "DepthExhaustedError"):
        assert sym in hpp


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(L.DeviceError):
        L.CkksContext(L.CkksParams(ring_degree=1024, security=L.SecurityLevel.none))


def test_chunk_counts():  # test_distance.cpp:69-76
    assert L.chunk_count_for(1, 128) == 1
    assert L.chunk_count_for(128, 128) == 1
    assert L.chunk_count_for(129, 128) == 2
    assert L.chunk_count_for(61706, 4096) == 16
    with pytest.raises(L.ShapeError):
        L.chunk_count_for(0, 128)
    with pytest.raises(L.ShapeError):
        L.chunk_count_for(4, 0)


def test_prescale_trigger():  # test_distance.cpp:78-85
    assert L.distance_prescale(61706, math.ldexp(1.0, 20)) == 1.0
    assert L.distance_prescale(1 << 22, math.ldexp(1.0, 20)) == 1.0
    big = 1 << 23
    assert L.distance_prescale(big, math.ldexp(1.0, 20)) == pytest.approx(1 / math.sqrt(big))


def test_unfold_planning():  # test_distance.cpp:189-205
    assert L.plan_unfold(2.0, 1.0, 1.0, 4.0, 16).k == 4
    assert L.plan_unfold(1.0, 1.0, 1.0, 100.0, 16).k == 1
    assert L.plan_unfold(5.0, 1.0, 1.0, 2.0, 16).k == 2
    with pytest.raises(L.InfeasibleError):
        L.plan_unfold(1.0, 1.0, 4.0, 2.0, 16)
    with pytest.raises(L.WidthError):
        L.plan_unfold(1.0, 1.0, 1.0, 2.0, 12)
    with pytest.raises(L.ParameterError):
        L.plan_unfold(0.0, 1.0, 1.0, 2.0, 16)


def test_fixed_plans_and_steps():
    assert L.fixed_plan(L.HoistMode.off, 16).k == 1
    assert L.fixed_plan(L.HoistMode.full, 16).k == 5
    with pytest.raises(L.UsageError):
        L.fixed_plan(L.HoistMode.dynamic_lp, 16)
    assert L.slot_reduce_steps(16, 1) == [1, 2, 4, 8]
    assert L.slot_reduce_steps(16, 3) == [1, 2, 3, 4, 8]
    assert L.slot_reduce_steps(16, 5) == list(range(1, 16))
    assert L.slot_reduce_steps(1, 1) == []
    with pytest.raises(L.ParameterError):
        L.slot_reduce_steps(16, 0)
    with pytest.raises(L.WidthError):
        L.slot_reduce_steps(12, 1)


def test_params_validation():
    with pytest.raises(L.ParameterError):
        L.CkksParams(ring_degree=1000).validate()
    with pytest.raises(L.ParameterError):
        L.CkksParams(scale_bits=30).validate()
