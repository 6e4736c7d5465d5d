"""CPU tier: the C ABI library loads, exports every symbol include/convgpu.h
declares, follows the reference C API conventions (capi.cpp:39-89) without
a GPU, and its host-side partition planner is correct."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1711_00289_b200 as P

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "convgpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cvg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = P.load_library()
    names = declared_functions()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_defaults():
    lib = P.load_library()
    assert lib.cvg_version().decode().count(".") == 2
    o = P.KernelOptions()
    o.variant, o.activity_threshold = 7, 9.0
    lib.cvg_default_options(C.byref(o))
    assert (o.variant, o.activity_threshold, o.newton_tol, o.newton_max_iter) == (0, 0.5, 1e-12, 100)


def test_null_arguments_are_invalid():
    lib = P.load_library()
    assert lib.cvg_context_create(0, None) == 1
    assert b"null" in lib.cvg_last_error()
    assert lib.cvg_convect(None, None, None, 3, None, None, None) == 1
    assert b"null" in lib.cvg_last_error()
    lib.cvg_context_free(None)  # no-op


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.DeviceError):
        P.Context(0)
    # a successful call clears the thread-local message (capi.cpp:54)
    b = np.empty(3, dtype=np.int64)
    P.load_library().cvg_plan_partition(0, None, 0.5, 2, 0.0, 1.0, b.ctypes.data)
    assert P.load_library().cvg_last_error() == b""


def test_naive_partition_puts_remainder_last():
    # StaticBlock semantics, sched.cpp:66-75
    b = P.plan_partition(np.zeros(10), 0.5, 4, 0.0, 1.0)
    assert list(b) == [0, 2, 4, 7, 10]
    assert list(P.plan_partition(np.zeros(0), 0.5, 3, 0.0, 1.0)) == [0, 0, 0, 0]


@pytest.mark.parametrize("frac", [0.05, 0.5, 0.95])
@pytest.mark.parametrize("parts", [2, 4, 8])
def test_balanced_partition_equalises_cost(frac, parts):
    n = 100_000
    s = np.zeros(n)
    a = int(frac * n)
    lo = (n - a) // 2
    s[lo:lo + a] = 0.9  # one contiguous triggered block (config C5)
    dw, sw = 30000.0, 7750.0
    b = P.plan_partition(s, 0.5, parts, dw, sw)
    assert b[0] == 0 and b[-1] == n and (np.diff(b) >= 0).all()
    cost = np.where(s > 0.5, dw, 0.0) + sw
    per = np.array([cost[b[i]:b[i + 1]].sum() for i in range(parts)])
    assert per.max() - per.min() <= 2 * (dw + sw)
    naive = P.plan_partition(s, 0.5, parts, 0.0, 1.0)
    pn = np.array([cost[naive[i]:naive[i + 1]].sum() for i in range(parts)])
    assert per.max() <= pn.max() + 1e-6


def test_partition_rejects_bad_arguments():
    b = np.empty(3, dtype=np.int64)
    lib = P.load_library()
    assert lib.cvg_plan_partition(-1, None, 0.5, 2, 0.0, 1.0, b.ctypes.data) == 1
    assert lib.cvg_plan_partition(5, None, 0.5, 0, 0.0, 1.0, b.ctypes.data) == 1


def test_partition_bounds_are_aligned_and_monotone():
    from paper_1711_00289_b200 import gridgen, multigpu
    s, _, _ = gridgen.make_config("c5_50", shape=(48, 64), seed=4)
    for world in (1, 2, 3, 8):
        for mode in ("balanced", "overlap", "model", "naive"):
            b = multigpu.rank_bounds(s, 0.5, world, mode)
            assert b[0] == 0 and b[-1] == s.size and len(b) == world + 1
            assert np.all(np.diff(b) >= 0)
            assert np.all(b[1:-1] % multigpu.ALIGN == 0)
    # rounding moves a boundary by at most ALIGN / 2
    raw = P.plan_partition(s, 0.5, 8, *multigpu.partition_weights())
    assert np.max(np.abs(multigpu.align_bounds(raw) - raw)) <= multigpu.ALIGN // 2


def test_overlap_partition_minimises_the_largest_share():
    """overlap_bounds: no share's modelled cost exceeds the linear split's
    worst share (the bisection minimises the maximum)."""
    from paper_1711_00289_b200 import gridgen, multigpu
    s, _, _ = gridgen.make_config("c5_50", shape=(48, 64), seed=4)
    cost = lambda b: max(multigpu.share_cost(int((s[b[i]:b[i + 1]] > 0.5).sum()), b[i + 1] - b[i])
                         for i in range(len(b) - 1))
    for world in (2, 4):
        ov = multigpu.overlap_bounds(s, 0.5, world)
        lin = P.plan_partition(s, 0.5, world, *multigpu.partition_weights())
        assert ov[0] == 0 and ov[-1] == s.size and np.all(np.diff(ov) >= 0)
        assert cost(ov) <= cost(lin) + 1e-12


def test_multi_engine_conventions_without_device():
    """cvg_multi: null/size checks, and no CPU fallback without a device."""
    lib = P.load_library()
    h = C.c_void_p()
    assert lib.cvg_multi_create(None, 1, C.byref(h)) == 1
    assert b"null" in lib.cvg_last_error()
    assert lib.cvg_multi_create((C.c_int * 2)(0, 0), 0, C.byref(h)) == 1
    assert lib.cvg_multi_size(None) == 0
    assert lib.cvg_multi_context(None, 0) is None
    assert lib.cvg_multi_set_weights(None, 1.0, 1.0) == 1
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(P.DeviceError):
            P.MultiContext([0, 0])
