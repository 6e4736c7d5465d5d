"""GPU tier: the multi-device engine (cvg_multi, the G-device analogue of
HeteroEngine::step, hetero.cpp:252-466) against one single-device call --
bit for bit, since columns are independent -- and against the oracle, with
the reference's error semantics across ranges.  On a one-GPU box the
devices are listed repeatedly (independent contexts sharing the GPU)."""
import numpy as np
import pytest

import oracle as O
import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen as G

pytestmark = pytest.mark.gpu
FIELDS = ("tend_T", "tend_q", "precip", "work_units", "exited_early")


def same(a, b):
    for f in FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        if x.dtype == np.float64:
            assert np.array_equal(x.view(np.int64), y.view(np.int64)), f
        else:
            assert np.array_equal(x, y), f


@pytest.mark.parametrize("g", [2, 3, 8])
@pytest.mark.parametrize("cfg,kw", [("c2", {}), ("c5_50", {"shape": (96, 144)}), ("c3", {"shape": (48, 72)})])
def test_multi_union_equals_single_call(ctx, g, cfg, kw):
    s, T, q = G.make_config(cfg, seed=5, **kw)
    thr = G.config_threshold(cfg)
    o = P.KernelOptions(activity_threshold=thr)
    d1, s1 = ctx.convect(s, T, q, o)
    st1 = ctx.last_stats
    with P.MultiContext([0] * g) as m:
        d2, s2 = m.convect(s, T, q, o)
        st2 = m.last_stats
        b = m.last_bounds
    same(d1, d2)
    same(s1, s2)
    assert b[0] == 0 and b[-1] == s.size and np.all(np.diff(b) >= 0)
    assert all(x % 32 == 0 for x in b[1:-1])
    assert st2.n_triggered == st1.n_triggered
    assert st2.h2d_bytes == st1.h2d_bytes and st2.d2h_bytes == st1.d2h_bytes


def test_multi_partition_is_cost_balanced(ctx):
    """The load-imbalance stress layout (one contiguous triggered block,
    BASELINE config 5): ranges carry similar estimated cost, not similar
    column counts."""
    s, T, q = G.make_config("c5_50", shape=(96, 144), seed=3)
    with P.MultiContext([0] * 4) as m:
        m.convect(s, T, q, P.KernelOptions(), kernels=P.DEEP)
        b = m.last_bounds
    trig = np.concatenate([[0], np.cumsum(s > 0.5)])
    cost = [0.86 * (trig[b[i + 1]] - trig[b[i]]) + 0.154 * (b[i + 1] - b[i]) for i in range(4)]
    assert max(cost) / min(cost) < 1.1
    assert np.ptp(np.diff(b)) > 0.2 * s.size / 4   # not the naive equal split


def test_multi_matches_oracle_and_naive_split(ctx):
    s, T, q = G.make_config("c1", seed=9)
    with P.MultiContext([0, 0]) as m:
        m.set_weights(0.0, 1.0)   # naive equal-columns split
        d, sh = m.convect(s, T, q)
        assert abs(int(m.last_bounds[1]) - s.size // 2) <= 16
    od, osh = O.convection("deep", s, T, q), O.convection("shallow", s, T, q)
    assert np.array_equal(d.work_units, od.work) and np.array_equal(sh.work_units, osh.work)
    assert np.array_equal(d.exited_early, od.exited) and np.array_equal(sh.exited_early, osh.exited)
    assert np.allclose(d.tend_T, od.tend_T, rtol=1e-10, atol=1e-14)


def test_multi_reports_the_lowest_failing_column_across_ranges(ctx):
    """A failure in two ranges: the lowest failing column wins, deep before
    shallow (the serial driver's first throw, physics.cpp:227-245)."""
    s, T, q = G.make_config("c1", n=2048, seed=2)
    s = s.copy()
    T = T.copy()
    s[:] = 0.9
    T[5, 1900] = np.nan      # deep failure in the last range
    T[3, 700] = np.nan       # deep failure in an earlier range
    with P.MultiContext([0] * 4) as m:
        with pytest.raises(P.KernelError) as e:
            m.convect(s, T, q, kernels=P.DEEP)
    assert e.value.column == 700
    s2 = s.copy()
    s2[1500] = np.inf        # deep and shallow both fail at 1500; deep reported
    with P.MultiContext([0] * 4) as m:
        with pytest.raises(P.KernelError) as e:
            m.convect(s2, T, q)
        assert m.last_stats.failing_kernel == P.DEEP
    assert e.value.column == 700


def test_multi_rejects_device_buffers_and_bad_args():
    import ctypes as C
    lib = P.load_library()
    h = C.c_void_p()
    assert lib.cvg_multi_create((C.c_int * 1)(0), 0, C.byref(h)) == 1
    assert lib.cvg_multi_convect(None, None, None, 3, None, None, None, None) == 1
    assert b"null" in lib.cvg_last_error()
