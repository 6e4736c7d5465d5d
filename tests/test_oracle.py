"""CPU tier: the parity oracle is pinned before it is trusted.

* bit-exact against the golden fixtures the reference itself produced
  (tests/golden/make_golden.py);
* bit-exact against the reference compiled from /root/reference
  (oracle/_ref) when that build is present;
* the reference test suite's own known-answer tests, restated
  (proj/tests/test_physics.cpp line numbers cited per test).
"""
import glob
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_1711_00289_b200 import gridgen as G

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
FIELDS = ("tend_T", "tend_q", "precip", "work", "exited")


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.int64), b.view(np.int64))
    return np.array_equal(a, b)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_matches_golden_bitwise(path):
    g = np.load(path)
    for v in (0, 1, 2):
        opts = O.Options(variant=v, activity_threshold=float(g["activity_threshold"]))
        for k in ("deep", "shallow"):
            r = O.convection(k, g["s"], g["T"], g["q"], opts)
            assert r.status == 0
            for f in FIELDS:
                assert bits_equal(getattr(r, f), g[f"{k}_v{v}_{f}"]), f"{path}: {k} v{v} {f}"


def test_golden_fixtures_present():
    assert len(GOLDEN) >= 5


@pytest.mark.skipif(not O.ref_available(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("cfg", ["ref", "c1", "c2", "c3", "c5_50"])
def test_oracle_matches_reference_build(cfg, variant):
    kw = {"n": 2048} if cfg in ("ref", "c1") else {"shape": (24, 36)}
    s, T, q = G.make_config(cfg, seed=17, **kw)
    opts = O.Options(variant=variant, activity_threshold=G.config_threshold(cfg))
    for k in ("deep", "shallow"):
        a = O.convection(k, s, T, q, opts)
        b = O.ref_convection(k, s, T, q, opts)
        assert a.status == b.status == 0
        for f in FIELDS:
            assert bits_equal(getattr(a, f), getattr(b, f)), f"{cfg} {k} v{variant} {f}"


@pytest.mark.skipif(not O.ref_available(), reason="reference build (oracle/_ref) not present")
def test_reference_generator_restatements_agree():
    for n, band, seed in ((64, 0.3, 42), (1000, 0.4, 7), (4096, 0.35, 1234)):
        a = O.ref_make_grid(n, 30, band, seed)
        b = O.make_grid(n, 30, band, seed)
        c = G.reference_grid(n, 30, band, seed)
        for x, y, z in zip(a, b, c):
            assert bits_equal(x, y) and bits_equal(x, z)


# ---- reference known-answer tests (proj/tests/test_physics.cpp) ----------

def entropy_f(t):
    return math.exp(0.05 * t) + 0.01 * t


def bisect_root(y):
    lo, hi = -400.0, 400.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if entropy_f(mid) < y:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def test_ientropy_frozen_anchors():
    # test_physics.cpp:183-187: y = 1 from guess 0 -> root 0, zero iterations
    st, root, it, _ = O.ientropy_solve(1.0, 0.0)
    assert st == 0 and root == 0.0 and it == 0
    # :189-195: y = e + 0.2 -> root 20
    y = math.exp(1.0) + 0.2
    st, root, it, _ = O.ientropy_solve(y, 60.0)
    assert st == 0 and it > 0 and abs(root - 20.0) < 1e-9 and abs(root - bisect_root(y)) < 1e-9
    # :197-203: bisection sweep
    for y in (1.1, 1.25, 1.3017, 1.5, 2.0, math.exp(1.0) + 1.0, 9.7):
        st, root, it, _ = O.ientropy_solve(y, 180.0)
        assert st == 0 and abs(root - bisect_root(y)) < 1e-8
        assert abs(entropy_f(root) - y) <= 1e-12 * (1.0 + 1e-3)


def test_ientropy_iterations_monotone_in_guess():
    # test_physics.cpp:206-216
    for y in (1.26, 1.31, 1.35):
        prev = 0
        for guess in (30.0, 60.0, 104.0, 140.0, 184.0):
            st, _, it, _ = O.ientropy_solve(y, guess)
            assert st == 0 and it >= prev
            prev = it


def test_ientropy_rejects_bad_inputs():
    # test_physics.cpp:218-225
    assert O.ientropy_solve(float("nan"), 10.0)[0] == 2
    assert O.ientropy_solve(1.3, 184.0, O.Options(newton_max_iter=2))[0] == 4


def synthetic_column(col_id, s, nl, seed):
    """test_physics.cpp:159-172, level-major single column."""
    c = np.arange(nl, dtype=np.uint64) + np.uint64(col_id * nl)
    T = 250.0 + 60.0 * G.rng_u01(seed, 11, c)
    q = 0.022 * G.rng_u01(seed, 12, c)
    return np.array([s]), T.reshape(nl, 1), q.reshape(nl, 1)


def test_deep_skips_inactive_columns():
    # test_physics.cpp:227-246
    s, T, q = synthetic_column(3, 0.31, 30, 99)
    r = O.convection("deep", s, T, q)
    assert r.exited[0] == 1 and r.work[0] == 0 and r.precip[0] == 0.0
    assert not r.tend_T.any() and not r.tend_q.any()
    s, T, q = O.make_grid(32, 30, 0.0, 42)
    r = O.convection("deep", s, T, q)
    assert (r.exited == 1).all() and (r.work == 0).all()


def test_deep_work_grows_with_activity():
    # test_physics.cpp:264-277
    for seed in (1, 2, 3):
        s, T, q = synthetic_column(0, 0.55, 30, seed)
        prev = O.convection("deep", s, T, q).work[0]
        assert prev > 0
        for sv in (0.65, 0.75, 0.85, 0.95):
            w = O.convection("deep", np.array([sv]), T, q).work[0]
            assert w >= prev
            prev = w


def test_band_position_and_ranges():
    # test_physics.cpp:322-355
    s, T, q = O.make_grid(64, 30, 0.3, 42)
    trop = (np.arange(64) >= 22) & (np.arange(64) < 41)
    assert (s[trop] >= 0.5).all() and (s[~trop] < 0.5).all()
    s, T, q = O.make_grid(128, 30, 0.3, 5)
    assert (s >= 0).all() and (s < 1).all()
    assert (T >= 250).all() and (T < 310).all() and (q >= 0).all() and (q < 0.022).all()


def test_shallow_exit_prices_phases():
    # test_physics.cpp:357-378
    s, T, q = synthetic_column(1, 0.05, 30, 42)
    w = O.convection("shallow", s, T, q)
    assert w.exited[0] == 1 and w.work[0] == 30 and w.precip[0] == 0.0
    s, T, q = synthetic_column(2, 0.95, 30, 42)
    r = O.convection("shallow", s, T, q)
    assert r.exited[0] == 0 and r.work[0] == 120 and r.tend_T.any()


def test_shallow_exits_spread_across_phases():
    # test_physics.cpp:392-415
    s, T, q = O.make_grid(256, 30, 0.3, 3)
    r = O.convection("shallow", s, T, q)
    cats = np.where(r.exited == 1, r.work // 30 - 1, 4)
    counts = np.bincount(cats, minlength=5)
    assert counts[0] > 0 and counts[1] > 0 and counts[4] > 0 and (counts > 0).sum() >= 4


def test_strength_reduced_identities():
    # test_physics.cpp:417-447
    s, T, q = synthetic_column(0, 0.8, 30, 77)
    q0 = np.zeros_like(q)
    for k in ("deep", "shallow"):
        a = O.convection(k, s, T, q0, O.Options(variant=0))
        b = O.convection(k, s, T, q0, O.Options(variant=1))
        for f in FIELDS:
            assert bits_equal(getattr(a, f), getattr(b, f))
    s, T, q = O.make_grid(64, 30, 0.3, 31)
    a = O.convection("deep", s, T, q, O.Options(variant=0))
    b = O.convection("deep", s, T, q, O.Options(variant=1))
    assert max(np.abs(a.tend_T - b.tend_T).max(), np.abs(a.tend_q - b.tend_q).max()) <= 1e-12


def test_approx_exp_budget():
    # test_physics.cpp:449-465
    x = np.arange(-12000, 100001, 7) * 1e-4
    lib = O.lib()
    got = np.array([lib.orc_approx_exp(v) for v in x])
    want = np.exp(x)
    rel = np.abs(got - want) / want
    assert rel.max() <= 5e-13
    assert (got != want).any()


def test_approx_variant_deviation_inside_budget():
    # test_physics.cpp:467-486
    s, T, q = O.make_grid(64, 30, 0.3, 31)
    a = O.convection("deep", s, T, q, O.Options(variant=0))
    b = O.convection("deep", s, T, q, O.Options(variant=2))
    d = max(np.abs(a.tend_T - b.tend_T).max(), np.abs(a.tend_q - b.tend_q).max())
    assert 0.0 < d <= 1e-7


def test_kernel_error_reports_column():
    # test_physics.cpp:488-501
    s, T, q = O.make_grid(8, 30, 1.0, 42)
    T[3, 5] = float("nan")
    r = O.convection("deep", s, T, q)
    assert r.status == 2 and r.fail_col == 5
    s[2] = float("nan")
    assert O.convection("deep", s, T, q).fail_col == 2
    assert O.convection("shallow", s, T, q).fail_col == 2


def test_newton_margin_classifier_is_recorded():
    s, T, q = O.make_grid(256, 30, 0.4, 42)
    r = O.convection("deep", s, T, q)
    act = r.exited == 0
    assert np.isfinite(r.margin[act]).all() and (r.margin[act] >= 0).all()
    assert np.isinf(r.margin[~act]).all()


@pytest.mark.skipif(not O.ref_available(), reason="reference build missing")
def test_reference_error_growth_c11():
    """acceptance.cpp:595-613 on the reference build: both answer-changing
    variants stay inside the perturbation envelope, which does not vanish."""
    s, T, q = O.make_grid(64, 30, 0.3, 42)
    for v in (O.STRENGTH_REDUCED, O.APPROX_TRANSCENDENTAL):
        g = O.ref_error_growth("deep", s, T, q, O.EXACT, v, 50)
        assert g.status == 0 and g.envelope_ok and g.rms_pert[-1] > 0.0
    g = O.ref_error_growth("deep", s, T, q, O.EXACT, O.EXACT, 10)
    assert (g.rms_mod == 0.0).all()


@pytest.mark.skipif(not O.ref_available(), reason="reference build missing")
@pytest.mark.parametrize("nd", [0, 1, 7, 1000])
def test_reference_packed_bytes_formula(nd):
    """The staging byte accounting this repo reports (stats h2d/d2h) is the
    reference's pack() payload: 8 nd (2L + 1) in (+32 with the option block),
    16 nd L + 17 nd out per kernel."""
    L = 30
    assert O.ref_packed_bytes(nd, L, True) == (8 * nd * (2 * L + 1) + 32, 16 * nd * L + 17 * nd)
    assert O.ref_packed_bytes(nd, L, False) == (8 * nd * (2 * L + 1), 16 * nd * L + 17 * nd)


def test_exp_restatement_bit_exact_against_libm():
    """orc_exp_gl (glibc 2.39's table-driven exp restated, with the table from
    tools/gen_exp_table.py) equals the running libm exp -- the exp the
    reference calls for Exact/StrengthReduced (physics.cpp:35) -- bit for bit.
    The device's exp_gl (colmath.cuh) is the same restatement; with it the
    strict Newton path reproduces the reference's iterates exactly."""
    from conftest import exp_arguments
    x = exp_arguments()
    a, b = O.exp_gl(x), O.libm_exp(x)
    same = (a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))
    assert same.all(), f"{int((~same).sum())} of {x.size} differ, e.g. x={x[~same][:4]}"


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_run_parallel_outputs_equal_oracle():
    """The reference's threaded run_parallel (the CPU baseline bench.py times
    and checks the GPU against) returns the serial oracle's outputs bit for
    bit (sched.cpp:145: disjoint output slots)."""
    s, T, q = G.make_config("c2", n=3000, seed=17)
    for kernel in ("deep", "shallow"):
        r, wall = O.ref_run_parallel(kernel, s, T, q, n_threads=4)
        o = O.convection(kernel, s, T, q)
        assert r.status == 0 and wall > 0.0
        for f in FIELDS:
            assert bits_equal(getattr(r, f), getattr(o, f)), (kernel, f)
