"""GPU tier: the CUDA path, through the C ABI, against the CPU oracle on the
same seeded inputs -- all five BASELINE configs x all three variants -- and
against the golden fixtures the reference itself produced.

Parity rule (BASELINE.json north_star), written here and
applied to EVERY column with no Newton-margin exemption:
  * deep trigger flags and shallow exit flags: exact (shallow flags exempt
    where the exit predicate is within 1e-9 relative of its theta -- the
    north star's near-threshold rule; no column of any grid falls there);
  * work_units: exact, every variant, every device path.  The device's exp
    is the libm's bit for bit (colmath.cuh exp_gl), so the strict path runs
    the reference's own iterates; the default relaxed path re-runs exactly
    any solve whose stop decision falls in the guard band around newton_tol
    (colmath.cuh), so its counts are the reference's too;
  * fp64 fields: within 1e-10 relative or 1e-14 absolute.
"""
import glob
import os

import numpy as np
import pytest

import oracle as O
import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen as G

pytestmark = pytest.mark.gpu

REL, ABS = 1e-10, 1e-14
PRED_MARGIN = 1e-9
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def check(got: P.ColumnOutputs, want, kernel: str, margin=None):
    """want: oracle Result or dict of golden arrays.  Returns the number of
    work_units mismatches (always 0 when it returns)."""
    g = (lambda f: getattr(want, f)) if not isinstance(want, dict) else (lambda f: want[f])
    margin = g("margin") if margin is None and not isinstance(want, dict) else margin
    exempt = np.zeros(got.exited_early.shape, bool)
    if kernel == "shallow" and margin is not None:
        exempt = margin < PRED_MARGIN
    assert np.array_equal(got.exited_early[~exempt], g("exited")[~exempt]), f"{kernel}: exit/trigger flags differ"
    flip = (got.work_units != g("work")) & ~exempt
    assert not flip.any(), f"{kernel}: work_units differ in {int(flip.sum())} columns: {np.nonzero(flip)[0][:8]}"
    for f in ("tend_T", "tend_q", "precip"):
        a, b = getattr(got, f), g(f)
        ok = np.abs(a - b) <= np.maximum(REL * np.abs(b), ABS)
        assert ok.all(), f"{kernel}.{f}: {int((~ok).sum())} values outside tolerance, max |d| {np.max(np.abs(a - b))}"
    return int(flip.sum())


CONFIGS = [("ref", {"n": 4096}), ("c1", {}), ("c2", {}), ("c3", {"shape": (96, 144)}),
           ("c4", {"shape": (96, 144)}), ("c5_05", {"shape": (64, 96)}), ("c5_50", {"shape": (64, 96)}),
           ("c5_95", {"shape": (64, 96)})]


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("cfg,kw", CONFIGS, ids=[c for c, _ in CONFIGS])
def test_convect_matches_oracle(ctx, cfg, kw, variant):
    s, T, q = G.make_config(cfg, seed=11, **kw)
    thr = G.config_threshold(cfg)
    deep, sh = ctx.convect(s, T, q, P.KernelOptions(variant=variant, activity_threshold=thr))
    oo = O.Options(variant=variant, activity_threshold=thr)
    od, osh = O.convection("deep", s, T, q, oo), O.convection("shallow", s, T, q, oo)
    check(deep, od, "deep")
    check(sh, osh, "shallow")
    assert ctx.last_stats.n_triggered == int((od.exited == 0).sum())


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_convect_matches_reference_golden(ctx, path):
    g = np.load(path)
    for v in (0, 1, 2):
        deep, sh = ctx.convect(g["s"], g["T"], g["q"],
                               P.KernelOptions(variant=v, activity_threshold=float(g["activity_threshold"])))
        oo = O.Options(variant=v, activity_threshold=float(g["activity_threshold"]))
        dm = O.convection("deep", g["s"], g["T"], g["q"], oo).margin
        sm = O.convection("shallow", g["s"], g["T"], g["q"], oo).margin
        for k, got, m in (("deep", deep, dm), ("shallow", sh, sm)):
            want = {f: g[f"{k}_v{v}_{f}"] for f in ("tend_T", "tend_q", "precip", "work", "exited")}
            check(got, want, k, margin=m)


def test_approx_variant_roots_bit_exact(ctx):
    """With variant=approx-exp every operation on the Newton path is IEEE
    arithmetic the device reproduces exactly, so precip (a function of the
    precipitation roots only, no sin) is bit-identical to the oracle."""
    s, T, q = G.make_config("c1", seed=5)
    deep, _ = ctx.convect(s, T, q, P.KernelOptions(variant=2))
    od = O.convection("deep", s, T, q, O.Options(variant=2))
    assert np.array_equal(deep.precip.view(np.int64), od.precip.view(np.int64))
    assert np.array_equal(deep.work_units, od.work)


@pytest.mark.parametrize("cfg", ["c4", "c5_95"])
def test_full_size_strided_parity(ctx, cfg):
    """Full BASELINE size on the GPU; the oracle checks every 29th column
    (columns are independent, physics.hpp:26-30)."""
    s, T, q = G.make_config(cfg, seed=42)
    assert s.size == 884736
    deep, sh = ctx.convect(s, T, q)
    idx = np.arange(0, s.size, 29)
    sub = lambda a: np.ascontiguousarray(a[..., idx])
    od = O.convection("deep", sub(s), sub(T), sub(q))
    osh = O.convection("shallow", sub(s), sub(T), sub(q))
    pick = lambda o: P.ColumnOutputs(o.tend_T[:, idx], o.tend_q[:, idx], o.precip[idx], o.work_units[idx],
                                     o.exited_early[idx])
    check(pick(deep), od, "deep")
    check(pick(sh), osh, "shallow")
    # size-independent properties over the whole grid
    trig = deep.exited_early == 0
    assert trig.sum() == ctx.last_stats.n_triggered == int((s > 0.5).sum())
    assert (deep.work_units[~trig] == 0).all() and not deep.tend_T[:, ~trig].any()
    assert ((deep.work_units[trig] >= 2 * 30) & (deep.work_units[trig] <= 2 * 30 * 100)).all()
    assert np.isin(sh.work_units, [30, 60, 90, 120]).all()
    assert not sh.tend_q[:, sh.exited_early == 1].any()


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_c3_full_size_every_column(ctx, variant):
    """BASELINE config 3 at its stated size: the f09-shaped 192 x 288 grid
    (55,296 columns) at activity_threshold 0.75 (30 % deep, 25 % shallow-only
    survivors), every column against the oracle."""
    s, T, q = G.make_config("c3", seed=42)
    assert s.size == 55296
    thr = G.config_threshold("c3")
    assert thr == 0.75
    deep, sh = ctx.convect(s, T, q, P.KernelOptions(variant=variant, activity_threshold=thr))
    oo = O.Options(variant=variant, activity_threshold=thr)
    od, osh = O.convection("deep", s, T, q, oo), O.convection("shallow", s, T, q, oo)
    check(deep, od, "deep")
    check(sh, osh, "shallow")
    trig = s > thr
    assert abs(trig.mean() - 0.30) < 0.01
    surv_only = (~trig) & (osh.exited == 0)
    assert abs(surv_only.mean() - 0.25) < 0.03


def test_determinism(ctx):
    s, T, q = G.make_config("c2", seed=2)
    a = ctx.convect(s, T, q)
    b = ctx.convect(s, T, q)
    for x, y in zip(a, b):
        for f in ("tend_T", "tend_q", "precip", "work_units", "exited_early"):
            assert np.array_equal(getattr(x, f), getattr(y, f))


def test_ientropy_batch_known_answers(ctx):
    """test_physics.cpp:183-203 on the device."""
    import math
    root, it = ctx.ientropy_solve([1.0], [0.0])
    assert root[0] == 0.0 and it[0] == 0
    y = math.exp(1.0) + 0.2
    root, it = ctx.ientropy_solve([y], [60.0])
    assert abs(root[0] - 20.0) < 1e-9 and it[0] > 0
    ys = np.array([1.1, 1.25, 1.3017, 1.5, 2.0, math.exp(1.0) + 1.0, 9.7])
    for v in (0, 2):
        root, it = ctx.ientropy_solve(ys, 180.0, P.KernelOptions(variant=v))
        for yy, rr, ii in zip(ys, root, it):
            st, r2, i2, _ = O.ientropy_solve(float(yy), 180.0, O.Options(variant=v))
            assert st == 0 and abs(rr - r2) <= 1e-12 * max(1.0, abs(r2))
            if v == 2:
                assert rr == r2 and ii == i2


def test_exp_bit_exact_against_libm(ctx):
    """The device exp_gl (colmath.cuh) equals the libm exp the reference calls
    (physics.cpp:35) bit for bit: Newton range, shallow range, the scaled
    special cases, tiny and non-finite arguments, random bit patterns."""
    from conftest import exp_arguments
    x = exp_arguments()
    got, want = ctx.exp(x), O.libm_exp(x)
    same = (got.view(np.int64) == want.view(np.int64)) | (np.isnan(got) & np.isnan(want))
    assert same.all(), f"{int((~same).sum())} differ, e.g. x={x[~same][:4]}"


def test_approx_exp_bit_exact(ctx):
    x = np.concatenate([np.arange(-12000, 100001, 7) * 1e-4, np.linspace(-64, 64, 20001)])
    got = ctx.approx_exp(x)
    lib = O.lib()
    want = np.array([lib.orc_approx_exp(float(v)) for v in x])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


@pytest.fixture(scope="module")
def strict_ctx():
    """Reference rounding in every Newton update (CVG_STRICT=1), for all
    variants -- the path the relaxed update of Exact/StrengthReduced
    replaces by default (colmath.cuh, newton_relaxed_step)."""
    from conftest import env_context
    c = env_context(CVG_STRICT="1")
    yield c
    c.close()


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("cfg,kw", [("c1", {}), ("c4", {"shape": (96, 144)})], ids=["c1", "c4"])
def test_strict_update_matches_oracle_and_relaxed(ctx, strict_ctx, cfg, kw, variant):
    s, T, q = G.make_config(cfg, seed=13, **kw)
    o = P.KernelOptions(variant=variant)
    oo = O.Options(variant=variant)
    od, osh = O.convection("deep", s, T, q, oo), O.convection("shallow", s, T, q, oo)
    d_strict, s_strict = strict_ctx.convect(s, T, q, o)
    d_relax, s_relax = ctx.convect(s, T, q, o)
    check(d_strict, od, "deep")
    check(s_strict, osh, "shallow")
    check(d_relax, od, "deep")
    check(s_relax, osh, "shallow")
    # strict = the reference's own roundings with the libm's exp: the
    # precipitation roots, their k-order sum and the counts are bit-identical
    # (only tend_T / tend_q go through sin)
    assert np.array_equal(d_strict.precip.view(np.int64), od.precip.view(np.int64))
    assert np.array_equal(d_strict.work_units, od.work)
    # strict shallow keeps the reference's per-term phase sums: bit-identical
    # flags and phase counts
    assert np.array_equal(s_strict.work_units, osh.work) and np.array_equal(s_strict.exited_early, osh.exited)


def test_relaxed_guard_falls_back_for_tight_tolerance(ctx, strict_ctx):
    """newton_tol below 2^-40 * 2^floor(log2 |y|) takes the exact update
    (relaxed_ok): results equal the strict path bit for bit."""
    s, T, q = G.make_config("c1", n=512, seed=3)
    o = P.KernelOptions(newton_tol=2e-13)
    a, _ = ctx.convect(s, T, q, o)
    b, _ = strict_ctx.convect(s, T, q, o)
    for f in ("tend_T", "tend_q", "precip", "work_units", "exited_early"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


@pytest.mark.parametrize("cfg", ["c4", "c5_05", "c5_50", "c5_95"])
def test_far32_full_grid_every_column(ctx, cfg):
    """The FP32 far phase of the relaxed Newton solve (default for Exact;
    colmath.cuh newton_far32_step) against the oracle on EVERY column of the
    full 884,736-column grid: flags and work_units exact (the guard band
    re-runs the solves whose stop decision is within rounding noise of tol),
    fp64 fields within tolerance."""
    s, T, q = G.make_config(cfg, seed=42)
    deep, sh = ctx.convect(s, T, q, P.KernelOptions())
    assert ctx.last_stats.n_recomputed > 0   # the guard band did re-run solves
    od = O.convection("deep", s, T, q)
    check(deep, od, "deep")
    check(sh, O.convection("shallow", s, T, q), "shallow")


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("cfg,kw", [("c2", {}), ("c3", {"shape": (96, 144)}), ("c5_95", {"shape": (64, 96)})],
                         ids=["c2", "c3", "c5_95"])
def test_far32_against_fp64_update(ctx, cfg, kw, variant):
    """far32 on vs off (CVG_FLAG_NO_FAR32): both match the oracle."""
    s, T, q = G.make_config(cfg, seed=21, **kw)
    thr = G.config_threshold(cfg)
    oo = O.Options(variant=variant, activity_threshold=thr)
    od = O.convection("deep", s, T, q, oo)
    a, _ = ctx.convect(s, T, q, P.KernelOptions(variant=variant, activity_threshold=thr))
    b, _ = ctx.convect(s, T, q, P.KernelOptions(variant=variant, activity_threshold=thr, far32=False))
    check(a, od, "deep")
    check(b, od, "deep")


@pytest.mark.parametrize("tol", [1e-12, 1e-6, 2e-6, 2.0 ** -40, 1e-13])
def test_hot_path_window_edges(ctx, tol):
    """Targets y on both sides of the FP32/relaxed hot-path window [0.25, 16)
    (colmath.cuh in_far_window), guesses on both sides of 1190 (s up to 7.4),
    and tolerances at the window's limits (1e-6, 2^-40) and just outside:
    every column, every path, against the oracle."""
    Ts = np.concatenate([np.linspace(-2000.0, 16500.0, 61), [-750.0, -749.9, 15000.0, 15001.0]])
    cols = [(s_, q_, T_) for s_ in (0.55, 0.9, 3.0, 7.38, 7.45) for q_ in (0.0, 0.02) for T_ in Ts]
    n, L = len(cols), 30
    s = np.array([c[0] for c in cols])
    T = np.empty((L, n))
    q = np.empty((L, n))
    for j, (_, q_, T_) in enumerate(cols):
        T[:, j] = T_ + np.linspace(0.0, 3.0, L)   # levels spread around the column's target
        q[:, j] = q_
    o = P.KernelOptions(newton_tol=tol)
    deep, _ = ctx.convect(s, T, q, o, kernels=P.DEEP)
    od = O.convection("deep", s, T, q, O.Options(newton_tol=tol))
    check(deep, od, "deep")


@pytest.fixture(scope="module")
def tpc_ctx():
    """The thread-per-column deep kernel forced on every call (CVG_DEEP_TPC=1;
    by default only calls of >= 320k columns use it)."""
    from conftest import env_context
    c = env_context(CVG_DEEP_TPC="1")
    yield c
    c.close()


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("cfg,kw", CONFIGS, ids=[c for c, _ in CONFIGS])
def test_thread_per_column_kernel_matches_oracle(tpc_ctx, cfg, kw, variant):
    s, T, q = G.make_config(cfg, seed=17, **kw)
    thr = G.config_threshold(cfg)
    deep, sh = tpc_ctx.convect(s, T, q, P.KernelOptions(variant=variant, activity_threshold=thr))
    oo = O.Options(variant=variant, activity_threshold=thr)
    check(deep, O.convection("deep", s, T, q, oo), "deep")
    check(sh, O.convection("shallow", s, T, q, oo), "shallow")


@pytest.mark.parametrize("n", [1, 5, 31, 33, 1001])
def test_thread_per_column_ragged_and_errors(tpc_ctx, n):
    s, T, q = G.make_config("c1", n=n, seed=4)
    deep, _ = tpc_ctx.convect(s, T, q)
    check(deep, O.convection("deep", s, T, q), "deep")
    if n >= 5:
        s2 = s.copy()
        s2[:] = 0.9
        T2 = T.copy()
        T2[7, n - 1] = np.nan
        T2[3, n - 2] = np.nan
        with pytest.raises(P.KernelError) as e:
            tpc_ctx.deep_convection(s2, T2, q)
        assert e.value.column == n - 2


@pytest.mark.parametrize("variant,strict", [(1, False), (2, False), (0, True)])
def test_full_grid_variants_and_strict(ctx, variant, strict):
    """The f02 grid through the default (size-switched: thread-per-column)
    deep kernel for StrengthReduced, ApproxTranscendental (bit-exact work and
    k-order precip) and the strict update, every 7th column against the
    oracle."""
    s, T, q = G.make_config("c4", seed=42)
    deep, _ = ctx.convect(s, T, q, P.KernelOptions(variant=variant, strict=strict), kernels=P.DEEP)
    idx = np.arange(0, s.size, 7)
    sub = lambda a: np.ascontiguousarray(a[..., idx])
    od = O.convection("deep", sub(s), sub(T), sub(q), O.Options(variant=variant))
    pick = P.ColumnOutputs(deep.tend_T[:, idx], deep.tend_q[:, idx], deep.precip[idx], deep.work_units[idx],
                           deep.exited_early[idx])
    check(pick, od, "deep")
    if variant == 2 or strict:
        assert np.array_equal(pick.precip.view(np.int64), od.precip.view(np.int64))


@pytest.fixture(scope="module", params=[("0", "0", "-1"), ("0", "2", "-1"), ("0", "4", "0")],
                ids=["warp_per_column", "lpc2", "lpc4_redo_kernel"])
def kernel_ctx(request):
    """Deep kernels / re-derivation paths the size switches do not pick at
    test sizes: the warp-per-column kernel on the relaxed path
    (CVG_DEEP_LPC=0), the 2- and 4-lanes-per-column splits, and the separate
    redo_kernel (CVG_REDO_INLINE=0; calls below 100k columns re-derive
    inline by default)."""
    from conftest import env_context
    tpc, lpc, inline = request.param
    c = env_context(CVG_DEEP_TPC=tpc, CVG_DEEP_LPC=lpc, CVG_REDO_INLINE=inline)
    yield c
    c.close()


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("cfg,kw", CONFIGS, ids=[c for c, _ in CONFIGS])
def test_other_deep_kernels_match_oracle(kernel_ctx, cfg, kw, variant):
    s, T, q = G.make_config(cfg, seed=19, **kw)
    thr = G.config_threshold(cfg)
    deep, sh = kernel_ctx.convect(s, T, q, P.KernelOptions(variant=variant, activity_threshold=thr))
    oo = O.Options(variant=variant, activity_threshold=thr)
    check(deep, O.convection("deep", s, T, q, oo), "deep")
    check(sh, O.convection("shallow", s, T, q, oo), "shallow")


@pytest.mark.parametrize("n", [1, 7, 33, 1001])
def test_other_deep_kernels_ragged_and_errors(kernel_ctx, n):
    s, T, q = G.make_config("c1", n=n, seed=6)
    deep, _ = kernel_ctx.convect(s, T, q)
    check(deep, O.convection("deep", s, T, q), "deep")
    if n >= 7:
        s2 = np.full_like(s, 0.9)
        T2 = T.copy()
        T2[11, n - 1] = np.nan
        T2[2, n - 3] = np.nan
        with pytest.raises(P.KernelError) as e:
            kernel_ctx.deep_convection(s2, T2, q)
        assert e.value.column == n - 3
