"""GPU tier: error semantics and edge cases at the C ABI, checked against the
reference's behaviour (the serial driver's first -- i.e. lowest -- failing
column, physics.cpp:227-245; KernelError taxonomy, errors.hpp:26-36,
capi.cpp:51-81) and against the oracle for ragged/odd shapes."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen as G

pytestmark = pytest.mark.gpu


def both_close(got, want):
    for f, g in (("tend_T", "tend_T"), ("tend_q", "tend_q"), ("precip", "precip")):
        a, b = getattr(got, f), getattr(want, g)
        assert (np.abs(a - b) <= np.maximum(1e-10 * np.abs(b), 1e-14)).all(), f
    assert np.array_equal(got.exited_early, want.exited)


def test_kernel_error_reports_lowest_column(ctx):
    # test_physics.cpp:488-501: NaN T in active column 5 -> KernelError column 5
    s, T, q = O.make_grid(8, 30, 1.0, 42)
    T[3, 5] = np.nan
    with pytest.raises(P.KernelError) as e:
        ctx.deep_convection(s, T, q)
    assert e.value.column == 5 and "column 5" in str(e.value) and "non-finite input" in str(e.value)
    # several failing columns: the lowest is reported
    T[7, 2] = np.nan
    T[0, 7] = np.inf
    with pytest.raises(P.KernelError) as e:
        ctx.deep_convection(s, T, q)
    assert e.value.column == 2
    # first_col offsets the reported id (ColumnState::col_id)
    with pytest.raises(P.KernelError) as e:
        ctx.deep_convection(s, T, q, first_col=1000)
    assert e.value.column == 1002


def test_nan_activity_fails_both_kernels(ctx):
    s, T, q = G.make_config("c1", n=256, seed=1)
    s[100] = np.nan
    s[200] = np.inf
    for kern in ("deep_convection", "shallow_convection"):
        with pytest.raises(P.KernelError) as e:
            getattr(ctx, kern)(s, T, q)
        assert e.value.column == 100 and "non-finite activity" in str(e.value)


def test_nan_moisture_in_inactive_deep_column_is_not_an_error(ctx):
    # deep throws on NaN T/q only for active columns (physics.cpp:111-113)
    s, T, q = O.make_grid(64, 30, 0.3, 7)
    inactive = int(np.nonzero(s <= 0.5)[0][0])
    q[4, inactive] = np.nan
    deep = ctx.deep_convection(s, T, q)
    od = O.convection("deep", s, T, q)
    assert od.status == 0
    both_close(deep, od)
    # shallow propagates NaN into outputs without failing (predicate false)
    sh = ctx.shallow_convection(s, T, q)
    osh = O.convection("shallow", s, T, q)
    assert osh.status == 0
    assert np.array_equal(sh.exited_early, osh.exited) and np.array_equal(sh.work_units, osh.work)
    assert np.array_equal(np.isnan(sh.tend_T), np.isnan(osh.tend_T))


def test_max_iter_exceeded_is_no_convergence(ctx):
    # test_physics.cpp:223-224 (max_iter = 2), at batch level
    s, T, q = O.make_grid(16, 30, 0.5, 3)
    opts = P.KernelOptions(newton_max_iter=2)
    with pytest.raises(P.KernelError) as e:
        ctx.deep_convection(s, T, q, opts)
    od = O.convection("deep", s, T, q, O.Options(newton_max_iter=2))
    assert od.status == 4 and e.value.column == od.fail_col
    assert "no convergence within 2 iterations" in str(e.value)
    with pytest.raises(P.KernelError):
        ctx.ientropy_solve([1.3], [184.0], opts)


def test_exact_max_iter_boundary(ctx):
    # a solve needing exactly U updates passes with max_iter = U and fails with U - 1
    st, root, it, _ = O.ientropy_solve(1.3, 184.0)
    r, i = ctx.ientropy_solve([1.3], [184.0], P.KernelOptions(newton_max_iter=it))
    assert i[0] == it
    with pytest.raises(P.KernelError):
        ctx.ientropy_solve([1.3], [184.0], P.KernelOptions(newton_max_iter=it - 1))


@pytest.mark.parametrize("n", [0, 1, 31, 33, 4095, 4097, 12345])
def test_ragged_sizes(ctx, n):
    s, T, q = G.make_config("ref", n=max(n, 1), seed=n + 1)
    s, T, q = s[:n], np.ascontiguousarray(T[:, :n]), np.ascontiguousarray(q[:, :n])
    deep, sh = ctx.convect(s, T, q)
    if n == 0:
        assert deep.tend_T.shape == (30, 0)
        return
    both_close(deep, O.convection("deep", s, T, q))
    both_close(sh, O.convection("shallow", s, T, q))


@pytest.mark.parametrize("L", [1, 7, 30, 32, 33, 64])
def test_level_counts(ctx, L):
    s, T, q = G.make_config("ref", n=700, L=L, seed=L)
    for v in (0, 2):
        deep, sh = ctx.convect(s, T, q, P.KernelOptions(variant=v))
        oo = O.Options(variant=v)
        od = O.convection("deep", s, T, q, oo)
        both_close(deep, od)
        both_close(sh, O.convection("shallow", s, T, q, oo))
        if v == 2:
            assert np.array_equal(deep.work_units, od.work)


def test_strided_rows_and_host_ld(ctx):
    """ld > n on input and output (a column block inside a wider grid)."""
    s, T, q = G.make_config("c1", n=1000, seed=4)
    n, L = 900, T.shape[0]
    lib = P.load_library()
    cols = P._Columns(n, L, 0, T.shape[1], s.ctypes.data, T.ctypes.data, q.ctypes.data, 0)
    out = P.ColumnOutputs(np.zeros((L, 1000)), np.zeros((L, 1000)), np.zeros(n), np.zeros(n, np.int64),
                          np.zeros(n, np.uint8))
    st = P.Stats()
    o = P._Outputs(out.tend_T.ctypes.data, out.tend_q.ctypes.data, out.precip.ctypes.data,
                   out.work_units.ctypes.data, out.exited_early.ctypes.data, 1000, 0)
    rc = lib.cvg_deep_convection(ctx._h, C.byref(cols), C.byref(P.KernelOptions()), C.byref(o), C.byref(st))
    assert rc == 0
    od = O.convection("deep", s[:n], np.ascontiguousarray(T[:, :n]), np.ascontiguousarray(q[:, :n]))
    got = P.ColumnOutputs(out.tend_T[:, :n], out.tend_q[:, :n], out.precip, out.work_units, out.exited_early)
    both_close(got, od)
    assert not out.tend_T[:, n:].any()   # untouched padding


def test_invalid_arguments(ctx):
    lib = P.load_library()
    s, T, q = G.make_config("ref", n=64, seed=1)
    cols = P._Columns(64, 30, 0, 32, s.ctypes.data, T.ctypes.data, q.ctypes.data, 0)  # ld < n
    assert lib.cvg_convect(ctx._h, C.byref(cols), C.byref(P.KernelOptions()), 3, None, None, None) == 1
    cols = P._Columns(64, 0, 0, 64, s.ctypes.data, T.ctypes.data, q.ctypes.data, 0)   # L = 0
    assert lib.cvg_convect(ctx._h, C.byref(cols), C.byref(P.KernelOptions()), 3, None, None, None) == 1
    assert lib.cvg_last_error()
    with pytest.raises(ValueError):
        ctx.convect(s, T, q, P.KernelOptions(variant=5))


def test_device_resident_async_path(ctx):
    import torch
    s, T, q = G.make_config("c2", seed=9)
    dev = torch.device("cuda", 0)
    ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s, T, q))
    L, n = T.shape

    def outs():
        return (torch.empty((L, n), dtype=torch.float64, device=dev), torch.empty((L, n), dtype=torch.float64, device=dev),
                torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.int64, device=dev),
                torch.empty(n, dtype=torch.uint8, device=dev))
    do, so = outs(), outs()
    stream = torch.cuda.Stream()
    ctx.convect_async(ds, dT, dq, do, so, stream=stream)
    st = ctx.check(stream)
    assert st.n_triggered == int((s > 0.5).sum())
    got = P.ColumnOutputs(*[t.cpu().numpy() for t in do])
    both_close(got, O.convection("deep", s, T, q))
    # latched device error surfaces at check()
    ds[7] = float("nan")
    ctx.convect_async(ds, dT, dq, do, so, stream=stream)
    with pytest.raises(P.KernelError) as e:
        ctx.check(stream)
    assert e.value.column == 7


@pytest.fixture(scope="module")
def small_chunk_ctx():
    """A context whose host-buffer calls pipeline 1000-column chunks, so a
    few thousand columns cross several chunks and reuse every workspace slot."""
    from conftest import env_context
    c = env_context(CVG_CHUNK_COLS="1000")
    yield c
    c.close()


@pytest.mark.parametrize("n", [999, 1000, 1001, 7777])
def test_chunked_pipeline_matches_single_chunk(ctx, small_chunk_ctx, n):
    s, T, q = G.make_config("c1", n=n, seed=n)
    for v in (0, 2):
        o = P.KernelOptions(variant=v)
        d1, s1 = ctx.convect(s, T, q, o, first_col=50)
        d2, s2 = small_chunk_ctx.convect(s, T, q, o, first_col=50)
        for a, b in ((d1, d2), (s1, s2)):
            for f in ("tend_T", "tend_q", "precip", "work_units", "exited_early"):
                assert np.array_equal(getattr(a, f), getattr(b, f), equal_nan=True), f
        assert small_chunk_ctx.last_stats.n_triggered == int((s > 0.5).sum())
        assert small_chunk_ctx.last_stats.h2d_bytes == 8 * n * (1 + 2 * T.shape[0])


def test_chunked_pipeline_error_is_lowest_column_over_chunks(small_chunk_ctx):
    s, T, q = G.make_config("c1", n=5000, seed=3)
    active = np.nonzero(s > 0.5)[0]
    late, early = int(active[active > 4000][0]), int(active[(active > 1000) & (active < 2000)][0])
    T[2, late] = np.nan
    with pytest.raises(P.KernelError) as e:
        small_chunk_ctx.deep_convection(s, T, q, first_col=7)
    assert e.value.column == late + 7
    T[5, early] = np.inf
    with pytest.raises(P.KernelError) as e:
        small_chunk_ctx.deep_convection(s, T, q, first_col=7)
    assert e.value.column == early + 7
    # a deep failure is reported before a shallow one even when the shallow
    # failure sits in an earlier chunk (the reference runs deep first)
    s[10] = np.nan
    with pytest.raises(P.KernelError) as e:
        small_chunk_ctx.convect(s, T, q)
    assert e.value.column == 10 and "deep: non-finite activity" in str(e.value)
    s[10] = 0.1
    with pytest.raises(P.KernelError) as e:
        small_chunk_ctx.convect(s, T, q)
    assert e.value.column == early and "ientropy" in str(e.value)
    s[early - 1] = np.inf
    with pytest.raises(P.KernelError) as e:
        small_chunk_ctx.shallow_convection(s, T, q)
    assert e.value.column == early - 1 and "shallow" in str(e.value)
    # and the context is usable afterwards
    s, T, q = G.make_config("c1", n=3000, seed=4)
    both_close(small_chunk_ctx.deep_convection(s, T, q), O.convection("deep", s, T, q))


def test_chunked_pipeline_strided_host_rows(small_chunk_ctx):
    s, T, q = G.make_config("c1", n=3500, seed=5)
    n, L = 3200, T.shape[0]
    lib = P.load_library()
    cols = P._Columns(n, L, 0, T.shape[1], s.ctypes.data, T.ctypes.data, q.ctypes.data, 0)
    out = P.ColumnOutputs(np.zeros((L, 3500)), np.zeros((L, 3500)), np.zeros(n), np.zeros(n, np.int64),
                          np.zeros(n, np.uint8))
    o = P._Outputs(out.tend_T.ctypes.data, out.tend_q.ctypes.data, out.precip.ctypes.data,
                   out.work_units.ctypes.data, out.exited_early.ctypes.data, 3500, 0)
    st = P.Stats()
    rc = lib.cvg_deep_convection(small_chunk_ctx._h, C.byref(cols), C.byref(P.KernelOptions()), C.byref(o),
                                 C.byref(st))
    assert rc == 0
    od = O.convection("deep", s[:n], np.ascontiguousarray(T[:, :n]), np.ascontiguousarray(q[:, :n]))
    got = P.ColumnOutputs(out.tend_T[:, :n], out.tend_q[:, :n], out.precip, out.work_units, out.exited_early)
    both_close(got, od)
    assert not out.tend_T[:, n:].any()


def test_nan_activity_in_later_chunk_reports_absolute_column(small_chunk_ctx, ctx):
    """The trigger kernel keys failures by absolute column id (first_col +
    offset of the chunk), as the shallow and deep kernels do."""
    s, T, q = G.make_config("c1", n=4000, seed=8)
    s[2500] = np.nan
    for c in (small_chunk_ctx, ctx):
        with pytest.raises(P.KernelError) as e:
            c.deep_convection(s, T, q, first_col=7)
        assert e.value.column == 2507 and "non-finite activity" in str(e.value)
        with pytest.raises(P.KernelError) as e:
            c.convect(s, T, q, first_col=7)
        assert e.value.column == 2507 and "deep" in str(e.value)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 4093])
def test_group_tails(ctx, n):
    """Column counts that leave a partial 4-column group at the end; an
    all-triggered and an all-untriggered grid."""
    s, T, q = G.make_config("c1", n=max(n, 8), seed=n)
    s, T, q = s[:n].copy(), np.ascontiguousarray(T[:, :n]), np.ascontiguousarray(q[:, :n])
    for sv in (None, 0.9, 0.1):
        if sv is not None:
            s[:] = sv
        deep, sh = ctx.convect(s, T, q)
        both_close(deep, O.convection("deep", s, T, q))
        both_close(sh, O.convection("shallow", s, T, q))


@pytest.mark.parametrize("kernels,nk", [(P.DEEP, 1), (P.SHALLOW, 1), (P.BOTH, 2)])
def test_staging_bytes_follow_reference_pack(ctx, kernels, nk):
    """Host-buffer calls report the staging bytes of the reference's packed
    device transfer (hetero.cpp pack(), HeteroMetrics bytes_in / bytes_out):
    inputs T, q, s with the option scalars resident (kernel parameters), and
    tend_T, tend_q, precip, work_units, exited per kernel."""
    if not O.ref_available():
        pytest.skip("reference build missing")
    s, T, q = G.make_config("c1", n=3333, seed=2)
    ctx.convect(s, T, q, kernels=kernels)
    st = ctx.last_stats
    bi, bo = O.ref_packed_bytes(s.size, T.shape[0], send_scalars=False)
    assert st.h2d_bytes == bi and st.d2h_bytes == nk * bo


def test_graph_replay_tracks_buffer_contents(ctx):
    """Device-resident calls replay a captured CUDA graph per argument set:
    new input VALUES in the same buffers, a second output set (new graph)
    and a latched failure after replay all behave like fresh launches."""
    import torch
    dev = torch.device("cuda", 0)
    s0, T0, q0 = G.make_config("c1", n=3000, seed=21)
    L, n = T0.shape
    ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s0, T0, q0))

    def outs():
        return (torch.empty((L, n), dtype=torch.float64, device=dev), torch.empty((L, n), dtype=torch.float64, device=dev),
                torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.int64, device=dev),
                torch.empty(n, dtype=torch.uint8, device=dev))
    sets = [(outs(), outs()), (outs(), outs())]
    for it, seed in enumerate((21, 22, 23, 24)):
        s, T, q = G.make_config("c1", n=3000, seed=seed)
        ds.copy_(torch.from_numpy(s)); dT.copy_(torch.from_numpy(T)); dq.copy_(torch.from_numpy(q))
        do, so = sets[it % 2]
        for _ in range(2):
            ctx.convect_async(ds, dT, dq, do, so)
        st = ctx.check()
        assert st.n_triggered == int((s > 0.5).sum())
        both_close(P.ColumnOutputs(*[t.cpu().numpy() for t in do]), O.convection("deep", s, T, q))
        both_close(P.ColumnOutputs(*[t.cpu().numpy() for t in so]), O.convection("shallow", s, T, q))
    ds[11] = float("nan")
    ctx.convect_async(ds, dT, dq, *sets[0])
    with pytest.raises(P.KernelError) as e:
        ctx.check()
    assert e.value.column == 11
    ds[11] = 0.3
    ctx.convect_async(ds, dT, dq, *sets[0])
    ctx.check()   # the failure word was reset for the next call


def test_option_flags(ctx):
    s, T, q = G.make_config("c1", n=256, seed=2)
    o = P.KernelOptions()
    o.flags = 4   # unknown bit
    with pytest.raises(ValueError):
        ctx.convect(s, T, q, o)
    a, _ = ctx.convect(s, T, q, P.KernelOptions(far32=False))
    b, _ = ctx.convect(s, T, q, P.KernelOptions(far32=False, strict=True))
    od = O.convection("deep", s, T, q)
    both_close(a, od)
    both_close(b, od)


def test_async_call_inside_a_caller_graph(ctx):
    """convect_async recorded into the caller's own CUDA graph (torch
    capture) and replayed matches a direct call."""
    import torch
    dev = torch.device("cuda", 0)
    s, T, q = G.make_config("c2", n=4096, seed=31)
    L, n = T.shape
    ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s, T, q))

    def outs():
        return (torch.zeros((L, n), dtype=torch.float64, device=dev), torch.zeros((L, n), dtype=torch.float64, device=dev),
                torch.zeros(n, dtype=torch.float64, device=dev), torch.zeros(n, dtype=torch.int64, device=dev),
                torch.zeros(n, dtype=torch.uint8, device=dev))
    do, so = outs(), outs()
    st = torch.cuda.Stream()
    ctx.convect_async(ds, dT, dq, do, so, stream=st)   # warm (workspace sized)
    ctx.check(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        ctx.convect_async(ds, dT, dq, do, so, stream=st)
    for t in do + so:
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    both_close(P.ColumnOutputs(*[t.cpu().numpy() for t in do]), O.convection("deep", s, T, q))
    both_close(P.ColumnOutputs(*[t.cpu().numpy() for t in so]), O.convection("shallow", s, T, q))


def test_async_argument_validation(ctx):
    """convect_async checks devices, dtypes, shapes and strides before the
    kernels see a pointer (a wrong pitch would read out of bounds)."""
    import torch
    dev = torch.device("cuda", 0)
    s, T, q = G.make_config("c1", n=256, seed=3)
    L, n = T.shape
    ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s, T, q))

    def outs(dt=torch.float64):
        return (torch.empty((L, n), dtype=dt, device=dev), torch.empty((L, n), dtype=torch.float64, device=dev),
                torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.int64, device=dev),
                torch.empty(n, dtype=torch.uint8, device=dev))
    do, so = outs(), outs()
    bad_cases = [
        (ds.cpu(), dT, dq, do, so),                               # host tensor
        (ds.float(), dT, dq, do, so),                             # dtype
        (ds, dT.t().contiguous().t(), dq, do, so),                # column stride != 1
        (ds, dT, torch.empty((L, 2 * n), dtype=torch.float64, device=dev)[:, :n], do, so),   # q pitch != T pitch
        (ds, dT, dq, outs(torch.float32), so),                    # output dtype
        (ds, dT, dq, do, so[:4] + (torch.empty(n, dtype=torch.int8, device=dev),)),          # exited dtype
    ]
    for args in bad_cases:
        with pytest.raises(ValueError):
            ctx.convect_async(*args)
    ctx.convect_async(ds, dT, dq, do, so)
    ctx.check()


def test_check_reports_a_failure_once(ctx):
    import torch
    dev = torch.device("cuda", 0)
    s, T, q = G.make_config("c1", n=512, seed=8)
    L, n = T.shape
    ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s, T, q))
    outs = lambda: (torch.empty((L, n), dtype=torch.float64, device=dev),   # noqa: E731
                    torch.empty((L, n), dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                    torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.uint8, device=dev))
    ds[40] = float("inf")
    ctx.convect_async(ds, dT, dq, outs(), outs())
    with pytest.raises(P.KernelError) as e:
        ctx.check()
    assert e.value.column == 40
    st = ctx.check()   # reported once
    assert st.failing_column == 0 and st.n_columns == 0


def test_capture_refuses_workspace_growth():
    """A call captured into a caller's graph must not allocate: on a fresh
    context the first (larger) call inside a capture is refused with
    CVG_ERR_INVALID, and the context keeps working."""
    import torch
    from conftest import env_context
    c = env_context(CVG_GRAPH="1")
    dev = torch.device("cuda", 0)
    s, T, q = G.make_config("c2", n=8192, seed=12)
    L, n = T.shape
    ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s, T, q))
    outs = lambda: (torch.zeros((L, n), dtype=torch.float64, device=dev),   # noqa: E731
                    torch.zeros((L, n), dtype=torch.float64, device=dev), torch.zeros(n, dtype=torch.float64, device=dev),
                    torch.zeros(n, dtype=torch.int64, device=dev), torch.zeros(n, dtype=torch.uint8, device=dev))
    do, so = outs(), outs()
    st = torch.cuda.Stream()
    refused = False
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            try:
                c.convect_async(ds, dT, dq, do, so, stream=st)
            except ValueError as e:
                refused = "capture" in str(e)
    except RuntimeError:
        pass   # torch may reject the empty capture
    assert refused
    torch.cuda.synchronize()
    c.convect_async(ds, dT, dq, do, so, stream=st)   # uncaptured: sizes the workspace
    c.check(st)
    both_close(P.ColumnOutputs(*[t.cpu().numpy() for t in do]), O.convection("deep", s, T, q))
    c.close()


@pytest.mark.parametrize("env", [{}, {"CVG_DEEP_LPC": "2"}, {"CVG_DEEP_TPC": "1"}, {"CVG_DEEP_LPC": "0", "CVG_DEEP_TPC": "0"},
                                 {"CVG_REDO_INLINE": "0"}, {"CVG_OVERLAP": "0"}, {"CVG_SHALLOW_TILE": "2"},
                                 {"CVG_PDL": "0"}],
                         ids=["default", "lpc2", "tpc", "warp", "redo_kernel", "serial", "tile_plain_loads", "no_pdl"])
@pytest.mark.parametrize("variant,strict", [(0, False), (1, False), (2, False), (0, True)])
def test_writes_stay_in_bounds_and_cover_outputs(env, variant, strict):
    """Canary check (compute-sanitizer is unavailable on this pool): every
    buffer sits inside a larger allocation filled with a sentinel -- a row
    pitch wider than n and guard rows / elements on both sides.  After the
    call the inputs are bit-identical, every output element inside the
    region was written (no sentinel left), and nothing outside it changed."""
    import torch
    from conftest import env_context
    c = env_context(**env)
    dev = torch.device("cuda", 0)
    n, L, pad = 1000 + 37, 30, 24          # ragged n (last group partial), pitch n + pad
    s, T, q = G.make_config("c1", n=n, seed=44)
    ld = n + pad
    SENT = float.fromhex("0x1.dead0beefp+1000")

    def rows(x=None):
        base = torch.full((L + 2, ld), SENT, dtype=torch.float64, device=dev)
        if x is not None:
            base[1:L + 1, :n] = torch.from_numpy(x)
        return base, base[1:L + 1, :n]

    def vec(dtype, x=None, fill=SENT):
        base = torch.full((n + 2 * pad,), fill, dtype=dtype, device=dev) if dtype == torch.float64 else \
            torch.full((n + 2 * pad,), 123, dtype=dtype, device=dev)
        if x is not None:
            base[pad:pad + n] = torch.from_numpy(x)
        return base, base[pad:pad + n]

    sb, sv = vec(torch.float64, s)
    Tb, Tv = rows(T)
    qb, qv = rows(q)
    ins = [t.clone() for t in (sb, Tb, qb)]
    bufs, outs = [], []
    for _ in range(2):
        tTb, tTv = rows()
        tqb, tqv = rows()
        pb, pv = vec(torch.float64)
        wb, wv = vec(torch.int64)
        xb, xv = vec(torch.uint8)
        bufs.append((tTb, tqb, pb, wb, xb))
        outs.append((tTv, tqv, pv, wv, xv))
    o = P.KernelOptions(variant=variant, strict=strict)
    c.convect_async(sv, Tv, qv, outs[0], outs[1], o)
    c.check()
    for a, b in zip(ins, (sb, Tb, qb)):
        assert torch.equal(a.view(torch.int64) if a.dtype == torch.float64 else a,
                           b.view(torch.int64) if b.dtype == torch.float64 else b), "an input was modified"
    for (tTb, tqb, pb, wb, xb), (tTv, tqv, pv, wv, xv) in zip(bufs, outs):
        for b, v in ((tTb, tTv), (tqb, tqv)):
            assert not (v == SENT).any(), "an output element was not written"
            mask = torch.ones_like(b, dtype=torch.bool)
            mask[1:L + 1, :n] = False
            assert (b[mask] == SENT).all(), "a write outside the [L][n] region (pitch gap or guard rows)"
        assert not (pv == SENT).any() and (pb[:pad] == SENT).all() and (pb[pad + n:] == SENT).all()
        for b in (wb, xb):
            assert (b[:pad] == 123).all() and (b[pad + n:] == 123).all(), "a write before / after a vector"
    od = O.convection("deep", s, T, q, O.Options(variant=variant))
    assert np.array_equal(outs[0][3].cpu().numpy(), od.work)
    c.close()


@pytest.mark.parametrize("n,pad", [(1037, 3), (4096 + 5, 27), (2048, 0), (31, 1)])
@pytest.mark.parametrize("variant,strict", [(0, False), (1, False), (2, False), (0, True)])
def test_tiled_shallow_kernel_matches_thread_per_column(n, pad, variant, strict):
    """shallow_tile_kernel forced at small sizes (default from 32k columns):
    TMA- and cp.async-staged tiles on aligned rows (even pitch), plain loads on
    an odd pitch, ragged last tiles; outputs bit-identical to the thread-per-column
    kernel's (same column code) and within the parity rule of the oracle."""
    import torch
    from conftest import env_context
    dev = torch.device("cuda", 0)
    L = 30
    s, T, q = G.make_config("c1", n=n, seed=45)
    ld = n + pad
    o = P.KernelOptions(variant=variant, strict=strict)
    got = []
    for env in ({"CVG_SHALLOW_TILE": "2"}, {"CVG_SHALLOW_TILE": "0"}, {"CVG_SHALLOW_TILE": "2", "CVG_TILE_TMA": "0"}):
        c = env_context(**env)
        ds = torch.from_numpy(s).to(dev)
        Tb = torch.zeros((L, ld), dtype=torch.float64, device=dev)
        qb = torch.zeros((L, ld), dtype=torch.float64, device=dev)
        Tb[:, :n] = torch.from_numpy(T)
        qb[:, :n] = torch.from_numpy(q)
        outs = [(torch.zeros((L, ld), dtype=torch.float64, device=dev)[:, :n],
                 torch.zeros((L, ld), dtype=torch.float64, device=dev)[:, :n],
                 torch.zeros(n, dtype=torch.float64, device=dev), torch.zeros(n, dtype=torch.int64, device=dev),
                 torch.zeros(n, dtype=torch.uint8, device=dev)) for _ in range(2)]
        c.convect_async(ds, Tb[:, :n], qb[:, :n], outs[0], outs[1], o)
        c.check()
        got.append([P.ColumnOutputs(*[t.cpu().numpy() for t in oo]) for oo in outs])
        c.close()
    for other in got[1:]:   # TMA tiles == thread-per-column == cp.async tiles
        for a, b in zip(got[0], other):
            for f in ("tend_T", "tend_q", "precip", "work_units", "exited_early"):
                x, y = getattr(a, f), getattr(b, f)
                assert np.array_equal(x.view(np.int64) if x.dtype == np.float64 else x,
                                      y.view(np.int64) if y.dtype == np.float64 else y), f
    oo = O.Options(variant=variant)
    both_close(got[0][0], O.convection("deep", s, T, q, oo))
    both_close(got[0][1], O.convection("shallow", s, T, q, oo))


@pytest.mark.parametrize("L", [1, 7, 33, 40])
def test_tiled_shallow_kernel_level_counts(L):
    """Tile stages scale with L (2 L rows of 256 bytes per warp); L = 40 does
    not fit beside the deep block and falls back to the thread-per-column
    kernel even when forced."""
    from conftest import env_context
    import torch
    dev = torch.device("cuda", 0)
    n = 3000 + 12   # even row pitch (cp.async path), ragged last tile
    s, T, q = G.make_config("ref", n=n, L=L, seed=L + 100)
    c = env_context(CVG_SHALLOW_TILE="2")
    ds, dT, dq = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (s, T, q))
    outs = [(torch.zeros((L, n), dtype=torch.float64, device=dev), torch.zeros((L, n), dtype=torch.float64, device=dev),
             torch.zeros(n, dtype=torch.float64, device=dev), torch.zeros(n, dtype=torch.int64, device=dev),
             torch.zeros(n, dtype=torch.uint8, device=dev)) for _ in range(2)]
    c.convect_async(ds, dT, dq, outs[0], outs[1])
    c.check()
    assert ("shallow_tile_kernel" in c.last_shallow_kernel) == (L <= 36)
    both_close(P.ColumnOutputs(*[t.cpu().numpy() for t in outs[0]]), O.convection("deep", s, T, q))
    both_close(P.ColumnOutputs(*[t.cpu().numpy() for t in outs[1]]), O.convection("shallow", s, T, q))
    c.close()


@pytest.mark.parametrize("variant,strict", [(0, False), (2, False), (0, True)])
def test_tiled_shallow_kernel_alone(variant, strict):
    """Shallow-only calls run the tiled kernel alone on the SM (12 warps per
    block, no deep zero-fill): forced at a small ragged size, bit-identical
    to the thread-per-column kernel; deep outputs are not touched."""
    import torch
    from conftest import env_context
    dev = torch.device("cuda", 0)
    n, L = 5000 + 6, 30
    s, T, q = G.make_config("c1", n=n, seed=46)
    o = P.KernelOptions(variant=variant, strict=strict)
    got = []
    for env in ({"CVG_SHALLOW_TILE": "2"}, {"CVG_SHALLOW_TILE": "0"}):
        c = env_context(**env)
        ds, dT, dq = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (s, T, q))
        outs = [(torch.full((L, n), 7.0, dtype=torch.float64, device=dev), torch.full((L, n), 7.0, dtype=torch.float64, device=dev),
                 torch.full((n,), 7.0, dtype=torch.float64, device=dev), torch.full((n,), 7, dtype=torch.int64, device=dev),
                 torch.full((n,), 7, dtype=torch.uint8, device=dev)) for _ in range(2)]
        c.convect_async(ds, dT, dq, outs[0], outs[1], o, P.SHALLOW)
        c.check()
        assert ("shallow_tile_kernel<warps=12" in c.last_shallow_kernel) == (env["CVG_SHALLOW_TILE"] == "2")
        assert all(bool((t == 7).all()) for t in outs[0]), "a shallow-only call wrote a deep output"
        got.append(P.ColumnOutputs(*[t.cpu().numpy() for t in outs[1]]))
        c.close()
    for f in ("tend_T", "tend_q", "precip", "work_units", "exited_early"):
        x, y = getattr(got[0], f), getattr(got[1], f)
        assert np.array_equal(x.view(np.int64) if x.dtype == np.float64 else x,
                              y.view(np.int64) if y.dtype == np.float64 else y), f
    both_close(got[0], O.convection("shallow", s, T, q, O.Options(variant=variant)))


@pytest.mark.parametrize("mode", ["0", "1", "2", "3"])
@pytest.mark.parametrize("variant,strict", [(0, False), (2, False), (0, True)])
def test_deep_only_schedules(mode, variant, strict):
    """Deep-only calls (cvg_deep_convection): every schedule of the zero-fill
    -- beside a 16-warp deep block, after two 16-warp blocks, beside the
    21-warp block, and the persistent deep_zero_kernel beside a 28-warp block
    (default from 400k columns, forced here) -- writes every deep output,
    nothing else, and matches the oracle."""
    import torch
    from conftest import env_context
    dev = torch.device("cuda", 0)
    n, L = 3000 + 17, 30
    s, T, q = G.make_config("c1", n=n, seed=47)
    c = env_context(CVG_DEEP_ONLY=mode)
    ds, dT, dq = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (s, T, q))
    SENT = 12345.0
    outs = [(torch.full((L, n), SENT, dtype=torch.float64, device=dev), torch.full((L, n), SENT, dtype=torch.float64, device=dev),
             torch.full((n,), SENT, dtype=torch.float64, device=dev), torch.full((n,), 7, dtype=torch.int64, device=dev),
             torch.full((n,), 7, dtype=torch.uint8, device=dev)) for _ in range(2)]
    c.convect_async(ds, dT, dq, outs[0], outs[1], P.KernelOptions(variant=variant, strict=strict), P.DEEP)
    c.check()
    if mode == "3":
        assert "deep_zero_kernel" in c.last_shallow_kernel and "warps=28" in c.last_deep_kernel
    assert not any(bool((t == SENT).any()) for t in outs[0][:3]), "a deep output element was not written"
    assert all(bool((t == SENT).all()) for t in outs[1][:3]) and bool((outs[1][3] == 7).all()), \
        "a deep-only call wrote a shallow output"
    od = O.convection("deep", s, T, q, O.Options(variant=variant))
    got = P.ColumnOutputs(*[t.cpu().numpy() for t in outs[0]])
    both_close(got, od)
    assert np.array_equal(got.work_units, od.work)
    c.close()
