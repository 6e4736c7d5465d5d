"""TEST INFRASTRUCTURE ONLY: ctypes bindings to the parity checkers.

* ``liboracle.so``   -- C restatement of the reference column physics
  (oracle/convproxy_oracle.c, each function cites physics.cpp lines).
* ``_ref/libconvref.so`` -- the reference's own physics.cpp/sched.cpp compiled
  in place from /root/reference by oracle/Makefile (absent if the build
  container had no reference tree).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(paper_1711_00289_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libconvref.so")

EXACT, STRENGTH_REDUCED, APPROX_TRANSCENDENTAL = 0, 1, 2
FAIL_NAMES = {0: "ok", 1: "non-finite activity", 2: "non-finite input",
              3: "iterate diverged", 4: "no convergence"}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class Options(C.Structure):
    """Mirrors convproxy::KernelOptions (physics.hpp:68-73)."""
    _fields_ = [("variant", C.c_int), ("activity_threshold", C.c_double),
                ("newton_tol", C.c_double), ("newton_max_iter", C.c_int)]

    def __init__(self, variant=EXACT, activity_threshold=0.5, newton_tol=1e-12,
                 newton_max_iter=100):
        super().__init__(variant, activity_threshold, newton_tol, newton_max_iter)


_orc = None
_ref = None


def lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle library missing: {ORACLE_SO} (run make -C oracle)")
        L = C.CDLL(ORACLE_SO)
        L.orc_rng_u64.restype = C.c_uint64
        L.orc_rng_u64.argtypes = [C.c_uint64] * 3
        L.orc_rng_u01.restype = C.c_double
        L.orc_rng_u01.argtypes = [C.c_uint64] * 3
        L.orc_approx_exp.restype = C.c_double
        L.orc_approx_exp.argtypes = [C.c_double]
        L.orc_ientropy_solve.restype = C.c_int
        L.orc_ientropy_solve.argtypes = [C.c_double, C.c_double, C.POINTER(Options),
                                         C.POINTER(C.c_double), C.POINTER(C.c_int),
                                         C.POINTER(C.c_double)]
        for name in ("orc_deep_convection", "orc_shallow_convection"):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = [C.c_longlong, C.c_int, C.c_longlong, C.c_longlong,
                          _dp, _dp, _dp, C.POINTER(Options), _dp, _dp, _dp, _i64p,
                          _u8p, _dp, C.POINTER(C.c_longlong)]
        for name in ("orc_exp_gl_vec", "orc_libm_exp_vec"):
            f = getattr(L, name)
            f.restype = None
            f.argtypes = [C.c_longlong, _dp, _dp]
        L.orc_exp_gl.restype = C.c_double
        L.orc_exp_gl.argtypes = [C.c_double]
        L.orc_make_grid.restype = None
        L.orc_make_grid.argtypes = [C.c_longlong, C.c_int, C.c_double, C.c_uint64,
                                    _dp, _dp, _dp]
        _orc = L
    return _orc


def exp_gl(x) -> np.ndarray:
    """The restatement of glibc's exp (orc_exp_gl) over an array."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().orc_exp_gl_vec(x.size, x, out)
    return out


def libm_exp(x) -> np.ndarray:
    """The running libm's exp (what the reference calls, physics.cpp:35)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().orc_libm_exp_vec(x.size, x, out)
    return out


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference build missing: {REF_SO}")
        L = C.CDLL(REF_SO)
        L.ref_convection.restype = C.c_int
        L.ref_convection.argtypes = [C.c_int, C.c_longlong, C.c_int, C.c_longlong,
                                     C.c_longlong, _dp, _dp, _dp, C.c_int, C.c_double,
                                     C.c_double, C.c_int, _dp, _dp, _dp, _i64p, _u8p,
                                     C.POINTER(C.c_longlong)]
        L.ref_ientropy_solve.restype = C.c_int
        L.ref_ientropy_solve.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double,
                                         C.c_int, C.POINTER(C.c_double),
                                         C.POINTER(C.c_int)]
        L.ref_approx_exp.restype = C.c_double
        L.ref_approx_exp.argtypes = [C.c_double]
        L.ref_make_grid.restype = None
        L.ref_make_grid.argtypes = [C.c_longlong, C.c_int, C.c_double, C.c_ulonglong,
                                    _dp, _dp, _dp]
        L.ref_chunk_create.restype = C.c_void_p
        L.ref_chunk_create.argtypes = [C.c_longlong, C.c_int, C.c_longlong,
                                       C.c_longlong, _dp, _dp, _dp]
        L.ref_chunk_free.restype = None
        L.ref_chunk_free.argtypes = [C.c_void_p]
        L.ref_run_parallel.restype = C.c_int
        L.ref_run_parallel.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double,
                                       C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(C.c_double), C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_packed_bytes.restype = C.c_int
        L.ref_packed_bytes.argtypes = [C.c_longlong, C.c_int, C.c_int, C.POINTER(C.c_longlong),
                                       C.POINTER(C.c_longlong)]
        L.ref_records_roundtrip.restype = C.c_int
        L.ref_records_roundtrip.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ref_error_growth.restype = C.c_int
        L.ref_error_growth.argtypes = [C.c_int, C.c_longlong, C.c_int, _dp, _dp, _dp, C.c_int, C.c_int,
                                       C.c_double, C.c_double, C.c_int, C.c_int, _dp, _dp,
                                       C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int)]
        _ref = L
    return _ref


class Result:
    """SoA outputs of one kernel pass (level-major [L][n])."""

    def __init__(self, n, L):
        self.tend_T = np.zeros((L, n))
        self.tend_q = np.zeros((L, n))
        self.precip = np.zeros(n)
        self.work = np.zeros(n, dtype=np.int64)
        self.exited = np.zeros(n, dtype=np.uint8)
        self.margin = np.full(n, np.inf)
        self.status = 0
        self.fail_col = -1


def _soa(s, T, q):
    s = np.ascontiguousarray(s, dtype=np.float64)
    T = np.ascontiguousarray(T, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    assert T.shape == q.shape and T.shape[1] == s.shape[0]
    return s, T, q


def convection(kernel: str, s, T, q, opts: Options | None = None, first_col=0) -> Result:
    """Oracle pass: kernel in {"deep", "shallow"}; returns Result (with the
    Newton / predicate margin diagnostics in ``margin``)."""
    opts = opts or Options()
    s, T, q = _soa(s, T, q)
    L, n = T.shape
    r = Result(n, L)
    fc = C.c_longlong(-1)
    f = lib().orc_deep_convection if kernel == "deep" else lib().orc_shallow_convection
    r.status = f(n, L, n, first_col, s, T, q, C.byref(opts), r.tend_T, r.tend_q,
                 r.precip, r.work, r.exited, r.margin, C.byref(fc))
    r.fail_col = fc.value
    return r


def convection_mt(kernel: str, s, T, q, opts: Options | None = None, first_col=0, threads=None) -> Result:
    """convection() over column chunks on host threads (ctypes releases the
    GIL; columns are independent, physics.hpp:26-30): the same Result, bit
    for bit, in a fraction of the wall time on large grids.  The failure is
    the lowest failing column over the chunks (the serial driver's)."""
    from concurrent.futures import ThreadPoolExecutor
    opts = opts or Options()
    s, T, q = _soa(s, T, q)
    L, n = T.shape
    threads = threads or min(32, os.cpu_count() or 1)
    if n < 4096 or threads <= 1:
        return convection(kernel, s, T, q, opts, first_col)
    bounds = np.linspace(0, n, 4 * threads + 1).astype(np.int64)
    r = Result(n, L)

    def run(i):
        a, b = int(bounds[i]), int(bounds[i + 1])
        part = convection(kernel, s[a:b], np.ascontiguousarray(T[:, a:b]), np.ascontiguousarray(q[:, a:b]),
                          opts, first_col + a)
        r.tend_T[:, a:b], r.tend_q[:, a:b] = part.tend_T, part.tend_q
        r.precip[a:b], r.work[a:b], r.exited[a:b], r.margin[a:b] = part.precip, part.work, part.exited, part.margin
        return part.status, part.fail_col

    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(run, range(len(bounds) - 1)))
    for st, fc in res:
        if st != 0:
            r.status, r.fail_col = st, fc
            break
    return r


def ref_convection(kernel: str, s, T, q, opts: Options | None = None, first_col=0) -> Result:
    """The reference's own deep_convection/shallow_convection (physics.hpp:155-158)."""
    opts = opts or Options()
    s, T, q = _soa(s, T, q)
    L, n = T.shape
    r = Result(n, L)
    fc = C.c_longlong(-1)
    r.status = ref_lib().ref_convection(0 if kernel == "deep" else 1, n, L, n, first_col,
                                        s, T, q, opts.variant, opts.activity_threshold,
                                        opts.newton_tol, opts.newton_max_iter, r.tend_T,
                                        r.tend_q, r.precip, r.work, r.exited, C.byref(fc))
    r.fail_col = fc.value
    return r


def ientropy_solve(y, guess, opts: Options | None = None):
    opts = opts or Options()
    root, it, mm = C.c_double(), C.c_int(), C.c_double()
    st = lib().orc_ientropy_solve(y, guess, C.byref(opts), C.byref(root), C.byref(it),
                                  C.byref(mm))
    return st, root.value, it.value, mm.value


def make_grid(n, L=30, tropics_band=0.3, seed=42):
    s = np.empty(n)
    T = np.empty((L, n))
    q = np.empty((L, n))
    lib().orc_make_grid(n, L, tropics_band, seed, s, T, q)
    return s, T, q


def ref_make_grid(n, L=30, tropics_band=0.3, seed=42):
    s = np.empty(n)
    T = np.empty((L, n))
    q = np.empty((L, n))
    ref_lib().ref_make_grid(n, L, tropics_band, seed, s, T, q)
    return s, T, q


def ref_run_parallel(kernel: str, s, T, q, opts: Options | None = None, n_threads=None, strategy=2, omp_chunk=1):
    """The reference's run_parallel (sched.hpp:73-74) with its outputs:
    (Result, wall seconds)."""
    opts = opts or Options()
    s, T, q = _soa(s, T, q)
    L, n = T.shape
    n_threads = n_threads or os.cpu_count() or 1
    R = ref_lib()
    h = R.ref_chunk_create(n, L, n, 0, s, T, q)
    if not h:
        raise RuntimeError("ref_chunk_create failed")
    try:
        r = Result(n, L)
        w = C.c_double()
        r.status = R.ref_run_parallel(h, 0 if kernel == "deep" else 1, opts.variant, opts.activity_threshold,
                                      opts.newton_tol, opts.newton_max_iter, n_threads, strategy, omp_chunk,
                                      C.byref(w), r.tend_T.ctypes.data, r.tend_q.ctypes.data, r.precip.ctypes.data,
                                      r.work.ctypes.data, r.exited.ctypes.data)
        return r, w.value
    finally:
        R.ref_chunk_free(h)


def ref_time_run_parallel(s, T, q, opts: Options | None = None, n_threads=None,
                          strategy=2, omp_chunk=1, kernels=("deep", "shallow")):
    """Wall seconds of the reference run_parallel over the sample, one entry
    per kernel (reference RunMetrics::wall_s, sched.cpp:196-201)."""
    opts = opts or Options()
    s, T, q = _soa(s, T, q)
    L, n = T.shape
    n_threads = n_threads or os.cpu_count() or 1
    R = ref_lib()
    h = R.ref_chunk_create(n, L, n, 0, s, T, q)
    if not h:
        raise RuntimeError("ref_chunk_create failed")
    try:
        out = {}
        for k in kernels:
            w = C.c_double()
            st = R.ref_run_parallel(h, 0 if k == "deep" else 1, opts.variant,
                                    opts.activity_threshold, opts.newton_tol,
                                    opts.newton_max_iter, n_threads, strategy, omp_chunk,
                                    C.byref(w), None, None, None, None, None)
            if st != 0:
                raise RuntimeError(f"reference run_parallel failed ({st})")
            out[k] = w.value
        return out
    finally:
        R.ref_chunk_free(h)


class GrowthSeries:
    """ErrorGrowthSeries (validate.hpp:64-69) plus the call's status: 0 ok,
    3 KernelError, 4 ValidationError (fail_step = the failing timestep)."""

    def __init__(self, steps):
        self.rms_mod = np.zeros(steps)
        self.rms_pert = np.zeros(steps)
        self.envelope_ok = True
        self.worst_ratio = 0.0
        self.status = 0
        self.fail_step = -1


def ref_error_growth(kernel: str, s, T, q, base_variant=EXACT, mod_variant=EXACT, timesteps=50,
                     opts: Options | None = None) -> GrowthSeries:
    """The reference's own error_growth (validate.cpp:168-206) on a SoA grid:
    baseline / modified variants, serial StaticBlock paths."""
    opts = opts or Options()
    s, T, q = _soa(s, T, q)
    L, n = T.shape
    g = GrowthSeries(timesteps)
    env, worst, fs = C.c_int(), C.c_double(), C.c_int(-1)
    g.status = ref_lib().ref_error_growth(0 if kernel == "deep" else 1, n, L, s, T, q, base_variant,
                                          mod_variant, opts.activity_threshold, opts.newton_tol,
                                          opts.newton_max_iter, timesteps, g.rms_mod, g.rms_pert,
                                          C.byref(env), C.byref(worst), C.byref(fs))
    g.envelope_ok, g.worst_ratio, g.fail_step = bool(env.value), worst.value, fs.value
    return g


def ref_packed_bytes(nd, L, send_scalars=True):
    """(bytes_in, bytes_out) of the reference's device staging for nd columns
    (hetero.cpp pack(), HeteroMetrics semantics)."""
    bi, bo = C.c_longlong(), C.c_longlong()
    if ref_lib().ref_packed_bytes(nd, L, int(send_scalars), C.byref(bi), C.byref(bo)) != 0:
        raise RuntimeError("ref_packed_bytes failed")
    return bi.value, bo.value


def ref_records_roundtrip(csv: str):
    """(status, n_records, text): the reference's records_from_csv then
    records_to_csv (bench.cpp:454-525); status 0 ok, 2 ConfigError."""
    n = C.c_int(0)
    buf = C.create_string_buffer(1 << 16)
    st = ref_lib().ref_records_roundtrip(csv.encode(), C.byref(n), buf, len(buf))
    return st, n.value, buf.value.decode()
