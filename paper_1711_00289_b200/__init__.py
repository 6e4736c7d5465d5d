"""B200-native (sm_100a) deep + shallow convection column path.

Python mirror of the reference's column-batch interface over the C ABI in
``include/convgpu.h`` (``libconvgpu.so``, built from ``csrc/``):

* ``deep_convection`` / ``shallow_convection``  <- physics.hpp:155-158
* ``ientropy_solve``                            <- physics.hpp:101
* ``approx_exp``                                <- physics.hpp:83
* ``KernelOptions`` / ``Variant``               <- physics.hpp:62-73
* ``KernelError`` (column id)                   <- errors.hpp:26-36
* ``plan_partition`` (G-way, count-balanced)    <- hetero.cpp:156-176

Columns travel as level-major structure-of-arrays: ``s[n]``, ``T[L][n]``,
``q[L][n]``.  There is no CPU fallback: if the CUDA library is missing or no
sm_100 device is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Variant", "KernelOptions", "KernelError", "DeviceError", "ValidationError", "ColumnOutputs", "Stats",
    "GrowthSeries",
    "Context", "deep_convection", "shallow_convection", "ientropy_solve", "approx_exp",
    "plan_partition", "library_path", "load_library", "DEEP", "SHALLOW", "BOTH", "MultiContext",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libconvgpu.so"
DEEP, SHALLOW, BOTH = 1, 2, 3


class Variant:
    """convproxy::Variant (physics.hpp:62-66)."""
    EXACT = 0
    STRENGTH_REDUCED = 1
    APPROX_TRANSCENDENTAL = 2


FLAG_STRICT = 1
FLAG_NO_FAR32 = 2


class KernelOptions(C.Structure):
    """convproxy::KernelOptions (physics.hpp:68-73), same defaults, plus
    ``strict``: reference rounding in every Newton update (CVG_FLAG_STRICT);
    ``far32=False``: no FP32 far phase in the relaxed solve (CVG_FLAG_NO_FAR32)."""
    _fields_ = [("variant", C.c_int), ("activity_threshold", C.c_double),
                ("newton_tol", C.c_double), ("newton_max_iter", C.c_int), ("flags", C.c_int)]

    def __init__(self, variant=Variant.EXACT, activity_threshold=0.5, newton_tol=1e-12,
                 newton_max_iter=100, strict=False, far32=True):
        super().__init__(int(variant), float(activity_threshold), float(newton_tol),
                         int(newton_max_iter),
                         (FLAG_STRICT if strict else 0) | (0 if far32 else FLAG_NO_FAR32))

    def __repr__(self):
        return (f"KernelOptions(variant={self.variant}, activity_threshold={self.activity_threshold},"
                f" newton_tol={self.newton_tol}, newton_max_iter={self.newton_max_iter}, flags={self.flags})")


class _Columns(C.Structure):
    _fields_ = [("n_columns", C.c_longlong), ("n_levels", C.c_int), ("first_col", C.c_longlong),
                ("ld", C.c_longlong), ("s", C.c_void_p), ("T", C.c_void_p), ("q", C.c_void_p),
                ("on_device", C.c_int)]


class _Outputs(C.Structure):
    _fields_ = [("tend_T", C.c_void_p), ("tend_q", C.c_void_p), ("precip", C.c_void_p),
                ("work_units", C.c_void_p), ("exited_early", C.c_void_p), ("ld", C.c_longlong),
                ("on_device", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("n_columns", C.c_longlong), ("n_triggered", C.c_longlong),
                ("failing_column", C.c_longlong), ("failure_kind", C.c_int),
                ("failing_kernel", C.c_int), ("device_ms", C.c_double), ("h2d_ms", C.c_double),
                ("d2h_ms", C.c_double), ("h2d_bytes", C.c_longlong), ("d2h_bytes", C.c_longlong),
                ("n_recomputed", C.c_longlong), ("n_corrected", C.c_longlong)]


CVG_OK, CVG_ERR_INVALID, CVG_ERR_NUMERIC, CVG_ERR_CHECK, CVG_ERR_DEVICE = 0, 1, 3, 4, 6


class KernelError(RuntimeError):
    """Numeric failure in a column kernel; ``column`` is the lowest failing
    column id (what the serial reference would have thrown on)."""

    def __init__(self, msg, column=-1, kind=0):
        super().__init__(msg)
        self.column = column
        self.kind = kind


class DeviceError(RuntimeError):
    pass


class ValidationError(RuntimeError):
    """A validation check failed (CVG_ERR_CHECK; the reference's
    ValidationError, errors.hpp:58-70): a diverged feedback-loop state or a
    non-finite value handed to perturb_lsb.  ``timestep`` is the failing step
    (-1 when not applicable)."""

    def __init__(self, msg, timestep=-1):
        super().__init__(msg)
        self.timestep = timestep


class _Growth(C.Structure):
    _fields_ = [("envelope_ok", C.c_int), ("worst_ratio", C.c_double), ("failing_step", C.c_int)]


@dataclass
class GrowthSeries:
    """convproxy::ErrorGrowthSeries (validate.hpp:64-69)."""
    rms_mod: np.ndarray
    rms_pert: np.ndarray
    envelope_ok: bool
    worst_ratio: float


def library_path() -> str:
    return os.environ.get("CONVGPU_LIB", os.path.join(HERE, LIB_NAME))


_lib = None


def load_library():
    """Loads libconvgpu.so; raises (no fallback) if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not os.path.exists(path):
        raise DeviceError(f"CUDA library {path} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    vp, i64, i32, dbl = C.c_void_p, C.c_longlong, C.c_int, C.c_double
    L.cvg_version.restype = C.c_char_p
    L.cvg_last_error.restype = C.c_char_p
    if hasattr(L, "cvg_last_deep_kernel"):
        L.cvg_last_deep_kernel.restype = C.c_char_p
        L.cvg_last_deep_kernel.argtypes = [vp]
        L.cvg_last_shallow_kernel.restype = C.c_char_p
        L.cvg_last_shallow_kernel.argtypes = [vp]
    L.cvg_default_options.argtypes = [C.POINTER(KernelOptions)]
    L.cvg_context_create.argtypes = [i32, C.POINTER(vp)]
    L.cvg_context_free.argtypes = [vp]
    L.cvg_context_free.restype = None
    L.cvg_convect.argtypes = [vp, C.POINTER(_Columns), C.POINTER(KernelOptions), i32,
                              C.POINTER(_Outputs), C.POINTER(_Outputs), C.POINTER(Stats)]
    L.cvg_convect_async.argtypes = [vp, C.POINTER(_Columns), C.POINTER(KernelOptions), i32,
                                    C.POINTER(_Outputs), C.POINTER(_Outputs), vp]
    L.cvg_convect_check.argtypes = [vp, vp, C.POINTER(Stats)]
    L.cvg_deep_convection.argtypes = [vp, C.POINTER(_Columns), C.POINTER(KernelOptions),
                                      C.POINTER(_Outputs), C.POINTER(Stats)]
    L.cvg_shallow_convection.argtypes = L.cvg_deep_convection.argtypes
    L.cvg_ientropy_solve.argtypes = [vp, i64, vp, vp, C.POINTER(KernelOptions), vp, vp]
    L.cvg_approx_exp.argtypes = [vp, i64, vp, vp]
    if hasattr(L, "cvg_exp"):   # (absent only in pre-0.3 builds used for A/B timing)
        L.cvg_exp.argtypes = [vp, i64, vp, vp]
        L.cvg_exp.restype = C.c_int
    L.cvg_plan_partition.argtypes = [i64, vp, dbl, i32, dbl, dbl, vp]
    L.cvg_profile_begin.argtypes = [vp, i32]
    L.cvg_profile_end.argtypes = [vp, C.POINTER(C.c_int), vp, i32]
    L.cvg_fp64_peak.argtypes = [vp, i32, C.POINTER(C.c_double)]
    L.cvg_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.cvg_host_free.argtypes = [vp]
    L.cvg_host_free.restype = None
    L.cvg_timestep.argtypes = [vp, i64, i32, i64, vp, vp, vp, i32, C.POINTER(KernelOptions), i32, i32,
                               C.POINTER(Stats)]
    L.cvg_multi_create.argtypes = [C.POINTER(C.c_int), i32, C.POINTER(vp)]
    L.cvg_multi_free.argtypes = [vp]
    L.cvg_multi_free.restype = None
    L.cvg_multi_size.argtypes = [vp]
    L.cvg_multi_size.restype = C.c_int
    L.cvg_multi_context.argtypes = [vp, i32]
    L.cvg_multi_context.restype = vp
    L.cvg_multi_set_weights.argtypes = [vp, dbl, dbl]
    L.cvg_multi_convect.argtypes = [vp, C.POINTER(_Columns), C.POINTER(KernelOptions), i32, C.POINTER(_Outputs),
                                    C.POINTER(_Outputs), C.POINTER(Stats), vp]
    L.cvg_error_growth.argtypes = [vp, C.POINTER(_Columns), i32, C.POINTER(KernelOptions),
                                   C.POINTER(KernelOptions), i32, vp, vp, C.POINTER(_Growth)]
    for f in ("cvg_profile_begin", "cvg_profile_end", "cvg_fp64_peak", "cvg_host_alloc",
              "cvg_context_create", "cvg_convect", "cvg_convect_async", "cvg_convect_check",
              "cvg_deep_convection", "cvg_shallow_convection", "cvg_ientropy_solve",
              "cvg_approx_exp", "cvg_plan_partition", "cvg_timestep", "cvg_error_growth",
              "cvg_multi_create", "cvg_multi_set_weights", "cvg_multi_convect"):
        getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _raise(rc, stats: Stats | None = None):
    if rc == CVG_OK:
        return
    msg = load_library().cvg_last_error().decode()
    if rc == CVG_ERR_NUMERIC:
        col = stats.failing_column if stats is not None else -1
        kind = stats.failure_kind if stats is not None else 0
        raise KernelError(msg, col, kind)
    if rc == CVG_ERR_DEVICE:
        raise DeviceError(msg)
    if rc == CVG_ERR_CHECK:
        raise ValidationError(msg)
    raise ValueError(f"convgpu status {rc}: {msg}")


@dataclass
class ColumnOutputs:
    """SoA form of std::vector<ColumnOutput> (physics.hpp:52-60)."""
    tend_T: np.ndarray   # [L][n]
    tend_q: np.ndarray   # [L][n]
    precip: np.ndarray   # [n]
    work_units: np.ndarray  # [n] int64
    exited_early: np.ndarray  # [n] uint8

    @classmethod
    def empty(cls, n, L):
        return cls(np.empty((L, n)), np.empty((L, n)), np.empty(n), np.empty(n, np.int64),
                   np.empty(n, np.uint8))

    def _struct(self):
        return _Outputs(self.tend_T.ctypes.data, self.tend_q.ctypes.data, self.precip.ctypes.data,
                        self.work_units.ctypes.data, self.exited_early.ctypes.data,
                        self.tend_T.shape[1] if self.tend_T.ndim == 2 else 0, 0)


def _host_columns(s, T, q, first_col):
    s = np.ascontiguousarray(s, dtype=np.float64)
    T = np.ascontiguousarray(T, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    if T.ndim != 2 or T.shape != q.shape or T.shape[1] != s.shape[0]:
        raise ValueError("expected s[n], T[L][n], q[L][n]")
    L, n = T.shape
    return (s, T, q), _Columns(n, L, first_col, n, s.ctypes.data, T.ctypes.data, q.ctypes.data, 0)


class Context:
    """One device context (cvg_context): persistent workspace, one call in
    flight.  Use one per GPU / per rank."""

    def __init__(self, device: int = 0):
        L = load_library()
        h = C.c_void_p()
        _raise(L.cvg_context_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self.last_stats = Stats()

    def close(self):
        if getattr(self, "_h", None):
            load_library().cvg_context_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- host (numpy) entry points -------------------------------------------
    def convect(self, s, T, q, opts: KernelOptions | None = None, kernels=BOTH, first_col=0,
                out_deep: ColumnOutputs | None = None, out_shallow: ColumnOutputs | None = None):
        """Runs deep and/or shallow over host SoA arrays; returns (deep, shallow)
        ColumnOutputs (None for a kernel not requested).  Preallocated (e.g.
        pinned) output buffers may be passed in."""
        opts = opts or KernelOptions()
        keep, cols = _host_columns(s, T, q, first_col)
        L, n = keep[1].shape
        deep = (out_deep or ColumnOutputs.empty(n, L)) if kernels & DEEP else None
        sh = (out_shallow or ColumnOutputs.empty(n, L)) if kernels & SHALLOW else None
        st = Stats()
        rc = load_library().cvg_convect(self._h, C.byref(cols), C.byref(opts), kernels,
                                        C.byref(deep._struct()) if deep else None,
                                        C.byref(sh._struct()) if sh else None, C.byref(st))
        self.last_stats = st
        _raise(rc, st)
        return deep, sh

    def deep_convection(self, s, T, q, opts=None, first_col=0) -> ColumnOutputs:
        return self.convect(s, T, q, opts, DEEP, first_col)[0]

    def shallow_convection(self, s, T, q, opts=None, first_col=0) -> ColumnOutputs:
        return self.convect(s, T, q, opts, SHALLOW, first_col)[1]

    def ientropy_solve(self, y, guess, opts: KernelOptions | None = None):
        opts = opts or KernelOptions()
        y = np.ascontiguousarray(np.atleast_1d(y), dtype=np.float64)
        g = np.ascontiguousarray(np.broadcast_to(np.asarray(guess, dtype=np.float64), y.shape))
        root = np.empty_like(y)
        it = np.empty(y.shape, dtype=np.int32)
        rc = load_library().cvg_ientropy_solve(self._h, y.size, y.ctypes.data, g.ctypes.data,
                                               C.byref(opts), root.ctypes.data, it.ctypes.data)
        _raise(rc)
        return root, it

    def approx_exp(self, x):
        x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float64)
        out = np.empty_like(x)
        _raise(load_library().cvg_approx_exp(self._h, x.size, x.ctypes.data, out.ctypes.data))
        return out

    def exp(self, x):
        """The Exact variant's exp_eval (physics.cpp:35) on the device:
        bit-identical to the libm exp the reference calls."""
        x = np.ascontiguousarray(np.atleast_1d(x), dtype=np.float64)
        out = np.empty_like(x)
        _raise(load_library().cvg_exp(self._h, x.size, x.ctypes.data, out.ctypes.data))
        return out

    # -- feedback loop (validate.cpp:113-206) ---------------------------------
    def timestep(self, s, T, q, opts: KernelOptions | None = None, kernel=DEEP, n_steps=1):
        """n_steps of the device-resident loop T += tend_T, q += tend_q with
        the deep (DEEP) or shallow (SHALLOW) kernel; returns the new (T, q)
        (host copies; the inputs are not modified)."""
        opts = opts or KernelOptions()
        s = np.ascontiguousarray(s, dtype=np.float64)
        T = np.array(T, dtype=np.float64, order="C", copy=True)
        q = np.array(q, dtype=np.float64, order="C", copy=True)
        L, n = T.shape
        st = Stats()
        rc = load_library().cvg_timestep(self._h, n, L, n, s.ctypes.data, T.ctypes.data, q.ctypes.data, 0,
                                         C.byref(opts), int(kernel), int(n_steps), C.byref(st))
        self.last_stats = st
        _raise(rc, st)
        return T, q

    def error_growth(self, s, T, q, kernel=DEEP, baseline: KernelOptions | None = None,
                     modified: KernelOptions | None = None, timesteps=50) -> GrowthSeries:
        """error_growth (validate.hpp:71-82) on the device: baseline, modified
        and LSB-perturbed legs; raises ValidationError (with .timestep) when a
        leg diverges."""
        baseline = baseline or KernelOptions()
        modified = modified or KernelOptions()
        keep, cols = _host_columns(s, T, q, 0)
        rm, rp = np.zeros(max(timesteps, 0)), np.zeros(max(timesteps, 0))
        g = _Growth()
        rc = load_library().cvg_error_growth(self._h, C.byref(cols), int(kernel), C.byref(baseline),
                                             C.byref(modified), int(timesteps), rm.ctypes.data, rp.ctypes.data,
                                             C.byref(g))
        if rc == CVG_ERR_CHECK:
            raise ValidationError(load_library().cvg_last_error().decode(), g.failing_step)
        _raise(rc)
        return GrowthSeries(rm, rp, bool(g.envelope_ok), g.worst_ratio)

    # -- device-resident entry points (torch CUDA tensors or raw pointers) ----
    def convect_async(self, s, T, q, deep, shallow, opts: KernelOptions | None = None,
                      kernels=BOTH, first_col=0, stream=None):
        """Enqueues on `stream` (a torch.cuda.Stream, raw handle or None for the
        context stream).  s/T/q and the output tuples are CUDA tensors
        (tend_T, tend_q, precip, work, exited)."""
        import torch
        opts = opts or KernelOptions()
        dev = torch.device("cuda", self.device)

        def need(cond, what):
            if not cond:
                raise ValueError(f"convect_async: {what}")

        def on_dev(t, dtype, name):
            need(isinstance(t, torch.Tensor) and t.is_cuda and t.device == dev, f"{name} must be a tensor on {dev}")
            need(t.dtype == dtype, f"{name} must be {dtype}")

        n = s.numel()
        on_dev(s, torch.float64, "s")
        need(s.dim() == 1 and s.stride(0) == 1, "s must be 1-D contiguous")
        for name, t in (("T", T), ("q", q)):
            on_dev(t, torch.float64, name)
            need(t.dim() == 2 and t.shape[1] == n and t.stride(1) == 1, f"{name} must be [L][n] with unit column stride")
        need(T.shape == q.shape and T.stride(0) == q.stride(0), "T and q must have the same shape and row pitch")
        L = T.shape[0]
        cols = _Columns(n, L, first_col, T.stride(0), s.data_ptr(), T.data_ptr(), q.data_ptr(), 1)

        def outs(o, name):
            if o is None:
                return None
            tT, tq, pr, wk, ex = o
            for nm, t in (("tend_T", tT), ("tend_q", tq)):
                on_dev(t, torch.float64, f"{name}.{nm}")
                need(t.dim() == 2 and tuple(t.shape) == (L, n) and t.stride(1) == 1,
                     f"{name}.{nm} must be [L][n] with unit column stride")
            need(tT.stride(0) == tq.stride(0), f"{name}: tend_T and tend_q must share a row pitch")
            for nm, t, dt in (("precip", pr, torch.float64), ("work_units", wk, torch.int64),
                              ("exited_early", ex, torch.uint8)):
                on_dev(t, dt, f"{name}.{nm}")
                need(t.dim() == 1 and t.numel() == n and t.stride(0) == 1, f"{name}.{nm} must be 1-D contiguous [n]")
            return C.byref(_Outputs(tT.data_ptr(), tq.data_ptr(), pr.data_ptr(), wk.data_ptr(),
                                    ex.data_ptr(), tT.stride(0), 1))

        h = None
        if stream is not None:
            h = getattr(stream, "cuda_stream", stream)
        rc = load_library().cvg_convect_async(self._h, C.byref(cols), C.byref(opts), kernels,
                                              outs(deep, "deep") if kernels & DEEP else None,
                                              outs(shallow, "shallow") if kernels & SHALLOW else None, h)
        _raise(rc)

    def profile_begin(self, max_steps: int):
        _raise(load_library().cvg_profile_begin(self._h, int(max_steps)))

    def profile_end(self, capacity: int = 4096) -> np.ndarray:
        """[n_steps][3] kernel durations (ms): trigger+compaction, deep, shallow."""
        buf = np.zeros((capacity, 3))
        n = C.c_int()
        _raise(load_library().cvg_profile_end(self._h, C.byref(n), buf.ctypes.data, capacity))
        return buf[: n.value].copy()

    @property
    def last_deep_kernel(self) -> str:
        """The deep kernel (and launch shape) of this context's last call."""
        return load_library().cvg_last_deep_kernel(self._h).decode()

    @property
    def last_shallow_kernel(self) -> str:
        """The shallow kernel of this context's last call."""
        return load_library().cvg_last_shallow_kernel(self._h).decode()

    def fp64_peak_tflops(self, reps: int = 5) -> float:
        v = C.c_double()
        _raise(load_library().cvg_fp64_peak(self._h, int(reps), C.byref(v)))
        return v.value

    def check(self, stream=None) -> Stats:
        st = Stats()
        h = None if stream is None else getattr(stream, "cuda_stream", stream)
        rc = load_library().cvg_convect_check(self._h, h, C.byref(st))
        self.last_stats = st
        _raise(rc, st)
        return st


class MultiContext:
    """Several device contexts driven as one (cvg_multi): a host-buffer call
    is split into contiguous column ranges balanced by estimated cost and
    run on every device concurrently (the reference's HeteroEngine::step,
    hetero.cpp:252-466, over G devices).  A device may be listed twice
    (independent contexts sharing one GPU)."""

    def __init__(self, devices):
        L = load_library()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _raise(L.cvg_multi_create(devs, len(devices), C.byref(h)))
        self._h = h
        self.devices = list(devices)
        self.last_stats = Stats()
        self.last_bounds = None

    def close(self):
        if getattr(self, "_h", None):
            load_library().cvg_multi_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_weights(self, deep_weight: float, shallow_weight: float):
        _raise(load_library().cvg_multi_set_weights(self._h, float(deep_weight), float(shallow_weight)))

    def convect(self, s, T, q, opts: KernelOptions | None = None, kernels=BOTH, first_col=0,
                out_deep: ColumnOutputs | None = None, out_shallow: ColumnOutputs | None = None):
        """As Context.convect, over all devices; the range offsets land in
        ``last_bounds``."""
        opts = opts or KernelOptions()
        keep, cols = _host_columns(s, T, q, first_col)
        L, n = keep[1].shape
        deep = (out_deep or ColumnOutputs.empty(n, L)) if kernels & DEEP else None
        sh = (out_shallow or ColumnOutputs.empty(n, L)) if kernels & SHALLOW else None
        st = Stats()
        b = np.zeros(len(self.devices) + 1, dtype=np.int64)
        rc = load_library().cvg_multi_convect(self._h, C.byref(cols), C.byref(opts), kernels,
                                              C.byref(deep._struct()) if deep else None,
                                              C.byref(sh._struct()) if sh else None, C.byref(st), b.ctypes.data)
        self.last_stats = st
        self.last_bounds = b
        _raise(rc, st)
        return deep, sh


class PinnedArray:
    """Page-locked host buffer (cvg_host_alloc) viewed as a numpy array."""

    def __init__(self, shape, dtype=np.float64):
        dt = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dt.itemsize
        p = C.c_void_p()
        _raise(load_library().cvg_host_alloc(nbytes, C.byref(p)))
        self._p = p
        buf = (C.c_char * max(nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)

    def free(self):
        if self._p:
            self.array = None
            load_library().cvg_host_free(self._p)
            self._p = None


_default_ctx: Context | None = None


def _ctx() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def deep_convection(s, T, q, opts=None, first_col=0) -> ColumnOutputs:
    """physics.hpp:155 -- deep convection over a column block on the GPU."""
    return _ctx().deep_convection(s, T, q, opts, first_col)


def shallow_convection(s, T, q, opts=None, first_col=0) -> ColumnOutputs:
    """physics.hpp:157 -- shallow convection over a column block on the GPU."""
    return _ctx().shallow_convection(s, T, q, opts, first_col)


def ientropy_solve(y, guess, opts=None):
    """physics.hpp:101 -- batched on the GPU; returns (root, iterations)."""
    return _ctx().ientropy_solve(y, guess, opts)


def approx_exp(x):
    """physics.hpp:83 -- evaluated on the GPU."""
    return _ctx().approx_exp(x)


def plan_partition(s, activity_threshold: float, n_parts: int, deep_weight: float = 1.0,
                   shallow_weight: float = 0.0) -> np.ndarray:
    """Contiguous G-way column split balanced by estimated cost (host C++,
    cvg_plan_partition).  deep_weight <= 0 gives the naive equal split."""
    s = np.ascontiguousarray(s, dtype=np.float64)
    b = np.empty(n_parts + 1, dtype=np.int64)
    rc = load_library().cvg_plan_partition(s.size, s.ctypes.data, float(activity_threshold),
                                           int(n_parts), float(deep_weight), float(shallow_weight),
                                           b.ctypes.data)
    _raise(rc)
    return b
