"""Seeded synthetic column grids for the five BASELINE.json configurations.

The reference generator (physics.cpp:247-277) draws i.i.d. uniform T, q and
places its active columns in one contiguous middle band; it has none of the
physically shaped profiles BASELINE.json describes.  This module writes them
(SURVEY.md section 8(d)), keeping the reference's counter-based determinism:
every random draw is ``rng_u01(seed, stream, counter)`` -- the splitmix64 of
prng.hpp:23-47 -- so any column can be regenerated in isolation and the
result never depends on evaluation order or thread count.

Only ``s``, ``T`` and ``q`` are read by the kernels (a column is
``(col_id, s, T[L], q[L])``, physics.hpp:32-37).  Pressure, the surface
fluxes and omega that BASELINE.json mentions shape nothing the kernels see;
``extras=True`` returns them for completeness, they are never counted as
algorithmic bytes.

Layout: level-major SoA, ``T[L][n]``, ``q[L][n]``, level 0 at the model top
(3.6 hPa), level L-1 at the surface; column index ``col = ilat * nlon + ilon``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _fin(z):
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def rng_u64(seed, stream, counter):
    """prng.hpp:37-41, vectorised over ``counter``."""
    with np.errstate(over="ignore"):
        keyed = _fin(np.uint64(seed) + _GAMMA * np.uint64(stream + 1))
        c = np.asarray(counter, dtype=np.uint64)
        return _fin(keyed + _GAMMA * (c + np.uint64(1)))


def rng_u01(seed, stream, counter):
    """prng.hpp:44-47: 53 random bits in [0, 1)."""
    return (rng_u64(seed, stream, counter) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def rng_normal(seed, stream, counter):
    """Box-Muller on two counter-based uniforms."""
    c = np.asarray(counter, dtype=np.uint64)
    u1 = rng_u01(seed, stream, c * np.uint64(2))
    u2 = rng_u01(seed, stream, c * np.uint64(2) + np.uint64(1))
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


# ---------------------------------------------------------------------------
# Reference generator (physics.cpp:247-277), for known-answer tests.
def reference_grid(n, L=30, tropics_band=0.3, seed=42):
    """Bit-identical restatement of make_grid (level-major output)."""
    band = int(math.floor(tropics_band * n + 0.5))  # llround for band >= 0
    lo = (n - band) // 2
    c = np.arange(n, dtype=np.uint64)
    us = rng_u01(seed, 0, c)
    trop = (c >= lo) & (c < lo + band)
    s = np.where(trop, 0.5 + 0.5 * us, 0.5 * us)
    ctr = c[None, :] * np.uint64(L) + np.arange(L, dtype=np.uint64)[:, None]
    T = 250.0 + 60.0 * rng_u01(seed, 1, ctr)
    q = 0.022 * rng_u01(seed, 2, ctr)
    return s, np.ascontiguousarray(T), np.ascontiguousarray(q)


# ---------------------------------------------------------------------------
# Thermodynamics used only to shape T and q.
RD, CPD, LV, EPS = 287.04, 1004.64, 2.501e6, 0.622


def esat_hpa(T):
    """Bolton (1980) saturation vapour pressure over water, hPa."""
    return 6.112 * np.exp(17.67 * (T - 273.15) / (T - 29.65))


def qsat(T, p_hpa):
    es = np.minimum(esat_hpa(T), 0.5 * p_hpa)
    return EPS * es / (p_hpa - (1.0 - EPS) * es)


def level_pressure(ps_hpa, L, p_top=3.6):
    """Hybrid-sigma-like levels: ln p runs from ln p_top (k=0) to ln ps
    (k=L-1), compressed towards the surface (x_k = 1 - (1 - k/(L-1))^2)."""
    k = np.arange(L, dtype=np.float64)
    x = 1.0 - (1.0 - k / max(L - 1, 1)) ** 2
    return p_top * np.exp(np.log(ps_hpa / p_top)[None, :] * x[:, None])  # [L][n]


_ADIABAT = None


def _moist_adiabat_table():
    """T(Ts, dlnp) along the pseudo-adiabat, integrated once with RK4 in ln p
    from ps = 1000 hPa; rows Ts = 230..315 K step 0.25, cols dlnp = 0..-6."""
    global _ADIABAT
    if _ADIABAT is None:
        ts = np.arange(230.0, 315.0001, 0.25)
        d = np.linspace(0.0, -6.0, 601)
        out = np.empty((ts.size, d.size))
        T = ts.copy()
        out[:, 0] = T
        h = d[1] - d[0]

        def f(T, lnp):
            p = np.exp(lnp)
            rs = qsat(T, p)
            return (RD * T + LV * rs) / (CPD + LV * LV * rs * EPS / (RD * T * T))

        lnp = math.log(1000.0)
        for j in range(1, d.size):
            k1 = f(T, lnp)
            k2 = f(T + 0.5 * h * k1, lnp + 0.5 * h)
            k3 = f(T + 0.5 * h * k2, lnp + 0.5 * h)
            k4 = f(T + h * k3, lnp + h)
            T = T + h / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
            lnp += h
            out[:, j] = T
        _ADIABAT = (ts, d, out)
    return _ADIABAT


def moist_adiabat(Ts, p, ps):
    """Bilinear lookup of the pseudo-adiabat through (Ts, ps) at pressure p."""
    ts, d, tab = _moist_adiabat_table()
    x = np.clip((Ts - ts[0]) / (ts[1] - ts[0]), 0, ts.size - 1.000001)
    y = np.clip(np.log(p / ps) / (d[1] - d[0]), 0, d.size - 1.000001)
    i = np.floor(x).astype(np.int64)
    j = np.floor(y).astype(np.int64)
    fx, fy = x - i, y - j
    return ((1 - fx) * (1 - fy) * tab[i, j] + fx * (1 - fy) * tab[i + 1, j] +
            (1 - fx) * fy * tab[i, j + 1] + fx * fy * tab[i + 1, j + 1])


# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class ConfigSpec:
    name: str
    nlat: int | None
    nlon: int | None
    n: int
    activity_threshold: float
    description: str


CONFIGS = {
    "c1": ConfigSpec("c1", None, None, 4096, 0.5,
                     "PR1: 4,096 columns, Ts~N(300,3), 40% uniform-random triggered (+2 K boundary layer)"),
    "c2": ConfigSpec("c2", 96, 144, 13824, 0.5,
                     "f19: 96x144, latitude-banded, ~35% triggered around the tropics"),
    "c3": ConfigSpec("c3", 192, 288, 55296, 0.75,
                     "f09: 192x288, 30% deep + 25% shallow-only (activity_threshold 0.75)"),
    "c4": ConfigSpec("c4", 768, 1152, 884736, 0.5,
                     "f02: 768x1152, 30% deep in Gaussian-random-field clusters (500 km)"),
    "c5_05": ConfigSpec("c5_05", 768, 1152, 884736, 0.5, "stress: 5% triggered, one contiguous block"),
    "c5_50": ConfigSpec("c5_50", 768, 1152, 884736, 0.5, "stress: 50% triggered, one contiguous block"),
    "c5_95": ConfigSpec("c5_95", 768, 1152, 884736, 0.5, "stress: 95% triggered, one contiguous block"),
}

# RNG stream ids (separate fields never share a stream)
_S_TS, _S_PS, _S_NOISE, _S_RH, _S_TRIG, _S_SVAL, _S_GRF, _S_EXTRA = 101, 102, 103, 104, 105, 106, 107, 108


def _place_s(trig, thr, v, lo_cap=None):
    """Triggered s in (thr, 1), others in [0, thr) (or [0, lo_cap)), each at
    least 1e-6 relative away from thr so no trigger sits on the threshold."""
    d = 1e-6
    hi = thr + (1.0 - thr) * (d + (1.0 - 2 * d) * v)
    cap = thr if lo_cap is None else lo_cap
    lo = cap * (1.0 - d) * v
    return np.where(trig, hi, lo)


def _top_fraction(score, frac):
    """Boolean mask of exactly round(frac * n) largest scores (stable ties)."""
    n = score.size
    k = int(round(frac * n))
    mask = np.zeros(n, dtype=bool)
    if k > 0:
        order = np.argsort(-score, kind="stable")
        mask[order[:k]] = True
    return mask


def _grf(nlat, nlon, seed, length_km=500.0, radius_km=6371.0):
    """Gaussian random field with a Gaussian covariance of length scale
    ``length_km``: white noise (counter-based normals) filtered in Fourier
    space (periodic in longitude; latitude padded)."""
    pad = nlat // 2
    ny = nlat + 2 * pad
    ctr = np.arange(ny * nlon, dtype=np.uint64)
    w = rng_normal(seed, _S_GRF, ctr).reshape(ny, nlon)
    dy = math.pi * radius_km / nlat
    dx = 2 * math.pi * radius_km / nlon
    sig = length_km / math.sqrt(2.0)
    ky = np.fft.fftfreq(ny, d=dy) * 2 * math.pi
    kx = np.fft.rfftfreq(nlon, d=dx) * 2 * math.pi
    filt = np.exp(-0.5 * (sig ** 2) * (ky[:, None] ** 2 + kx[None, :] ** 2))
    g = np.fft.irfft2(np.fft.rfft2(w) * filt, s=(ny, nlon))[pad:pad + nlat]
    g = (g - g.mean()) / g.std()
    return g.reshape(-1)


def make_config(name: str, n: int | None = None, seed: int = 42, L: int = 30,
                shape: tuple[int, int] | None = None, extras: bool = False):
    """Returns (s[n], T[L][n], q[L][n]) for a BASELINE config.  ``shape``
    (nlat, nlon) or ``n`` shrink the grid for tests; the recipe is unchanged."""
    if name == "ref":
        return reference_grid(n or 4096, L, 0.3, seed)
    spec = CONFIGS[name]
    thr = spec.activity_threshold
    if spec.nlat is None:
        n = n or spec.n
        nlat, nlon = 1, n
        lat = np.zeros(n)
    else:
        if shape is not None:
            nlat, nlon = shape
        elif n is not None and n != spec.n:
            nlat = max(2, int(round(math.sqrt(n * spec.nlat / spec.nlon))))
            nlon = max(1, n // nlat)
        else:
            nlat, nlon = spec.nlat, spec.nlon
        latc = -90.0 + (np.arange(nlat) + 0.5) * 180.0 / nlat
        lat = np.repeat(latc, nlon)
        n = nlat * nlon
    col = np.arange(n, dtype=np.uint64)
    lev = np.arange(L, dtype=np.uint64)
    ctr2 = col[None, :] * np.uint64(L) + lev[:, None]

    # surface state and levels
    ps = 950.0 + 80.0 * rng_u01(seed, _S_PS, col)
    p = level_pressure(ps, L)                       # [L][n] hPa
    cos2 = np.cos(np.deg2rad(lat)) ** 2
    if spec.nlat is None:
        Ts = 300.0 + 3.0 * rng_normal(seed, _S_TS, col)
        rh_scale = np.ones(n)
    else:
        Ts = 250.0 + 52.0 * cos2
        rh_scale = 0.75 + 0.25 * cos2              # latitude-dependent moistening

    # triggered (deep) columns and the activity scalar s
    u_trig = rng_u01(seed, _S_TRIG, col)
    u_s = rng_u01(seed, _S_SVAL, col)
    shallow_only = np.zeros(n, dtype=bool)
    if name == "c1":
        trig = _top_fraction(u_trig, 0.40)
        s = _place_s(trig, thr, u_s)
    elif name == "c2":
        trig = _top_fraction(-np.abs(lat) + 8.0 * u_trig, 0.35)
        s = _place_s(trig, thr, u_s)
    elif name == "c3":
        score = -np.abs(lat) + 8.0 * u_trig
        order = np.argsort(-score, kind="stable")
        nd, nsh = int(round(0.30 * n)), int(round(0.25 * n))
        trig = np.zeros(n, dtype=bool)
        trig[order[:nd]] = True
        shallow_only[order[nd:nd + nsh]] = True
        # deep in (0.75, 1); shallow-only in (0.64, 0.75): survives all four
        # shallow phases (needs s * 0.95 >= 0.60); the rest below 0.55
        s = _place_s(trig, thr, u_s, lo_cap=0.55)
        s = np.where(shallow_only, 0.64 + (0.75 - 0.64) * (1e-6 + (1 - 2e-6) * u_s), s)
    elif name == "c4":
        g = _grf(nlat, nlon, seed) + 0.8 * cos2
        trig = _top_fraction(g, 0.30)
        # s grows with the field's strength inside a cluster, with noise
        rank = np.empty(n)
        rank[np.argsort(g, kind="stable")] = np.arange(n) / max(n - 1, 1)
        v = np.clip(0.5 * (rank - 0.7) / 0.3 + 0.5 * u_s, 0.0, 1.0)
        v_lo = np.clip(0.5 * rank / 0.7 + 0.5 * u_s, 0.0, 1.0)
        s = np.where(trig, _place_s(trig, thr, v), _place_s(trig, thr, v_lo))
    elif name.startswith("c5"):
        frac = int(name.split("_")[1]) / 100.0
        a = int(round(frac * n))
        lo = (n - a) // 2
        trig = (np.arange(n) >= lo) & (np.arange(n) < lo + a)
        s = _place_s(trig, thr, u_s)
    else:
        raise KeyError(name)

    # temperature: moist adiabat below 100 hPa (floored at a 200 K
    # tropopause), 210 K isothermal above,
    # +-1 K per-level noise; C1's triggered columns get a +2 K boundary layer
    T = np.maximum(moist_adiabat(Ts[None, :], p, ps[None, :]), 200.0)  # tropopause floor
    T = np.where(p < 100.0, 210.0, T)
    T = T + (2.0 * rng_u01(seed, _S_NOISE, ctr2) - 1.0)
    if name == "c1":
        T = T + np.where((p > 850.0) & trig[None, :], 2.0, 0.0)

    # moisture: RH * qsat, RH ~ U(0.6, 0.95) below 700 hPa, U(0.1, 0.5) above
    u_rh = rng_u01(seed, _S_RH, ctr2)
    rh = np.where(p >= 700.0, 0.6 + 0.35 * u_rh, 0.1 + 0.4 * u_rh) * rh_scale[None, :]
    q = np.clip(rh * qsat(T, p), 0.0, 0.025)

    s = np.ascontiguousarray(s, dtype=np.float64)
    T = np.ascontiguousarray(T, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    if not extras:
        return s, T, q
    ex = {
        "p_hpa": p, "ps_hpa": ps, "lat": lat,
        "shf": 50.0 * rng_u01(seed, _S_EXTRA, col * np.uint64(3)),
        "lhf": 250.0 * rng_u01(seed, _S_EXTRA, col * np.uint64(3) + np.uint64(1)),
        "omega": 0.1 * rng_normal(seed, _S_EXTRA + 1, ctr2),
        "triggered": trig, "shallow_only": shallow_only, "activity_threshold": thr,
    }
    return s, T, q, ex


def config_threshold(name: str) -> float:
    return 0.5 if name == "ref" else CONFIGS[name].activity_threshold
