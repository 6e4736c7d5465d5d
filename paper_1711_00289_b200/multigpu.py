"""Multi-GPU plumbing for the column partition (host side).

BASELINE.json partitions the f02 grid across 1/2/4/8 B200s "by triggered-
column count"; columns are independent (physics.hpp:26-30), so there is no
collective on the data path.  Each rank takes one contiguous column range
from cvg_plan_partition (the G-way generalisation of plan_partition,
hetero.cpp:156-176) and runs the hot path on its own GPU;
torch.distributed is used only for barriers and the max-over-ranks of the
device timings.
"""
from __future__ import annotations

import os

import numpy as np

from . import plan_partition

# FLOP model per column: triggered deep 159 L + 37 U with
# U ~ 694 Newton updates at the reference's guess range; the shallow /
# zero-fill work is HBM-bound and is priced as its bytes at the machine's
# FLOP/byte balance.
MEAN_UPDATES = 694.0
BYTES_PER_COLUMN_30 = 1482.0

# Measured per-unit step times on one B200 at L = 30 (the analogue of the
# reference's calibrate(), hetero.cpp:110-163), refit whenever the kernels
# change (tools/fit_partition.py: c4, c5_50 and c5_05 ranges of 1/2/4/8-way
# balanced and naive splits, each a whole step, least squares): t = 35 us +
# 0.86 ns per triggered column + 0.154 ns per column -- a triggered column
# weighs ~5.6 plain columns (profiles/r04_fit_partition.json, tiled shallow kernel).
MEASURED_NS_PER_TRIGGERED = float(os.environ.get("CVG_W_TRIGGERED", 0.86))   # (overrides: calibration runs)
MEASURED_NS_PER_COLUMN = float(os.environ.get("CVG_W_COLUMN", 0.154))


def partition_weights(L: int = 30, hbm_gbs: float = 6558.7, fp64_tflops: float = 34.0, mode: str = "balanced"):
    """(deep_weight, shallow_weight) for cvg_plan_partition: measured B200
    per-unit times ("balanced") or the FLOP/byte model ("model")."""
    if mode == "model":
        deep_w = 159.0 * L + 37.0 * MEAN_UPDATES
        bytes_per_col = 8 + 2 * 8 * L + 2 * (2 * 8 * L + 17)
        shallow_w = bytes_per_col * (fp64_tflops * 1e12) / (hbm_gbs * 1e9)
        return deep_w, shallow_w
    return MEASURED_NS_PER_TRIGGERED * L / 30.0, MEASURED_NS_PER_COLUMN * L / 30.0


def rank_bounds(s, activity_threshold: float, world: int, mode: str = "balanced", L: int = 30,
                hbm_gbs: float = 6558.7, fp64_tflops: float = 34.0) -> np.ndarray:
    """world + 1 column offsets; rank r owns [b[r], b[r+1]).  mode:
    "balanced" (measured per-unit costs), "model" (FLOP/byte model) or
    "naive" (equal columns, StaticBlock).  Interior boundaries are rounded
    to multiples of ALIGN columns (a rank's rows then start on 256-byte
    boundaries and its 4-column groups are whole sectors; the rounding moves
    at most 16 columns per boundary)."""
    if mode == "naive":
        b = plan_partition(s, activity_threshold, world, 0.0, 1.0)
    elif mode == "overlap":
        b = overlap_bounds(s, activity_threshold, world, L)
    else:
        dw, sw = partition_weights(L, hbm_gbs, fp64_tflops, mode)
        b = plan_partition(s, activity_threshold, world, dw, sw)
    return align_bounds(b, ALIGN)


# Overlap-aware share cost (the deep and shallow kernels run concurrently):
# t = C0 + max(D, S) + GAMMA * min(D, S), D = A_DEEP * triggered columns,
# S = B_SHALLOW * columns -- a deep-bound share hides most of its shallow
# work and vice versa.  Fit on one B200: all-triggered c5_50 shares (deep
# bound), its mixed shares (shallow bound) and the f02 step (GAMMA).
C0_MS, A_DEEP_MS, B_SHALLOW_MS, GAMMA = 0.019, 1.29e-6, 0.27e-6, 0.25


def share_cost(n_trig, n_cols):
    d, sh = A_DEEP_MS * n_trig, B_SHALLOW_MS * n_cols
    return C0_MS + np.maximum(d, sh) + GAMMA * np.minimum(d, sh)


def overlap_bounds(s, activity_threshold: float, world: int, L: int = 30) -> np.ndarray:
    """Contiguous ranges minimising the largest share_cost: bisection on the
    target cost, each rank taking the longest prefix within it (the cost of
    a range grows with its end)."""
    n = int(np.asarray(s).size)
    trig = np.concatenate([[0], np.cumsum(np.asarray(s) > activity_threshold)]).astype(np.int64)
    scale = L / 30.0

    def cost(lo, e):
        return scale * share_cost(trig[e] - trig[lo], e - lo)

    def last_end(lo, target):
        """Largest end e in [lo, n] with cost(lo, e) <= target (the cost of a
        range grows with its end): bisection, O(log n) evaluations."""
        a, b = lo, n
        if cost(lo, n) <= target:
            return n
        while b - a > 1:
            mid = (a + b) // 2
            if cost(lo, mid) <= target:
                a = mid
            else:
                b = mid
        return a

    def greedy(target):
        b = [0]
        for _ in range(world - 1):
            b.append(last_end(b[-1], target))
        b.append(n)
        return np.array(b, dtype=np.int64)

    def worst(b):
        return max(cost(b[i], b[i + 1]) for i in range(world))

    lo_t, hi_t = 0.0, float(cost(0, n))
    for _ in range(40):
        mid = 0.5 * (lo_t + hi_t)
        if worst(greedy(mid)) <= mid + 1e-12:
            hi_t = mid
        else:
            lo_t = mid
    return greedy(hi_t)


ALIGN = 32


def align_bounds(b, align: int = ALIGN) -> np.ndarray:
    """Rounds the interior offsets of a partition to the nearest multiple of
    `align` (ends kept), preserving monotonicity."""
    b = np.asarray(b, dtype=np.int64).copy()
    n = int(b[-1])
    for i in range(1, len(b) - 1):
        b[i] = min(n, max(int(b[i - 1]), int(np.rint(b[i] / align)) * align))
    return b


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max)."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])
