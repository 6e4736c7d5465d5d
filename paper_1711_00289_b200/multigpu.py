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

import numpy as np

from . import plan_partition

# FLOP model per column: triggered deep 159 L + 37 U with
# U ~ 694 Newton updates at the reference's guess range; the shallow /
# zero-fill work is HBM-bound and is priced as its bytes at the machine's
# FLOP/byte balance.
MEAN_UPDATES = 694.0
BYTES_PER_COLUMN_30 = 1482.0


def partition_weights(L: int = 30, hbm_gbs: float = 6558.7, fp64_tflops: float = 34.0):
    deep_w = 159.0 * L + 37.0 * MEAN_UPDATES
    bytes_per_col = 8 + 2 * 8 * L + 2 * (2 * 8 * L + 17)
    shallow_w = bytes_per_col * (fp64_tflops * 1e12) / (hbm_gbs * 1e9)
    return deep_w, shallow_w


def rank_bounds(s, activity_threshold: float, world: int, mode: str = "balanced", L: int = 30,
                hbm_gbs: float = 6558.7, fp64_tflops: float = 34.0) -> np.ndarray:
    """world + 1 column offsets; rank r owns [b[r], b[r+1])."""
    if mode == "naive":
        return plan_partition(s, activity_threshold, world, 0.0, 1.0)
    dw, sw = partition_weights(L, hbm_gbs, fp64_tflops)
    return plan_partition(s, activity_threshold, world, dw, sw)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max)."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t[0])
