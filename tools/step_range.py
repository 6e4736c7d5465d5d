#!/usr/bin/env python3
"""One device-resident step between cudaProfilerStart / Stop, for an ncu RANGE
capture (the two kernels overlapped as in production, which per-kernel replay
serialises):

    ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python tools/step_range.py [--config c4]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1711_00289_b200 as P
    from paper_1711_00289_b200 import gridgen as G

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    thr = G.config_threshold(a.config)
    s, T, q = G.make_config(a.config, seed=42)
    L, n = T.shape
    dev = torch.device("cuda", 0)
    ldp = (n + 31) // 32 * 32

    def rows(x=None):
        t = torch.empty((L, ldp), dtype=torch.float64, device=dev)[:, :n]
        if x is not None:
            t.copy_(torch.from_numpy(np.ascontiguousarray(x)))
        return t

    ds = torch.from_numpy(np.ascontiguousarray(s)).to(dev)
    dT, dq = rows(T), rows(q)
    outs = [(rows(), rows(), torch.empty(n, dtype=torch.float64, device=dev),
             torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.uint8, device=dev))
            for _ in range(2)]
    opts = P.KernelOptions(activity_threshold=thr)
    ctx = P.Context(0)
    st = torch.cuda.Stream(device=dev)
    for _ in range(3):
        ctx.convect_async(ds, dT, dq, outs[0], outs[1], opts, P.BOTH, stream=st)
    ctx.check(st)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        ctx.convect_async(ds, dT, dq, outs[0], outs[1], opts, P.BOTH, stream=st)
    st.synchronize()
    torch.cuda.profiler.stop()
    ctx.check(st)
    print("step_range done")


if __name__ == "__main__":
    main()
