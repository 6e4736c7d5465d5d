#!/usr/bin/env python3
"""Calibrate the multi-GPU partition weights (the analogue of the reference's
calibrate(), hetero.cpp:110-163): time column ranges of several layouts on
one GPU and fit  t = C0 + a * triggered + b * columns  by least squares.

    python tools/fit_partition.py [--out gpurun_out/fit_partition.json]

Each range is timed as a whole step (trigger, deep, re-derivation, shallow)
with CUDA events, median of 5 x 40 steps.  The fitted a, b (ns per unit)
are the cvg_multi / multigpu.py weights; C0 is the fixed per-step cost that
bounds strong scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1711_00289_b200 as P
    from paper_1711_00289_b200 import gridgen as G
    from paper_1711_00289_b200 import multigpu

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "fit_partition.json"))
    ap.add_argument("--configs", default="c4,c5_50,c5_05")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = P.Context(0)
    stream = torch.cuda.Stream(device=dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rows = []
    for cfg in a.configs.split(","):
        thr = G.config_threshold(cfg)
        s, T, q = G.make_config(cfg, seed=42)
        L = T.shape[0]
        for W in (1, 2, 4, 8):
            for mode in (("balanced", "naive") if W > 1 else ("naive",)):
                b = multigpu.rank_bounds(s, thr, W, mode, L)
                for r in range(W):
                    lo, hi = int(b[r]), int(b[r + 1])
                    n = hi - lo
                    if n <= 0:
                        continue
                    ldp = (n + 31) // 32 * 32

                    def rows2(x=None):
                        t = torch.empty((L, ldp), dtype=torch.float64, device=dev)[:, :n]
                        if x is not None:
                            t.copy_(torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])))
                        return t
                    ds = torch.from_numpy(np.ascontiguousarray(s[lo:hi])).to(dev)
                    dT, dq = rows2(T), rows2(q)
                    outs = [(rows2(), rows2(), torch.empty(n, dtype=torch.float64, device=dev),
                             torch.empty(n, dtype=torch.int64, device=dev),
                             torch.empty(n, dtype=torch.uint8, device=dev)) for _ in range(2)]
                    o = P.KernelOptions(activity_threshold=thr)
                    for _ in range(3):
                        ctx.convect_async(ds, dT, dq, outs[0], outs[1], o, P.BOTH, first_col=lo, stream=stream)
                    ctx.check(stream)
                    ts = []
                    for _ in range(5):
                        ev0.record(stream)
                        for _ in range(40):
                            ctx.convect_async(ds, dT, dq, outs[0], outs[1], o, P.BOTH, first_col=lo, stream=stream)
                        ev1.record(stream)
                        stream.synchronize()
                        ts.append(ev0.elapsed_time(ev1) / 40)
                    trig = int((s[lo:hi] > thr).sum())
                    rows.append({"config": cfg, "W": W, "mode": mode, "rank": r, "n": n, "triggered": trig,
                                 "ms": float(np.median(ts))})
                    print(json.dumps(rows[-1]), flush=True)
                    del ds, dT, dq, outs
    A = np.array([[1.0, r["triggered"], r["n"]] for r in rows])
    y = np.array([r["ms"] for r in rows])
    coef, *_ = np.linalg.lstsq(A, y, rcond=None)
    pred = A @ coef
    fit = {"C0_ms": float(coef[0]), "ns_per_triggered": float(coef[1] * 1e6), "ns_per_column": float(coef[2] * 1e6),
           "max_rel_residual": float(np.max(np.abs(pred - y) / y)), "rows": rows}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(fit, f, indent=1)
    print(json.dumps({k: v for k, v in fit.items() if k != "rows"}))
    ctx.close()


if __name__ == "__main__":
    main()
