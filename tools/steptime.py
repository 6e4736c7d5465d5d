#!/usr/bin/env python3
"""A/B step timing on one GPU with low noise: one process, the grid generated
once, one context per configuration (CVG_* switches are read at context
creation), configurations timed round-robin, median over repetitions.

    python tools/steptime.py [--config c4] [--steps 100] [--reps 7] \
        base "guard0:CVG_GUARD=0" "lpc4:CVG_DEEP_LPC=4" ...

Each argument is label[:ENV=VAL,ENV=VAL]; opts via --opts strict,nofar32.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    import paper_1711_00289_b200 as P
    from conftest import env_context
    from paper_1711_00289_b200 import gridgen as G

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--opts", default="")
    ap.add_argument("--slice", default=None, help="R/W: rank R's share of a W-way partition")
    ap.add_argument("--kernels", action="store_true", help="also a profiled pass (per-kernel medians)")
    ap.add_argument("--mask", default="both", choices=["both", "deep", "shallow"], help="kernels of the call")
    ap.add_argument("--thr", type=float, default=None,
                    help="activity threshold override (2.0: nothing triggers -- the shallow kernel alone)")
    ap.add_argument("specs", nargs="+")
    a = ap.parse_args()
    thr = G.config_threshold(a.config)
    s, T, q = G.make_config(a.config, seed=42)
    if a.thr is not None:
        thr = a.thr
    L = T.shape[0]
    if a.slice:
        from paper_1711_00289_b200 import multigpu
        r, w = (int(x) for x in a.slice.split("/"))
        b = multigpu.rank_bounds(s, thr, w, "balanced", L, 6531.0)
        s, T, q = s[b[r]:b[r + 1]], T[:, b[r]:b[r + 1]], q[:, b[r]:b[r + 1]]
    n = s.size
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
    flags = {"strict": {"strict": True}, "nofar32": {"far32": False}}
    kw = {}
    for o in filter(None, a.opts.split(",")):
        kw.update(flags[o])
    opts = P.KernelOptions(variant=a.variant, activity_threshold=thr, **kw)
    MASK = {"both": P.BOTH, "deep": P.DEEP, "shallow": P.SHALLOW}[a.mask]
    stream = torch.cuda.Stream(device=dev)
    runs = []
    for spec in a.specs:
        label, _, envs = spec.partition(":")
        env = dict(e.split("=", 1) for e in envs.split(",") if e)
        ctx = env_context(**env)
        for _ in range(3):
            ctx.convect_async(ds, dT, dq, outs[0], outs[1], opts, MASK, stream=stream)
        st = ctx.check(stream)
        runs.append((label, ctx, [], st))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(a.reps):
        for label, ctx, ts, _ in runs:
            torch.cuda.synchronize()
            ev0.record(stream)
            for _ in range(a.steps):
                ctx.convect_async(ds, dT, dq, outs[0], outs[1], opts, MASK, stream=stream)
            ev1.record(stream)
            stream.synchronize()
            ts.append(ev0.elapsed_time(ev1) / a.steps)
    for label, ctx, ts, st in runs:
        ctx.check(stream)
        kern = ""
        if a.kernels:   # one profiled pass: event pairs between the kernels
            ctx.profile_begin(a.steps)
            for _ in range(a.steps):
                ctx.convect_async(ds, dT, dq, outs[0], outs[1], opts, MASK, stream=stream)
            stream.synchronize()
            k = ctx.profile_end(a.steps)
            kern = "  trig %.4f deep %.4f shallow(after deep) %.4f" % tuple(np.median(k, axis=0))
        print(f"{label:24s} {a.config} n={n} median {np.median(ts):.4f} ms  min {np.min(ts):.4f}  max {np.max(ts):.4f}"
              f"  rederived {st.n_recomputed} rewritten {getattr(st, 'n_corrected', 0)}{kern}", flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
