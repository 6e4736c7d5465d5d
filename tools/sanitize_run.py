#!/usr/bin/env python3
"""Small workload that launches every kernel of the library, for
compute-sanitizer (one tool per run):

    compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_run.py
    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py
    compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py

c1 at 4,096 columns: trigger + compaction, every deep kernel
(split 2/4/8 lanes, thread- and warp-per-column), every variant, the strict
and no-far32 paths, the guard-band re-derivation (redo_kernel, and inline),
the shallow kernel with and without the deep zero-fill, the tiled shallow
kernel (forced at this size), programmatic and plain deep launches, the host-buffer
pipeline with small chunks, the fused feedback loop (deep and shallow),
error growth, the multi-device engine, the batched ientropy / exp entry
points and a latched failure.  Results are checked against the oracle at the
end (test infrastructure), so a sanitizer run is also a parity run.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import oracle as O
    import paper_1711_00289_b200 as P
    from conftest import env_context
    from paper_1711_00289_b200 import gridgen as G

    n = int(os.environ.get("SAN_COLUMNS", "4096"))
    s, T, q = G.make_config("c1", n=n, seed=7)
    checks = 0
    envs = [{}, {"CVG_DEEP_LPC": "2"}, {"CVG_DEEP_LPC": "4"}, {"CVG_DEEP_LPC": "8"}, {"CVG_DEEP_TPC": "1"},
            {"CVG_DEEP_LPC": "0", "CVG_DEEP_TPC": "0"}, {"CVG_REDO_INLINE": "1"}, {"CVG_OVERLAP": "0"},
            {"CVG_CHUNK_COLS": "1000"}, {"CVG_SHALLOW_TILE": "2"}, {"CVG_SHALLOW_TILE": "2", "CVG_TILE_WARPS": "3"},
            {"CVG_PDL": "0"}]
    for env in envs:
        ctx = env_context(**env)
        for variant in (0, 1, 2):
            for kw in ({}, {"strict": True}, {"far32": False}):
                if variant == 2 and kw:
                    continue
                deep, sh = ctx.convect(s, T, q, P.KernelOptions(variant=variant, **kw))
                od = O.convection("deep", s, T, q, O.Options(variant=variant))
                osh = O.convection("shallow", s, T, q, O.Options(variant=variant))
                assert np.array_equal(deep.work_units, od.work), (env, variant, kw)
                assert np.array_equal(sh.work_units, osh.work), (env, variant, kw)
                checks += 1
        ctx.close()
    ctx = P.Context(0)
    # deep-only and shallow-only calls (the zero-fill path and without it)
    ctx.convect(s, T, q, kernels=P.DEEP)
    ctx.convect(s, T, q, kernels=P.SHALLOW)
    # fused feedback loop, both kernels, more steps than the check interval
    ctx.timestep(s, T, q, kernel=P.DEEP, n_steps=18)
    ctx.timestep(s, T, q, kernel=P.SHALLOW, n_steps=3)
    g = ctx.error_growth(s[:512], T[:, :512], q[:, :512], P.DEEP, P.KernelOptions(), P.KernelOptions(variant=1), 3)
    assert g.envelope_ok
    # batched entry points
    ctx.ientropy_solve(np.linspace(1.1, 2.0, 257), 150.0)
    ctx.exp(np.linspace(-700.0, 700.0, 1001))
    ctx.approx_exp(np.linspace(-60.0, 60.0, 1001))
    # a latched failure
    s2 = s.copy()
    s2[123] = np.nan
    try:
        ctx.convect(s2, T, q)
        raise AssertionError("expected a KernelError")
    except P.KernelError as e:
        assert e.column == 123
    ctx.close()
    with P.MultiContext([0, 0, 0]) as m:
        d3, s3 = m.convect(s, T, q)
        assert np.array_equal(d3.work_units, O.convection("deep", s, T, q).work)
    print(f"sanitize_run ok: {checks} parity-checked calls plus loop / growth / batched / failure / multi paths")


if __name__ == "__main__":
    main()
