#!/usr/bin/env python3
"""GPU parity report: every BASELINE config at its stated size, every variant,
every device path, EVERY column against the CPU oracle (test infrastructure).

    python tools/parity_report.py --out profiles/parity_r05.json [--quick]

Per (config, variant, path) and kernel it records, for tend_T / tend_q /
precip, the worst absolute and relative deviation and the number of values
outside the north-star tolerance (1e-10 relative or 1e-14 absolute); the
trigger / exit flag mismatches and the work_units mismatches (both must be
0); the columns the rule would exempt (shallow predicates within 1e-9 of
their theta -- the north star's near-threshold rule) with their deviations;
the Newton-margin class size (columns whose reference residual came within
1e-3 of newton_tol: where a device exp or rounding difference could flip a
count); and the number of solves the guard band re-ran on the exact path
(cvg_stats.n_recomputed: levels re-derived; n_corrected: columns rewritten).  A guard sweep (CVG_GUARD = 0 .. default) on the
f02 and stress grids shows what the guard removes: the count flips a
relaxed path makes without it.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402  (test infrastructure: the checker)
import paper_1711_00289_b200 as P  # noqa: E402
from paper_1711_00289_b200 import gridgen as G  # noqa: E402

REL, ABS = 1e-10, 1e-14
PRED_MARGIN, NEWTON_MARGIN = 1e-9, 1e-3
CONFIGS = ["ref", "c1", "c2", "c3", "c4", "c5_05", "c5_50", "c5_95"]
PATHS = {"default": {}, "strict": {"strict": True}, "no_far32": {"far32": False}}


def compare(got, want, kernel, margin):
    exempt = margin < PRED_MARGIN if kernel == "shallow" else np.zeros(margin.shape, bool)
    rec = {"flag_mismatch": int((got.exited_early != want.exited)[~exempt].sum()),
           "work_mismatch": int((got.work_units != want.work)[~exempt].sum())}
    worst = {}
    bad_cols = np.zeros(margin.shape, bool)
    for f in ("tend_T", "tend_q", "precip"):
        a, b = getattr(got, f), getattr(want, f)
        d = np.abs(a - b)
        viol = d > np.maximum(REL * np.abs(b), ABS)
        rel = np.where(np.abs(b) > 0, d / np.maximum(np.abs(b), 1e-300), np.where(d > 0, np.inf, 0.0))
        worst[f] = {"max_abs": float(d.max()) if d.size else 0.0,
                    "max_rel_nonzero": float(rel[np.abs(b) > 0].max()) if (np.abs(b) > 0).any() else 0.0,
                    "violations": int(viol[..., ~exempt].sum())}
        bad_cols |= viol.any(axis=0) if viol.ndim == 2 else viol
    rec["fields"] = worst
    rec["exempt_columns"] = [{"column": int(c), "margin": float(margin[c]),
                              "flag_equal": bool(got.exited_early[c] == want.exited[c])}
                             for c in np.nonzero(exempt)[0][:100]]
    rec["columns_outside_tolerance"] = [int(c) for c in np.nonzero(bad_cols & ~exempt)[0][:50]]
    return rec


def context(**env):
    from conftest import env_context
    return env_context(**{k: str(v) for k, v in env.items()})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity_r04.json"))
    ap.add_argument("--quick", action="store_true", help="small grids only (smoke of the tool)")
    ap.add_argument("--seed", type=int, default=42)
    args = ap.parse_args()
    t0 = time.time()
    ctx = P.Context(0)
    report = {"rule": "flags and work_units exact; tend_T, tend_q, precip within 1e-10 relative or 1e-14 "
                      "absolute, every column; shallow exit flags exempt within 1e-9 of theta (none occur)",
              "host": platform.node(), "host_cores": os.cpu_count(), "seed": args.seed, "runs": [],
              "guard_sweep": []}
    configs = ["ref", "c1", "c2"] if args.quick else CONFIGS
    for cfg in configs:
        kw = {"shape": (24, 36)} if (args.quick and cfg not in ("ref", "c1", "c2")) else {}
        s, T, q = G.make_config(cfg, seed=args.seed, **kw)
        thr = G.config_threshold(cfg)
        for variant in (0, 1, 2):
            oo = O.Options(variant=variant, activity_threshold=thr)
            od = O.convection_mt("deep", s, T, q, oo)
            osh = O.convection_mt("shallow", s, T, q, oo)
            trig = od.exited == 0
            for path, extra in PATHS.items():
                if variant == 2 and path != "default":
                    continue   # ApproxTranscendental always runs the exact update
                opts = P.KernelOptions(variant=variant, activity_threshold=thr, **extra)
                deep, sh = ctx.convect(s, T, q, opts)
                st = ctx.last_stats
                run = {"config": cfg, "n_columns": int(s.size), "activity_threshold": thr, "variant": variant,
                       "path": path, "triggered": int(trig.sum()),
                       "newton_margin_class": int((od.margin[trig] < NEWTON_MARGIN).sum()),
                       "min_shallow_predicate_margin": float(osh.margin.min()),
                       "rederived_levels": int(st.n_recomputed), "rewritten_columns": int(st.n_corrected),
                       "deep": compare(deep, od, "deep", od.margin),
                       "shallow": compare(sh, osh, "shallow", osh.margin)}
                run["precip_bit_identical"] = bool(np.array_equal(deep.precip.view(np.int64),
                                                                  od.precip.view(np.int64)))
                run["ok"] = all(run[k]["flag_mismatch"] == 0 and run[k]["work_mismatch"] == 0 and
                                all(v["violations"] == 0 for v in run[k]["fields"].values())
                                for k in ("deep", "shallow"))
                report["runs"].append(run)
                print(f"{cfg:6s} v{variant} {path:8s} ok={run['ok']} rederived={run['rederived_levels']} "
                      f"rewritten={run['rewritten_columns']} margin_class={run['newton_margin_class']}", flush=True)
    # guard sweep: what the band removes (relaxed default path, Exact)
    sweep_cfgs = ["c1"] if args.quick else ["c4", "c5_95"]
    for cfg in sweep_cfgs:
        s, T, q = G.make_config(cfg, seed=args.seed)
        od = O.convection_mt("deep", s, T, q)
        trig = od.exited == 0
        for g in (0.0, 1e-3, 1.0 / 256, 1.0 / 128, 1.0 / 64):
            c = context(CVG_GUARD=g)
            deep, _ = c.convect(s, T, q, P.KernelOptions(), kernels=P.DEEP)
            flips = deep.work_units != od.work
            report["guard_sweep"].append({
                "config": cfg, "guard": g, "work_flips": int(flips.sum()),
                "flips_outside_margin_class": int((flips & (od.margin >= NEWTON_MARGIN)).sum()),
                "flipped_columns": [int(x) for x in np.nonzero(flips)[0][:40]],
                "rederived_levels": int(c.last_stats.n_recomputed),
                "rewritten_columns": int(c.last_stats.n_corrected), "triggered": int(trig.sum())})
            print(f"guard {cfg} g={g:.5f} flips={int(flips.sum())} rederived={c.last_stats.n_recomputed} "
                  f"rewritten={c.last_stats.n_corrected}", flush=True)
            c.close()
    report["all_ok"] = all(r["ok"] for r in report["runs"])
    report["wall_s"] = time.time() - t0
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(report, f, indent=1)
    print(f"all_ok={report['all_ok']} -> {args.out} ({report['wall_s']:.0f} s)")
    ctx.close()
    return 0 if report["all_ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
