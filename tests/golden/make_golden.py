"""Generates tests/golden/*.npz from the REFERENCE ITSELF.

Run in the build container (needs oracle/_ref/libconvref.so, i.e. the
reference's physics.cpp compiled from /root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Each fixture holds the level-major inputs (s, T, q), the KernelOptions, and
the reference's deep_convection / shallow_convection outputs
(physics.hpp:155-158) for all three variants.  The reference publishes no
stored golden vectors; these pin the restatement
oracle/convproxy_oracle.c and, on the GPU box, the CUDA path.  Values depend
on the host libm (glibc 2.39 here) only through exp/sin.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1711_00289_b200 import gridgen  # noqa: E402

CASES = {
    # reference generator, the reference tests' own shapes/seeds
    "ref_n64_seed7": dict(kind="ref", n=64, band=0.3, seed=7),
    "ref_n128_band04_seed42": dict(kind="ref", n=128, band=0.4, seed=42),
    # BASELINE configs, shrunk
    "c1_n96": dict(kind="cfg", name="c1", n=96, seed=3),
    "c3_12x18": dict(kind="cfg", name="c3", shape=(12, 18), seed=5),
    "c4_12x16": dict(kind="cfg", name="c4", shape=(12, 16), seed=9),
}


def make(case):
    if case["kind"] == "ref":
        s, T, q = O.ref_make_grid(case["n"], 30, case["band"], case["seed"])
        thr = 0.5
    else:
        kw = {k: case[k] for k in ("n", "shape") if k in case}
        s, T, q = gridgen.make_config(case["name"], seed=case["seed"], **kw)
        thr = gridgen.config_threshold(case["name"])
    out = {"s": s, "T": T, "q": q, "activity_threshold": thr, "newton_tol": 1e-12, "newton_max_iter": 100}
    for v in (0, 1, 2):
        opts = O.Options(variant=v, activity_threshold=thr)
        for k in ("deep", "shallow"):
            r = O.ref_convection(k, s, T, q, opts)
            assert r.status == 0
            for f in ("tend_T", "tend_q", "precip", "work", "exited"):
                out[f"{k}_v{v}_{f}"] = getattr(r, f)
    return out


def main():
    if not O.ref_available():
        sys.exit("oracle/_ref/libconvref.so missing: run `make -C oracle ref` in the build container")
    for name, case in CASES.items():
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **make(case))
        print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
