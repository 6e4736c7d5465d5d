import numpy as np, sys
sys.path.insert(0, '.')
import oracle as O, paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen as G
for cfg in ["c5_95", "c4"]:
    s, T, q = G.make_config(cfg, seed=42)
    od = O.convection("deep", s, T, q)
    with P.Context(0) as ctx:
        for far in (True, False):
            d, _ = ctx.convect(s, T, q, P.KernelOptions(far32=far), kernels=P.DEEP)
            flip = d.work_units != od.work
            for f in ("tend_T", "tend_q", "precip"):
                a, b = getattr(d, f), getattr(od, f)
                bad = np.abs(a - b) > np.maximum(1e-10 * np.abs(b), 1e-14)
                if bad.ndim == 2: badc = bad.any(axis=0)
                else: badc = bad
                idx = np.nonzero(badc)[0]
                print(cfg, "far", far, f, "bad cols", idx[:5], "flip", flip[idx][:5], "margin", od.margin[idx][:5],
                      "got", a[..., idx][:5] if a.ndim==1 else None, "want", b[idx][:5] if b.ndim==1 else None)
            print(cfg, "far", far, "flips", flip.sum(), "maxrel precip among nonflip",
                  np.max((np.abs(d.precip - od.precip) / np.maximum(np.abs(od.precip), 1e-300))[~flip]))
