"""One step with CVG_TRACE: per-block (kernel, SM, start, end) timeline summary.

python tools/trace_overlap.py [config] [R/W]   (R/W: rank R's share of a W-way partition)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen, multigpu
os.environ.setdefault("CVG_TRACE", "gpurun_out/trace.txt")
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
s, T, q = gridgen.make_config(cfg, seed=42)
thr = gridgen.config_threshold(cfg)
if len(sys.argv) > 2:
    r, w = (int(x) for x in sys.argv[2].split("/"))
    b = multigpu.rank_bounds(s, thr, w)
    lo, hi = int(b[r]), int(b[r + 1])
    s, T, q = s[lo:hi], np.ascontiguousarray(T[:, lo:hi]), np.ascontiguousarray(q[:, lo:hi])
dev = torch.device("cuda", 0)
ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s, T, q))
L, n = T.shape
mk = lambda: (torch.empty((L, n), dtype=torch.float64, device=dev), torch.empty((L, n), dtype=torch.float64, device=dev),
              torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.int64, device=dev),
              torch.empty(n, dtype=torch.uint8, device=dev))
ctx = P.Context(0)
do, so = mk(), mk()
opts = P.KernelOptions(activity_threshold=thr)
for _ in range(3):
    ctx.convect_async(ds, dT, dq, do, so, opts)
    ctx.check()
rows = [l.split() for l in open(os.environ["CVG_TRACE"])]
t0 = min(int(r[2]) for r in rows)
tend = max(int(r[3]) for r in rows)
print(f"{cfg} n={n}: trace span {(tend - t0) / 1e3:.1f} us")
for kind in ("deep", "shallow"):
    rr = [(int(r[1]), (int(r[2]) - t0) / 1e3, (int(r[3]) - t0) / 1e3) for r in rows if r[0] == kind]
    if not rr:
        continue
    st = np.array([x[1] for x in rr]); en = np.array([x[2] for x in rr])
    print(f"{kind}: blocks {len(rr)} start [{st.min():.1f}, {np.median(st):.1f}, {st.max():.1f}] us  "
          f"end [{en.min():.1f}, {np.percentile(en, 10):.1f}, {np.median(en):.1f}, {np.percentile(en, 90):.1f}, {en.max():.1f}] us")
    if kind == "shallow":
        dmax = max((int(r[3]) - t0) / 1e3 for r in rows if r[0] == "deep")
        print(f"  shallow blocks finished before deep end: {(en <= dmax).sum()} / {len(en)}")
# active blocks over time (10 bins)
span = (tend - t0) / 1e3
for kind in ("deep", "shallow"):
    rr = [((int(r[2]) - t0) / 1e3, (int(r[3]) - t0) / 1e3) for r in rows if r[0] == kind]
    bins = np.linspace(0, span, 11)
    act = [sum(1 for a, b in rr if a < hi_ and b > lo_) for lo_, hi_ in zip(bins[:-1], bins[1:])]
    print(f"{kind:8s} active blocks per {span / 10:.1f} us bin: {act}")
