"""One C4 step with CVG_TRACE: per-block (kernel, SM, start, end) timeline summary."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen
os.environ.setdefault("CVG_TRACE", "gpurun_out/trace.txt")
s, T, q = gridgen.make_config("c4", seed=42)
dev = torch.device("cuda", 0)
ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s, T, q))
L, n = T.shape
mk = lambda: (torch.empty((L, n), dtype=torch.float64, device=dev), torch.empty((L, n), dtype=torch.float64, device=dev),
              torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.int64, device=dev),
              torch.empty(n, dtype=torch.uint8, device=dev))
ctx = P.Context(0)
do, so = mk(), mk()
for _ in range(3):
    ctx.convect_async(ds, dT, dq, do, so)
    ctx.check()
rows = [l.split() for l in open(os.environ["CVG_TRACE"])]
t0 = min(int(r[2]) for r in rows)
for kind in ("deep", "shallow"):
    rr = [(int(r[1]), (int(r[2]) - t0) / 1e3, (int(r[3]) - t0) / 1e3) for r in rows if r[0] == kind]
    st = np.array([x[1] for x in rr]); en = np.array([x[2] for x in rr])
    print(f"{kind}: blocks {len(rr)} start [{st.min():.1f}, {np.median(st):.1f}, {st.max():.1f}] us  end [{en.min():.1f}, {np.median(en):.1f}, {en.max():.1f}] us")
    if kind == "shallow":
        dmax = max(x[2] for x in [(int(r[1]), 0, (int(r[3]) - t0) / 1e3) for r in rows if r[0] == "deep"])
        print(f"  shallow blocks finished before deep end: {(en <= dmax).sum()} / {len(en)}")
