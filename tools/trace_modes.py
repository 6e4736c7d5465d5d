"""Repeated traced steps (CVG_TRACE): per repetition the step span, deep and
shallow block start/end spreads and how many SMs ran deep and shallow blocks
at the same time -- to tell apart overlapped and serialised schedules."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen, multigpu
os.environ.setdefault("CVG_TRACE", "gpurun_out/trace.txt")
s, T, q = gridgen.make_config("c4", seed=42)
if len(sys.argv) > 1:
    r, w = (int(x) for x in sys.argv[1].split("/"))
    b = multigpu.rank_bounds(s, 0.5, w)
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
for rep in range(int(os.environ.get("REPS", "8"))):
    for _ in range(20):
        ctx.convect_async(ds, dT, dq, do, so)
    ctx.check()
    rows = [l.split() for l in open(os.environ["CVG_TRACE"])]
    t0 = min(int(r[2]) for r in rows)
    dp = [(int(r[1]), (int(r[2]) - t0) / 1e3, (int(r[3]) - t0) / 1e3) for r in rows if r[0] == "deep"]
    sh = [(int(r[1]), (int(r[2]) - t0) / 1e3, (int(r[3]) - t0) / 1e3) for r in rows if r[0] == "shallow"]
    span = max(x[2] for x in dp + sh)
    dstart = np.array([x[1] for x in dp]); dend = np.array([x[2] for x in dp])
    sstart = np.array([x[1] for x in sh]); send = np.array([x[2] for x in sh])
    # SMs where a shallow block ran while that SM's deep block was running
    dsm = {x[0]: (x[1], x[2]) for x in dp}
    co = len({sm for sm, a, b_ in sh if sm in dsm and a < dsm[sm][1] and b_ > dsm[sm][0]})
    print(f"rep {rep}: span {span:6.1f} us | deep start med {np.median(dstart):6.1f} max {dstart.max():6.1f} end med {np.median(dend):6.1f} max {dend.max():6.1f} "
          f"| shallow start min {sstart.min():6.1f} med {np.median(sstart):6.1f} end max {send.max():6.1f} | SMs co-running {co}")
