"""Deep kernel time vs Newton work: times deep-only calls on the f02 grid at
several newton_tol values (fewer updates per solve as tol grows) and fits
time = a * columns + b * warp-iterations, splitting per-column overhead from
Newton-loop cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen

s, T, q = gridgen.make_config("c4", seed=42)
dev = torch.device("cuda", 0)
ds, dT, dq = (torch.from_numpy(a).to(dev) for a in (s, T, q))
L, n = T.shape
mk = lambda: (torch.empty((L, n), dtype=torch.float64, device=dev), torch.empty((L, n), dtype=torch.float64, device=dev),
              torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.int64, device=dev),
              torch.empty(n, dtype=torch.uint8, device=dev))
ctx = P.Context(0)
do = mk()
st = torch.cuda.Stream()
rows = []
for tol in (1e-12, 1e-9, 1e-6, 1e-3, 1e-1, 10.0):
    o = P.KernelOptions(newton_tol=tol)
    for _ in range(2):
        ctx.convect_async(ds, dT, dq, do, None, o, kernels=P.DEEP, stream=st)
        ctx.check(st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        ctx.convect_async(ds, dT, dq, do, None, o, kernels=P.DEEP, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    work = int(do[3].sum().item())
    trig = int((s > 0.5).sum())
    rows.append((tol, ms, work, trig))
    print(f"tol {tol:8.0e}  {ms:.4f} ms  updates {work}  per column {work / trig:.1f}", flush=True)
A = np.array([[1.0, r[2] / 60.0] for r in rows])   # per-lane-solve-pair iterations ~ work / 60 per column... summed
y = np.array([r[1] for r in rows])
coef, *_ = np.linalg.lstsq(A, y, rcond=None)
print(f"fit: ms = {coef[0]:.4f} + {coef[1] * 1e6:.4f}e-6 * (updates / 60)")
