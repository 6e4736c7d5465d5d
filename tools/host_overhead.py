"""Host enqueue time of convect_async versus device time per step (is a small
step host-bound?).  python tools/host_overhead.py [R/W]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1711_00289_b200 as P
from paper_1711_00289_b200 import gridgen, multigpu
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
st = torch.cuda.Stream()
for _ in range(5):
    ctx.convect_async(ds, dT, dq, do, so, stream=st)
torch.cuda.synchronize()
K = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
t0 = time.perf_counter()
for _ in range(K):
    ctx.convect_async(ds, dT, dq, do, so, stream=st)
t1 = time.perf_counter()
e1.record(st)
torch.cuda.synchronize()
print(f"n={n}: host enqueue {1e6 * (t1 - t0) / K:.1f} us/step, device {1e3 * e0.elapsed_time(e1) / K:.1f} us/step")
# the same with bench.py's NVML clock sampler thread running
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler
with ClockSampler(0):
    e0.record(st)
    t0 = time.perf_counter()
    for _ in range(K):
        ctx.convect_async(ds, dT, dq, do, so, stream=st)
    t1 = time.perf_counter()
    e1.record(st)
    torch.cuda.synchronize()
print(f"with clock sampler: host enqueue {1e6 * (t1 - t0) / K:.1f} us/step, device {1e3 * e0.elapsed_time(e1) / K:.1f} us/step")
