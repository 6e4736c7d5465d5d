"""Deep-worker phase breakdown (debug build tools/libconvgpu_phases.so, built
with -DCVG_PHASE_CLOCKS): SM cycles per phase summed over warps, for one
deep-only call on the f02 grid."""
import ctypes as C
import os
import sys

os.environ["CONVGPU_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("PHASES_LIB", "libconvgpu_phases.so"))

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
out = (C.c_ulonglong * 8)()
for rep in range(3):
    ctx.convect_async(ds, dT, dq, do, None, kernels=P.DEEP, stream=st)
    ctx.check(st)
    P.load_library().cvg_debug_phases(out)
names = ["prologue (wait, stage, guess, e0)", "levels (m, y, Newton, sin, tend)", "reductions",
         "group flush + advance", "  of which relaxed FP64 Newton loop", "  of which FP32 far loop", "  of which staged-column wait"]
tot = sum(out[i] for i in range(4))
trig = int((s > 0.5).sum())
for i, nm in enumerate(names):
    print(f"{nm:40s} {out[i] / 1e9:8.3f} Gcyc  {100 * out[i] / tot:5.1f}%  {out[i] / trig:9.0f} cyc/column")
