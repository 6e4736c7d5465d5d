"""PCIe floor for the e2e path: pinned H2D of the step's inputs, D2H of its
outputs, separately and concurrently on two streams (C4 sizes by default)."""
import sys
import time

import torch

h2d_mb = float(sys.argv[1]) if len(sys.argv) > 1 else 431.75
d2h_mb = float(sys.argv[2]) if len(sys.argv) > 2 else 879.43
dev = torch.device("cuda", 0)
hi = torch.empty(int(h2d_mb * 1e6), dtype=torch.uint8).pin_memory()
ho = torch.empty(int(d2h_mb * 1e6), dtype=torch.uint8).pin_memory()
di = torch.empty_like(hi, device=dev)
do = torch.empty_like(ho, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    best = 1e9
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                di.copy_(hi, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                ho.copy_(do, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


th = run(True, False)
td = run(False, True)
tb = run(True, True)
print(f"h2d {h2d_mb:.0f} MB {th:.2f} ms ({h2d_mb / th:.1f} GB/s); d2h {d2h_mb:.0f} MB {td:.2f} ms "
      f"({d2h_mb / td:.1f} GB/s); both concurrent {tb:.2f} ms")
