import numpy as np, time, os
from concurrent.futures import ThreadPoolExecutor
n = 880*2**20//8
a = np.empty(n); a[:] = 1.0
b = np.empty(n); b[:] = 2.0
print("cpus", os.cpu_count())
for threads in (1, 4, 8, 16, 32):
    if threads > os.cpu_count(): break
    chunks = np.array_split(np.arange(n), threads)
    bounds = [(c[0], c[-1]+1) for c in chunks]
    def z(bb): a[bb[0]:bb[1]] = 0.0
    def cp(bb): a[bb[0]:bb[1]] = b[bb[0]:bb[1]]
    with ThreadPoolExecutor(threads) as ex:
        for f, name in ((z, "zero"), (cp, "copy")):
            best = 1e9
            for _ in range(3):
                t = time.perf_counter(); list(ex.map(f, bounds)); best = min(best, time.perf_counter() - t)
            print(f"threads {threads:2d} {name}: {880/1024/best:.1f} GB/s ({best*1e3:.1f} ms for 880 MB)")
