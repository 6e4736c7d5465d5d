"""Instructions executed (warp-level) and average active threads per CUDA
source line of one kernel in an ncu report (--import-source, -lineinfo):
python tools/ncu_inst.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout.splitlines()
res, fname, hdr = [], None, None
for r in csv.reader(out):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            inst = float(r[hdr.index("Instructions Executed")])
            thr = float(r[hdr.index("Avg. Threads Executed")] or 0)
        except ValueError:
            continue
        if inst > 0:
            res.append((inst, thr, fname, r[0], r[1].strip()[:80]))
tot = sum(x[0] for x in res) or 1
print(f"total warp instructions {tot:.4g}")
for inst, thr, f, ln, src in sorted(res, reverse=True)[:n]:
    print(f"{100*inst/tot:5.1f}%  {inst:10.4g}  thr {thr:4.1f}  {f}:{ln:5s} {src}")
