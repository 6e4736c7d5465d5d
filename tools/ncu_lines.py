"""Warp-stall samples of a kernel aggregated by CUDA source line (needs
-lineinfo and --import-source): top lines with their main stall reasons."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout.splitlines()
res, fname, hdr = [], None, None
num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
for r in csv.reader(out):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        s = num(r[4])
        if s > 0:
            st = sorted(((num(r[i]), hdr[i][6:]) for i in range(len(hdr))
                         if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]), reverse=True)[:3]
            res.append((s, fname, r[0], r[1].strip()[:72], st))
tot = sum(x[0] for x in res) or 1
for s, f, ln, src, st in sorted(res, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:5s} {src:72s} " + " ".join(f"{k}={v:.0f}" for v, k in st if v > 0))
