"""Per CUDA source line: executed warp instructions and stall samples of a
kernel (ncu source page, sass+cuda), sorted by instructions."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout.splitlines()
num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
res, fname, hdr = [], None, None
for r in csv.reader(out):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iE = hdr.index("Instructions Executed")
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        res.append((num(r[iE]), num(r[4]), fname, r[0], r[1].strip()[:80]))
ti = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
for e, s, f, ln, src in sorted(res, reverse=True)[:n]:
    print(f"inst {100*e/ti:5.1f}%  samp {100*s/ts:5.1f}%  {f}:{ln:5s} {src}")
