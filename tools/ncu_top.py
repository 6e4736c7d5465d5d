"""Top SASS instructions of a kernel by stall samples, with their main stall reasons."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
exec_filter = int(sys.argv[4]) if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out)); hdr = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if len(r) == len(hdr) and r[0] != "Address" and r[0] not in seen:
        seen.add(r[0]); data.append(r)
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed"); iSrc = hdr.index("Source")
f = lambda x: float(x) if x.replace('.', '', 1).isdigit() else 0.0
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
idx = {r[0]: i for i, r in enumerate(data)}
sel = [r for r in data if exec_filter is None or int(f(r[iE])) == exec_filter]
for r in sorted(sel, key=lambda r: -f(r[iS]))[:n]:
    st = sorted(((f(r[i]), hdr[i][6:]) for i in sc), reverse=True)[:3]
    print(f"{idx[r[0]]:5d} {f(r[iS]):6.0f} {r[iSrc][:60]:60s} " + " ".join(f"{k}={v:.0f}" for v, k in st if v > 0))
