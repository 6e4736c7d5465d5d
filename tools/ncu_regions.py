"""Summarise an ncu source (SASS) page: samples grouped by execution count
(loop bodies share a count) and the top stall reasons."""
import csv, collections, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if len(r) == len(hdr) and r[0] != "Address" and r[0] not in seen:
        seen.add(r[0]); data.append(r)
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed"); iSrc = hdr.index("Source")
f = lambda x: float(x) if x.replace('.', '', 1).isdigit() else 0.0
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
by = collections.defaultdict(lambda: [0.0, 0, collections.Counter()])
for r in data:
    e = int(f(r[iE])); b = by[e]; b[0] += f(r[iS]); b[1] += 1
    for i in stall_cols: b[2][hdr[i]] += f(r[i])
tot = sum(v[0] for v in by.values()) or 1
print(f"total samples {tot:.0f}")
for e, v in sorted(by.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 8]:
    top = ", ".join(f"{k[6:]}={c:.0f}" for k, c in v[2].most_common(4))
    print(f"exec={e:9d} ninstr={v[1]:4d} samples={v[0]:7.0f} ({100*v[0]/tot:4.1f}%)  {top}")
