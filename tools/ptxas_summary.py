"""Registers and spills per kernel from `nvcc -Xptxas -v` output (stdin):
python tools/ptxas_summary.py [substring] < build.log"""
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur and "spill stores" in line:
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        rows.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    if cur and "Used" in line:
        m = re.search(r"Used (\d+) registers", line)
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
names = {}
if rows:
    out = subprocess.run(["c++filt"], input="\n".join(rows), capture_output=True, text=True).stdout.split("\n")
    names = dict(zip(rows, out))
for k, v in rows.items():
    n = names.get(k, k)
    if pat in n:
        print(f"{v.get('regs', '?'):>4} regs  spill {v.get('spill', ('?', '?'))}  {n}")
