"""Print the SASS of one kernel (substring match on the mangled name) from
libconvgpu.so, instruction lines only."""
import re
import subprocess
import sys

pat = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1711_00289_b200/libconvgpu.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
on = False
for line in out.splitlines():
    if "Function :" in line:
        on = pat in line
        if on:
            print(line.strip())
        continue
    if on:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            print(m.group(1), m.group(2))
