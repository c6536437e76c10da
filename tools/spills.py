"""Spill (STL/LDL) sites and instruction count of one kernel in an object
file, attributed to source lines (profiling aid, not product code).
usage: python tools/spills.py obj.o kernel_mangled_substring"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

obj, name = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = txt.split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and name in l)
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//----")), len(lines))
cur = None
spill, n = Counter(), 0
for l in lines[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,5}\*/", l):
        n += 1
        if re.search(r"\b(STL|LDL)\b", l):
            spill[cur] += 1
print(lines[start].strip(), "instructions", n)
for k, v in spill.most_common(30):
    print(f"  {k[0]}:{k[1]}  {v}")
