"""Local-memory (spill) instructions per source line of one kernel: python tools/spills.py lib.so kernel_substr"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

so, kname = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = out.split("\n")
st = [i for i, l in enumerate(lines) if l.startswith(".text.") and kname in l][0]
en = st + 1
while en < len(lines) and not lines[en].startswith(".text."):
    en += 1
cur = None
cnt = Counter()
n = 0
for l in lines[st:en]:
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    if re.search(r"/\*[0-9a-f]{4,}\*/", l):
        n += 1
        if re.search(r"\b(LDL|STL)", l):
            cnt[cur] += 1
print("instructions", n, "local ld/st", sum(cnt.values()))
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:30]:
    print(k, v)
