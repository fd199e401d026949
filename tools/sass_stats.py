"""Instruction histogram of one kernel's SASS (cuobjdump), by substring of its mangled name."""
import re, subprocess, sys
from collections import Counter
lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, buf = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); buf[cur] = []; continue
    if cur:
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m: buf[cur].append(m.group(2))
for name, ins in buf.items():
    if pat in name:
        c = Counter(ins)
        print(name, "total", len(ins))
        print("  ", ", ".join(f"{k}:{v}" for k, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30)))
