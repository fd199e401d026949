"""Histogram of the instructions inside the largest loop (backward branch span) of one kernel's SASS."""
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
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)(.*)", line)
        if m: buf[cur].append((int(m.group(1), 16), m.group(3), m.group(4)))
for name, ins in buf.items():
    if pat not in name:
        continue
    loops = []
    for addr, op, rest in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if t and int(t.group(1), 16) < addr:
                loops.append((addr - int(t.group(1), 16), int(t.group(1), 16), addr))
    loops.sort(reverse=True)
    print(name, "total", len(ins))
    for span, a, b in loops[:4]:
        body = [op for (ad, op, _) in ins if a <= ad <= b]
        c = Counter(o.split(".")[0] for o in body)
        print(f"  loop [{a:#x},{b:#x}] {len(body)} instr:", ", ".join(f"{k}:{v}" for k, v in c.most_common(25)))
