"""Evidence table for the TMA/mbarrier kernels: per kernel of libgbs_b200.so, counts of the SASS
instructions that prove the Blackwell data path (B200_PROFILING.md "What proves a Blackwell-native
kernel": UTMALDG = cp.async.bulk.tensor loads, SYNCS = mbarrier operations, UBLKCP = bulk copies),
plus the FP64 and shared-memory instruction counts of the same kernels and their registers.

    python tools/sass_counts.py [lib] > profiles/r02_sass_counts.txt
"""
import re
import subprocess
import sys
from collections import Counter

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1907_11771_b200/lib/libgbs_b200.so"
KEYS = ["UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "UTMAPF", "DFMA", "DADD", "DMUL", "LDS", "LDG", "STG", "SHFL"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True, check=True).stdout
regs = {}
cur = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        cur = m.group(1)
    m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
    if m and cur:
        regs[cur] = (int(m.group(1)), int(m.group(2)))
buf, cur = {}, None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        buf[cur] = Counter()
        continue
    if cur:
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", line)
        if m:
            buf[cur][m.group(2)] += 1


def short(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


print("# SASS instruction counts per kernel (cuobjdump -sass %s); static counts, not executed" % LIB)
print("# kernel | regs | " + " | ".join(KEYS))
for name in sorted(buf):
    if not any(k in name for k in ("tma", "cluster", "wave3d", "acoustic2d", "adv1d", "spectral", "local_sum")):
        continue
    c = buf[name]
    r = regs.get(name, ("?", "?"))[0]
    print(f"{short(name)[:110]} | {r} | " + " | ".join(str(sum(v for k, v in c.items() if k.startswith(key)))
                                                     for key in KEYS))
