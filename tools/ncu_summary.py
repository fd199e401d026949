"""Summarise ncu output for profiles/: kernel share of a launch list, and the key
metrics of a --set full capture (run here, on the CPU box, with `ncu -i`).

    python tools/ncu_summary.py launches <launches.csv>            > profiles/rNN_launch_shares.txt
    python tools/ncu_summary.py full <prof.ncu-rep> [--traffic CFG] > profiles/rNN_ncu_<kernel>.txt
    python tools/ncu_summary.py stalls <prof.ncu-rep>                > profiles/rNN_ncu_<kernel>_stalls.txt
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

TO_MS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
        "launch__shared_mem_per_block_dynamic"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        ms = float(r[vi].replace(",", "")) * TO_MS[r[ui]]
        tot[r[ki].split("(")[0]] += ms
        cnt[r[ki].split("(")[0]] += 1
    T = sum(tot.values())
    print(f"# ncu launch list ({path}): {sum(cnt.values())} launches, {T:.2f} ms total "
          f"(cold-cache, serialised: compare shares, not absolutes)")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:48s} launches={cnt[k]:5d}  total_ms={tot[k]:10.3f}  avg_ms={tot[k] / cnt[k]:8.4f}  "
              f"share={tot[k] / T:.4f}")


def full(path, traffic_cfg=None, cls=0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"# ncu --set full: {d.get('Kernel Name')}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:60s} {r[i]:>20s} {units[i]}")
        rd = float(d["dram__bytes_read.sum"]) * (1e9 if units[hdr.index("dram__bytes_read.sum")] == "Gbyte" else 1)
        wr = float(d["dram__bytes_write.sum"]) * (1e9 if units[hdr.index("dram__bytes_write.sum")] == "Gbyte" else 1)
        print(f"  dram bytes per launch (read + write) = {rd + wr:.6g}")
        if traffic_cfg:
            json.dump({"config": traffic_cfg, "class": cls, "lf_dram_bytes_per_launch": rd + wr,
                       "source": os.path.basename(path), "kernel": d.get("Kernel Name")},
                      open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "profiles", "ncu_traffic.json"), "w"), indent=1)
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    si, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    keep = {"GPU Speed Of Light Throughput", "Memory Workload Analysis", "Scheduler Statistics",
            "Warp State Statistics", "Occupancy", "Compute Workload Analysis"}
    print("# sections")
    for r in rows[1:]:
        if r[si] in keep:
            print(f"  {r[si][:28]:28s} {r[mi][:52]:52s} {r[vi]:>16s} {r[ui]}")


def stalls(path, top=10, skip=0):
    """Warp-stall sampling totals and the instructions with the most samples per reason
    (source page, SASS view; needs --import-source / -lineinfo) of the profiled launch `skip`."""
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr, data = rows[hi], []
    for r in rows[hi + 1:]:                 # the first kernel's table only
        if len(r) != len(hdr) or r[0] == "Address":
            break
        data.append(r)

    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    si = hdr.index("Warp Stall Sampling (All Samples)")
    total = sum(num(r[si]) for r in data)
    cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    print(f"# warp-stall samples ({os.path.basename(path)}, {rows[0][1] if len(rows[0]) > 1 else ''}): "
          f"{total:.0f} samples")
    sums = sorted(((sum(num(r[i]) for r in data), h, i) for i, h in cols), reverse=True)
    for v, h, _ in sums:
        if v > 0:
            print(f"  {h:28s} {v:10.0f}  {v / total:6.1%}")
    for v, h, i in sums[:4]:
        print(f"# top instructions by {h}")
        for r in sorted(data, key=lambda r: -num(r[i]))[:top]:
            print(f"  {r[0][-6:]} {num(r[i]):9.0f}  {r[1].strip()[:90]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "stalls":
        stalls(sys.argv[2], skip=int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else 0)
    else:
        cfg = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
        cls = int(sys.argv[sys.argv.index("--class") + 1]) if "--class" in sys.argv else 0
        full(sys.argv[2], cfg, cls)
