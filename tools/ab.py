"""Interleaved A/B timing of library options on ONE context (development tool).

Each round runs every option set in turn: set the options (gbs_set_option), one warm-up macro
step, then K macro steps timed with CUDA events on the context stream (graph replay, as the
bench's metric), then one macro step with time_kernels for the per-class launch times.
Rounds interleave the sets so the power-capped clock drifts equally over all of them.

    python tools/ab.py --config c5 --rounds 3 --steps 2 --set half=0 --set half=1 --set half=1,half_rpt=4
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gbs_inputs import get_config, make_ic, reduced  # noqa: E402
from paper_1907_11771_b200 import gbs, scheme  # noqa: E402

CLS = ["lf", "fe", "fin", "lf2", "lffin", "cluster", "half", "fea"]
# the library's defaults of the options a set may change (include/gbs.h)
DEFAULTS = {"half": 1, "half_fe": 0, "half_tall": 1, "half_rpt": 4, "l2hint_half": 11, "l2hint": 11,
            "l2hint_step": 0, "zchunk_fin": 0, "l2hint_fin": 11, "streams": 1, "fea": 1, "fea_ring": 1, "fin_ring": 0, "fuse": 1, "bulk": 1, "zchunk_pair": 0, "zchunk": 0, "band": 0, "overlap": 1}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--n", default="")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--set", action="append", default=[], help="comma-separated key=value options")
a = ap.parse_args()
w = get_config(a.config)
if a.n:
    w = reduced(a.config, tuple(int(x) for x in a.n.split(",")))
counts, ws, _ = scheme.weight_set(w.weights, w.steps)
wd = scheme.to_fp64(ws)
H = scheme.macro_step(w.pde, w.order, w.n, counts, wd, w.h_factor)
stream = torch.cuda.Stream()
sets = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in s.split(",") if kv) for s in (a.set or [""])]
keys = sorted({k for s in sets for k in s})
with torch.cuda.stream(stream):
    st = gbs.Stepper(w.pde, w.n, w.order, counts, wd, stream=stream.cuda_stream, torch_memory=True)
    st.write(torch.from_numpy(make_ic(w)).cuda())
    gbs.gbs_sync(st.ctx)
    res = {i: {"ms": [], "cls": {}} for i in range(len(sets))}
    for r in range(a.rounds):
        for i, s in enumerate(sets):
            for k in keys:                       # keys a set does not name take the library default
                gbs.gbs_set_option(st.ctx, k, s.get(k, DEFAULTS[k]))
            st.advance(1, H)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st.advance(a.steps, H)
            e1.record(stream)
            e1.synchronize()
            res[i]["ms"].append(e0.elapsed_time(e1) / a.steps)
            gbs.gbs_set_option(st.ctx, "time_kernels", 1)
            for c in range(len(CLS)):
                gbs.gbs_kernel_time(st.ctx, c, reset=True)
            st.advance(1, H)
            gbs.gbs_sync(st.ctx)
            for c, name in enumerate(CLS):
                ms, n = gbs.gbs_kernel_time(st.ctx, c, reset=True)
                if n:
                    res[i]["cls"].setdefault(name, []).append((ms / n, n))
            gbs.gbs_set_option(st.ctx, "time_kernels", 0)
    st.close()
S = w.substeps
for i, s in enumerate(sets):
    ms = statistics.median(res[i]["ms"])
    out = {"set": s, "ms_per_macro": round(ms, 3), "all_ms": [round(x, 2) for x in res[i]["ms"]],
           "G_pt_substeps_per_s": round(w.points * S / (ms * 1e-3) / 1e9, 2)}
    for name, v in res[i]["cls"].items():
        out[name] = {"ms": round(statistics.median(x[0] for x in v), 4), "n": v[0][1]}
    print(json.dumps(out), flush=True)
