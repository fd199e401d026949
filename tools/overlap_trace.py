"""Timeline evidence of the comm/compute overlap of the slabbed macro step (nsys is not in this
image; CUPTI activity tracing through torch.profiler records the library's kernels and copies
just the same).  Runs macro steps of a 3-D wave grid split into loopback slabs (the multi-GPU
halo code path on one GPU: the ghost-plane exchange is enqueued on the context's comm stream
while the interior planes are computed on the context stream, then one face-band launch), and
reports how much of the exchange time lies under interior kernels.

    python tools/overlap_trace.py [--n 512 512 256] [--slabs 4] [--out gpurun_out/overlap]
writes <out>.json (chrome trace) and prints a one-line JSON summary.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs=3, default=[512, 512, 256])
    ap.add_argument("--slabs", type=int, default=4)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--out", default="gpurun_out/overlap")
    a = ap.parse_args()
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    from gbs_inputs import reduced
    from gbs_inputs import make_ic
    from paper_1907_11771_b200 import gbs, scheme

    w = reduced("c5", tuple(a.n), macro_steps=a.steps)
    counts, ws, _ = scheme.weight_set(w.weights, w.steps)
    wd = scheme.to_fp64(ws)
    H = scheme.macro_step(w.pde, w.order, w.n, counts, wd, w.h_factor)
    opts = {"loopback": a.slabs, "graph": 0}
    opts.update({kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt})
    y0 = make_ic(w)
    st = gbs.Stepper(w.pde, w.n, w.order, counts, wd, **opts)
    st.write(torch.from_numpy(y0).cuda())
    st.advance(1, H)
    st.sync()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        st.advance(a.steps, H)
        st.sync()
    st.close()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    prof.export_chrome_trace(a.out + ".json")
    with open(a.out + ".json") as f:
        tr = json.load(f)
    ev = [e for e in tr.get("traceEvents", []) if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
    kern = [e for e in ev if e["cat"] == "kernel" and ("wave3d" in e["name"])]
    copies = [e for e in ev if e["cat"] == "gpu_memcpy"]
    streams = {}
    for e in kern:
        streams.setdefault(e["args"].get("stream"), []).append(e)
    # the interior launches run on the context stream (the one with the most stencil time)
    main_stream = max(streams, key=lambda s: sum(x["dur"] for x in streams[s])) if streams else None
    interior = sorted(((e["ts"], e["ts"] + e["dur"]) for e in streams.get(main_stream, [])))
    face = [e for s, es in streams.items() if s != main_stream for e in es]

    def covered(t0, t1):
        tot = 0.0
        for a0, a1 in interior:
            lo, hi = max(t0, a0), min(t1, a1)
            if hi > lo:
                tot += hi - lo
        return tot

    copy_us = sum(e["dur"] for e in copies)
    copy_under = sum(covered(e["ts"], e["ts"] + e["dur"]) for e in copies)
    face_us = sum(e["dur"] for e in face)
    face_under = sum(covered(e["ts"], e["ts"] + e["dur"]) for e in face)
    span = (max(e["ts"] + e["dur"] for e in ev) - min(e["ts"] for e in ev)) if ev else 0
    print(json.dumps({
        "grid": a.n, "slabs": a.slabs, "macro_steps": a.steps, "options": opts,
        "stencil_launches_context_stream": len(interior), "face_launches_comm_stream": len(face),
        "halo_copies": len(copies), "halo_copy_us": round(copy_us, 1),
        "halo_copy_us_under_interior_kernels": round(copy_under, 1),
        "halo_overlap_fraction": round(copy_under / copy_us, 4) if copy_us else None,
        "face_launch_us": round(face_us, 1), "face_launch_us_under_interior": round(face_under, 1),
        "interior_kernel_us": round(sum(b - a for a, b in interior), 1), "span_us": round(span, 1),
        "trace": a.out + ".json"}))


if __name__ == "__main__":
    main()
