"""Quick per-kernel timing probe (development tool): time the stencil kernels of a config
through the C ABI with gbs_kernel_time (CUDA events on the context stream)."""
import argparse, json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gbs_inputs import get_config, reduced
from paper_1907_11771_b200 import gbs, scheme

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--macro", type=int, default=2)
ap.add_argument("--zchunk", type=int, default=0)
ap.add_argument("--n", type=str, default="")
ap.add_argument("--fuse", type=int, default=-1)
ap.add_argument("--opt", action="append", default=[], help="key=value (gbs_set_option)")
a = ap.parse_args()
w = get_config(a.config)
if a.n:
    w = reduced(a.config, tuple(int(x) for x in a.n.split(",")))
counts, ws, _ = scheme.weight_set(w.weights, w.steps)
wd = scheme.to_fp64(ws)
H = scheme.macro_step(w.pde, w.order, w.n, counts, wd)
y0 = torch.randn(w.state_shape, dtype=torch.float64, device="cuda")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
st = gbs.Stepper(w.pde, w.n, w.order, counts, wd, stream=stream.cuda_stream)
if a.zchunk: gbs.gbs_set_option(st.ctx, "zchunk", a.zchunk)
if a.fuse >= 0: gbs.gbs_set_option(st.ctx, "fuse", a.fuse)
for kv in a.opt:
    k, v = kv.split("="); gbs.gbs_set_option(st.ctx, k, int(v))
res_opts = dict(kv.split("=") for kv in a.opt)
st.write(y0)
st.advance(1, H); gbs.gbs_sync(st.ctx)
gbs.gbs_set_option(st.ctx, "time_kernels", 1)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); t0.record(stream)
st.advance(a.macro, H)
t1.record(stream); torch.cuda.synchronize(); gbs.gbs_sync(st.ctx)
tot = t0.elapsed_time(t1)
F = w.fields; pts = w.points
res = {"config": w.name, "opts": res_opts, "total_ms": tot, "macro": a.macro}
for cls, name in enumerate(["lf", "fe", "fin", "lf2", "lffin"]):
    ms, n = gbs.gbs_kernel_time(st.ctx, cls)
    if n == 0: continue
    per = ms / max(n, 1)
    byts = {0: 24, 1: 16, 2: 24, 3: 48, 4: 48}[cls] * F * pts
    res[name] = {"ms_per_launch": per, "launches": n, "GBps_alg": byts / (per * 1e-3) / 1e9}
S = w.substeps
res["Gpt_substeps_per_s"] = pts * S * a.macro / (tot * 1e-3) / 1e9
res["GBps_alg_total"] = res["Gpt_substeps_per_s"] * 24 * F
print(json.dumps(res))
st.close()
