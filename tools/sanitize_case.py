"""Small runs through every kernel family, for compute-sanitizer (development tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gbs_inputs import make_ic, reduced
from paper_1907_11771_b200 import gbs, scheme

cases = [("c1", (77, 1, 1), {"persistent": 1}), ("c1", (77, 1, 1), {"persistent": 0}),
         ("c2", (70, 34, 1), {}), ("c3", (72, 40, 1), {"loopback": 2}),
         ("c4", (65, 33, 20), {}), ("c4", (64, 32, 20), {"fuse": 0}), ("c4", (64, 32, 20), {"fuse": 1}),
         ("c5", (64, 16, 24), {"fuse": 1, "loopback": 3}), ("c5", (64, 16, 24), {"fuse": 0, "loopback": 2}),
         ("c2", (128, 64, 1), {}), ("c3", (128, 96, 1), {"loopback": 2}),          # 2-D TMA kernel
         ("c5", (64, 48, 60), {"loopback": 3, "overlap": 1})]                         # overlapped halos
for cfg, n, opts in cases:
    w = reduced(cfg, n, macro_steps=1, weights="nonzero8" if cfg != "c1" else None)
    counts, ws, _ = scheme.weight_set(w.weights, w.steps)
    wd = scheme.to_fp64(ws)
    H = scheme.macro_step(w.pde, w.order, w.n, counts, wd)
    y0 = torch.from_numpy(make_ic(w)).cuda()
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd, **opts) as st:
        st.write(y0)
        st.advance(2, H)
        out = torch.empty_like(y0)
        st.read(out)
        assert torch.isfinite(out).all()
    print(cfg, n, opts, "ok", flush=True)
print("all ok")
