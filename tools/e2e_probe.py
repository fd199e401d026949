import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
from gbs_inputs import get_config, make_ic
from paper_1907_11771_b200 import gbs, scheme
w = get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
counts, ws, _ = scheme.weight_set(w.weights, w.steps)
wd = scheme.to_fp64(ws)
H = scheme.macro_step(w.pde, w.order, w.n, counts, wd)
y0 = make_ic(w)
st = gbs.Stepper(w.pde, w.n, w.order, counts, wd, torch_memory=True)
h_in = torch.from_numpy(y0).pin_memory()
h_out = [torch.empty(y0.shape, dtype=torch.float64).pin_memory() for _ in range(2)]
st.write(y0); st.advance(2, H); st.sync()
for mode in ["async", "async_noread", "async_nowrite", "advance_only", "sync"]:
    gbs.gbs_sync(st.ctx)
    t0 = time.perf_counter(); tc = []
    K = 16
    for k in range(K):
        a = time.perf_counter()
        if mode in ("async", "async_noread"): gbs.gbs_write_slab_async(st.ctx, h_in)
        if mode == "sync": gbs.gbs_write_state(st.ctx, h_in)
        b = time.perf_counter()
        gbs.gbs_advance(st.ctx, 1, H)
        c = time.perf_counter()
        if mode in ("async", "async_nowrite"): gbs.gbs_read_slab_async(st.ctx, h_out[k % 2])
        if mode == "sync": gbs.gbs_read_state(st.ctx, h_out[k % 2])
        d = time.perf_counter()
        tc.append((b - a, c - b, d - c))
    gbs.gbs_sync(st.ctx)
    dt = time.perf_counter() - t0
    m = np.mean(np.array(tc), axis=0) * 1e3
    print(f"{mode:14s} {dt / K * 1e3:8.3f} ms/step  host call ms: write {m[0]:.3f} advance {m[1]:.3f} read {m[2]:.3f}")
