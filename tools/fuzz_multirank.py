"""Randomised multi-rank cases through the in-process transport (development tool): world,
sequence groups, grid shape, weights and options drawn from a seed; every rank's gathered state
against the oracle (rel-L2 <= 1e-12, per element <= 1e-11 of the maximum).
    python tools/fuzz_multirank.py [seed] [count]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import importlib.util  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

spec = importlib.util.spec_from_file_location("tm", os.path.join(ROOT, "tests", "test_multirank_gpu.py"))
tm = importlib.util.module_from_spec(spec)
spec.loader.exec_module(tm)
from gbs_inputs import reduced  # noqa: E402
from oracle import c_oracle as C  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
count = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rng = np.random.default_rng(seed)
bad = 0
for _ in range(count):
    cfg = str(rng.choice(["c2", "c3", "c4", "c5", "c1"]))
    world = int(rng.choice([2, 3, 4, 6, 8]))
    m = {"c1": 4, "c2": 6, "c3": 6, "c4": 6, "c5": 8}[cfg]
    gs = [g for g in range(1, world + 1) if world % g == 0 and g <= m]
    if cfg == "c1":
        gs = [g for g in gs if g == world]
        if not gs:
            continue
    groups = int(rng.choice(gs))
    slabs = world // groups
    if cfg in ("c4", "c5"):
        nz = max(int(rng.choice([4, 6, 8, 12])) * slabs * 2, 9 + (-9) % slabs)   # >= 2r + 1
        n = (int(rng.choice([64, 128, 40, 72])), int(rng.choice([16, 32, 36])), nz)
    elif cfg in ("c2", "c3"):
        R = 2 if cfg == "c2" else 4
        rows = int(rng.choice([R, 16, 24, 32]))
        while rows * slabs < 2 * R + 1:                                           # >= 2r + 1
            rows += R
        n = (int(rng.choice([64, 128, 96, 80])), rows * slabs, 1)
    else:
        n = (int(rng.choice([64, 256, 300])), 1, 1)
    wset = "square8" if cfg == "c1" else str(rng.choice(["nonzero8", "fallback8"]))
    opts = {"overlap": int(rng.integers(0, 2))}
    if cfg in ("c4", "c5"):
        opts.update(fuse=int(rng.integers(0, 2)), half=int(rng.integers(0, 2)), fea=int(rng.integers(0, 2)))
        if groups > 1 and n[0] % 64 == 0 and n[1] % 16 == 0:
            opts["fused_combine"] = int(rng.integers(0, 2))
    try:
        w = reduced(cfg, n, macro_steps=2, weights=wset)
        counts, wd, H = tm.scheme_for(w, wset, cfg)
        y0, outs, infos = tm.run_ranks(torch, w, counts, wd, H, 2, world, groups, opts)
        assert infos[0]["groups"] == groups, (infos[0]["groups"], groups)
        ref = C.advance(w.pde, w.order, y0, counts, wd, H, 2)
        for o in outs:
            rel, _, mmax = tm.errors(o, ref)
            assert rel <= 1e-12 and mmax <= 1e-11, (rel, mmax)
    except Exception as e:    # noqa: BLE001
        bad += 1
        print("FAIL", cfg, n, world, groups, wset, opts, repr(e)[:300], flush=True)
print(f"multirank fuzz seed={seed}: {count - bad}/{count} passed")
