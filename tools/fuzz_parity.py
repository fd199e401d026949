"""One-off fuzzing of launch variants (development tool): many seeded random cases of
tests/test_parity_gpu.py::_random_cases, each against the oracle.  Usage:
    python tools/fuzz_parity.py [seed] [count]"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import importlib.util

import torch

spec = importlib.util.spec_from_file_location("tp", os.path.join(ROOT, "tests", "test_parity_gpu.py"))
tp = importlib.util.module_from_spec(spec)
spec.loader.exec_module(tp)
from paper_1907_11771_b200 import gbs

gbs.load()
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
count = int(sys.argv[2]) if len(sys.argv) > 2 else 100
bad = 0
for cfg, n, opts in tp._random_cases(seed, count, include_1d=True):
    try:
        wset = "square8" if cfg == "c1" else "nonzero8"
        w = tp.reduced(cfg, n, macro_steps=2, weights=wset)
        counts, wd, H = tp.scheme_for(w, wset)
        y0, g, _ = tp.run_gpu(torch, w, counts, wd, H, 2, opts=opts)
        o = tp.run_oracle(w, y0, counts, wd, H, 2)
        tp.assert_parity(g[0], o[0], what=f"{cfg} {n} {opts}")
    except Exception as e:
        bad += 1
        print("FAIL", cfg, n, opts, repr(e)[:300])
print(f"fuzz seed={seed}: {count - bad}/{count} passed")
