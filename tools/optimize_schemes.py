"""Generate the Appendix-B optimised weight sets for the configs' step sets (SURVEY.md
§8(f) NEXT-1) and write gbs_inputs/optimized_schemes.json (input data: free weights,
read by both the product and the oracle, which each compute the dependent weights).

    python tools/optimize_schemes.py

Order 8 with n_dep = {2,4,6,8} (the square set the configs fall back to) and the other
counts free, optimised for the imaginary stability boundary by
paper_1907_11771_b200.optimize (App. B, robust weighted-margin form; every
accepted step is re-checked by the independent ISB scan of the fp64 scheme).  Exact
weights are stored as "num/den" strings.
"""
import json
import os
import sys
import time
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_11771_b200 import optimize as O   # noqa: E402

SETS = {
    "opt8_12": ((2, 4, 6, 8), (10, 12), 3.8, 9.0),
    "opt8_16": ((2, 4, 6, 8), (10, 12, 14, 16), 3.8, 13.0),
}


def main():
    out = {}
    for name, (nd, nf, lo, hi) in SETS.items():
        t = time.time()
        counts, ws, isb = O.optimized_scheme(nd, nf, lo, hi, tol=1e-3, samples=1500)
        out[name] = {"order": 8, "n_dep": list(nd), "n_free": list(nf),
                     "c_free": [str(Fraction(w)) for n, w in zip(counts, ws) if n in nf],
                     "isb_scan": isb,
                     "note": "PAPER.md App. B optimiser (paper_1907_11771_b200/optimize.py), "
                             "weighted-margin subproblem, bisection tol 1e-3, 1500 samples"}
        print(name, counts, [float(w) for w in ws], isb, f"{time.time() - t:.1f}s", flush=True)
    path = os.path.join(ROOT, "gbs_inputs", "optimized_schemes.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
