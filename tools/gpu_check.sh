#!/bin/bash
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
for c in c5 c4; do timeout 300 python tools/probe_perf.py --config $c --fuse 0; done
python tools/sass_stats.py paper_1907_11771_b200/lib/libgbs_b200.so "wave3d_step_tmaILi4ELi1ELb0" 12
