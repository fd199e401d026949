#!/bin/bash
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
for f in 1 0; do timeout 300 python tools/probe_perf.py --config c5 --fuse $f; done
timeout 300 python tools/probe_perf.py --config c4 --fuse 1
