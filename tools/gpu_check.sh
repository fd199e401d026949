#!/bin/bash
# development: parity tests (not slow) then perf probes
set -x
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -30
for c in c5 c4 c3 c2; do timeout 300 python tools/probe_perf.py --config $c; done
