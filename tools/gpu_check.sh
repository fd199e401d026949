#!/bin/bash
set -x
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -5
for z in 128 256 512; do timeout 300 python tools/probe_perf.py --config c5 --zchunk $z; done
timeout 300 python tools/probe_perf.py --config c4
