#!/bin/bash
set -x
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -5
python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --config c4 2>&1 | tail -1
