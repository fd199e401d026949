#!/bin/bash
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
python bench.py --config c4 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline | cut -c1-300
