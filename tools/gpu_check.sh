#!/bin/bash
set -x
python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15
