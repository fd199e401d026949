#!/bin/bash
python -m pytest tests -m "gpu and slow" -x -q --durations=10 2>&1 | tail -20
