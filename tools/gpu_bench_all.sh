#!/bin/bash
# one bench line per BASELINE.json config (c5 is the default bench workload)
cd $GRAFT_REPO_ROOT
for c in c1 c2 c3 c4 c5; do
  python bench.py --config $c --steps 4 --warmup 3 --e2e-steps 1 2>/dev/null | tail -1
done > gpurun_out/bench_all.jsonl
