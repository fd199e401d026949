#!/bin/bash
cd $GRAFT_REPO_ROOT
PROBE="python tools/probe_perf.py --config c4 --macro 1 --fuse 1"
$PROBE > gpurun_out/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wave3d_pair_tma -s 3 -c 1 -o gpurun_out/prof_pair4 $PROBE > gpurun_out/ncu_pair.log 2>&1; echo "ncu rc=$?"
