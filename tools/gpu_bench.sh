#!/bin/bash
# bench + ncu launch list + one full ncu capture of the dominant (two-substep) kernel
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
SHORT="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$SHORT > gpurun_out/short_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
PROBE="python tools/probe_perf.py --config c5 --macro 1"
$PROBE > gpurun_out/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wave3d_pair_tma -s 3 -c 1 -o gpurun_out/prof_pair_c5 $PROBE > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
