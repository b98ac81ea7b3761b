#!/bin/bash
# Profiles for the judged bench line (run under gpurun, 1 GPU):
#   launch list of the bench command + ncu --set full of one config-1 frame.
set -u
CMD="python bench.py --config 1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
PYTHONPATH=. python tools/prof_frame.py 1 > gpurun_out/plain_frame.log 2>&1 || { echo "plain frame failed"; exit 1; }
PYTHONPATH=. ncu --set full --clock-control none --import-source on -s 0 -c 40 -o gpurun_out/prof_c1 \
    python tools/prof_frame.py 1 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
