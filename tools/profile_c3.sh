#!/bin/bash
# Config-3 profiles (run under gpurun, 1 GPU): the default bench line, the
# launch list of one engine step (32 views, batched projections), and
# ncu --set full (plus FP32-pipe and L2-atomic counters) of the step's main
# kernels.   usage: bash tools/profile_c3.sh [tag]
set -u
TAG=${1:-c3}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err || { echo "bench failed"; tail gpurun_out/bench_$TAG.err; exit 1; }
PYTHONPATH=. python tools/prof_step.py 3 32 1 > gpurun_out/plain_step_$TAG.log 2>&1 || { echo "plain step failed"; tail gpurun_out/plain_step_$TAG.log; exit 1; }
PYTHONPATH=. ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/prof_step.py 3 32 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
PYTHONPATH=. ncu --profile-from-start off --set full --clock-control none --import-source on \
    --metrics sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active \
    -k regex:"views_project|onesweep|et_expand|et_colsum|et_colscan|et_place|tile_scan|raster_fwd|raster_bwd_rec" -c 14 \
    -o gpurun_out/prof_$TAG python tools/prof_step.py 3 32 1 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
# the projection backward runs once per step, after every view's raster
# backward: a second capture picks it out
PYTHONPATH=. ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"views_project_bwd" -c 1 \
    -o gpurun_out/prof_${TAG}_pbwd python tools/prof_step.py 3 32 1 > gpurun_out/ncu_pbwd_$TAG.log 2>&1
echo "pbwd rc=$?"
