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
    -k regex:"views_project|depth_hist|onesweep|et_count|et_scan|et_emit|tile_scan|raster_fwd|raster_bwd_rec" -c 13 \
    -o gpurun_out/prof_$TAG python tools/prof_step.py 3 32 1 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
