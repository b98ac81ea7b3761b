#!/bin/bash
# Config-3 profiles (run under gpurun, 1 GPU): the default bench line, the
# launch list of the bench command, and ncu --set full (plus FP32-pipe and
# L2-atomic counters) of one config-3 view's frame.   usage: bash tools/profile_c3.sh [tag]
set -u
TAG=${1:-c3}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err || { echo "bench failed"; tail gpurun_out/bench_$TAG.err; exit 1; }
CMD="python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain bench failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 600 --csv --log-file gpurun_out/launches_$TAG.csv \
    $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
PYTHONPATH=. python tools/prof_frame.py 3 > gpurun_out/plain_frame_$TAG.log 2>&1 || { echo "plain frame failed"; exit 1; }
PYTHONPATH=. ncu --set full --clock-control none --import-source on \
    --metrics sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active \
    -s 16 -c 24 -o gpurun_out/prof_$TAG python tools/prof_frame.py 3 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full rc=$?"
