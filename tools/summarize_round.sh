#!/bin/bash
# Turn what tools/final_round.sh <tag> left in gpurun_out/ into the tracked files under profiles/
# (run here, after the gpurun call came back).   usage: bash tools/summarize_round.sh <tag>
set -e
T=${1:?tag}
python tools/ncu_summary.py launches gpurun_out/launches_$T.csv profiles/${T}_config3_launches.txt > /dev/null
python tools/ncu_summary.py full gpurun_out/prof_$T.ncu-rep,gpurun_out/prof_${T}_pbwd.ncu-rep \
    profiles/${T}_config3_ncu_full.txt profiles/ncu_traffic.json > /dev/null
cp gpurun_out/bench_$T.json profiles/${T}_config3_bench.json
cp gpurun_out/bench_reference_$T.json profiles/${T}_config3_bench_reference.json
cp gpurun_out/gpu_tests_$T.log profiles/${T}_config3_gpu_tests.log
cp gpurun_out/parity_$T.json profiles/parity_r2.json
cp gpurun_out/parity_$T.log profiles/parity_r2.log
python tools/show_bench.py profiles/${T}_config3_bench.json
