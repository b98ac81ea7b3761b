#!/bin/bash
# End-of-round evidence (run under gpurun, 1 GPU): the GPU test suite, the per-config parity report,
# the config-3 bench line + launch list + ncu --set full (tools/profile_c3.sh), and the reference arm.
#   usage: bash tools/final_round.sh <tag>
TAG=${1:-final}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
bash tools/profile_c3.sh $TAG
python bench.py --impl reference > gpurun_out/bench_reference_$TAG.json 2> gpurun_out/bench_reference_$TAG.err; echo "reference arm rc=$?"
python tests/parity_report.py --out gpurun_out/parity_$TAG.json > gpurun_out/parity_$TAG.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/parity_$TAG.log
