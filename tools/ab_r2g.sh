#!/bin/bash
# Round-2g A/B (config 3): record backward with alpha zeroed for non-contributing pixels (_ab/az1; needs rcp.approx(1.0) == 1.0).
mkdir -p gpurun_out
run() {  # name, env...
  n=$1; shift
  for rep in 1 2 3; do
    env "$@" timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/g_${n}_$rep.json 2>gpurun_out/g_${n}_$rep.err
  done
}
rm -f gpurun_out/g_*.json gpurun_out/g_*.err
[ -x tools/bin/rcp1 ] && tools/bin/rcp1  # nvcc -gencode arch=compute_100a,code=sm_100a -o tools/bin/rcp1 tools/src/rcp1.cu
GS_LIB_PATH=_ab/az1/libsplat_b200.so timeout 900 python -m pytest tests/test_gpu_frame.py tests/test_gpu_frame_parity.py tests/test_gpu_engine.py tests/test_gpu_golden.py -m gpu -x -q 2>&1 | tail -2
run cur A=1
run az1 GS_LIB_PATH=_ab/az1/libsplat_b200.so
python tools/show_bench.py gpurun_out/g_*.json
