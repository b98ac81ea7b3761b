#!/bin/bash
# Round-2g A/B (config 3): pairs between the forward's "whole warp retired" votes (_ab/de1, de2, de4, de8).
mkdir -p gpurun_out
run() {  # name, env...
  n=$1; shift
  for rep in 1 2; do
    env "$@" python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/g_${n}_$rep.json 2>gpurun_out/g_${n}_$rep.err
  done
}
rm -f gpurun_out/g_*.json gpurun_out/g_*.err
GS_LIB_PATH=_ab/de4/libsplat_b200.so python -m pytest tests/test_gpu_frame.py tests/test_gpu_frame_parity.py tests/test_gpu_golden.py -m gpu -x -q 2>&1 | tail -2
run base GS_LIB_PATH=_ab/base2/libsplat_b200.so
for v in de1 de2 de4 de8; do run $v GS_LIB_PATH=_ab/$v/libsplat_b200.so; done
python tools/show_bench.py gpurun_out/g_*.json
