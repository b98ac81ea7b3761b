#!/bin/bash
# Round-2g A/B (config 3): the grouped record backward's flush reading the splat ids from the staged records (_ab/ids1).
mkdir -p gpurun_out
run() {  # name, env...
  n=$1; shift
  for rep in 1 2 3; do
    env "$@" timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/g_${n}_$rep.json 2>gpurun_out/g_${n}_$rep.err
  done
}
rm -f gpurun_out/g_*.json gpurun_out/g_*.err
GS_LIB_PATH=_ab/ids1/libsplat_b200.so timeout 900 python -m pytest tests/test_gpu_frame.py tests/test_gpu_frame_parity.py tests/test_gpu_engine.py -m gpu -x -q 2>&1 | tail -2
run cur A=1
run ids1 GS_LIB_PATH=_ab/ids1/libsplat_b200.so
python tools/show_bench.py gpurun_out/g_*.json
