#!/bin/bash
# Round-2g A/B (config 3): forward with a producer warp and a two-batch ring (GS_FWD_WS=1).
mkdir -p gpurun_out
run() {  # name, env...
  n=$1; shift
  for rep in 1 2; do
    env "$@" timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/g_${n}_$rep.json 2>gpurun_out/g_${n}_$rep.err
  done
}
rm -f gpurun_out/g_*.json gpurun_out/g_*.err
GS_FWD_WS=1 timeout 900 python -m pytest tests/test_gpu_frame.py tests/test_gpu_frame_parity.py tests/test_gpu_engine.py tests/test_gpu_configs.py -m gpu -x -q 2>&1 | tail -5
run cur A=1
run ws GS_FWD_WS=1
run ws_nopad GS_FWD_WS=1 GS_FWD_CARVE=-1
python tools/show_bench.py gpurun_out/g_*.json
