#!/bin/bash
# Round-2g A/B (config 3): forward register budget (7 / 8 CTAs per SM: 72 / 64 registers) and entry-pair loop unrolled by 2.
mkdir -p gpurun_out
run() {  # name, env...
  n=$1; shift
  for rep in 1 2; do
    env "$@" python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/g_${n}_$rep.json 2>gpurun_out/g_${n}_$rep.err
  done
}
rm -f gpurun_out/g_*.json gpurun_out/g_*.err
run cur A=1
for v in fm7 fm8 fu2 fm7u2; do run $v GS_LIB_PATH=_ab/$v/libsplat_b200.so; done
run fm7_nopad GS_LIB_PATH=_ab/fm7/libsplat_b200.so GS_FWD_PAD=0
python tools/show_bench.py gpurun_out/g_*.json
