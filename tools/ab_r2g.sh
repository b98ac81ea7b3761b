#!/bin/bash
# Round-2g A/B (config 3): shared-memory carve-out preferences of the raster kernels; the backward with
# 16-record staging chunks (_ab/ch16: 18.6 KB per CTA, 8 CTAs in a 164 KB carve-out).
mkdir -p gpurun_out
run() {  # name, env...
  n=$1; shift
  for rep in 1 2; do
    env "$@" python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/g_${n}_$rep.json 2>gpurun_out/g_${n}_$rep.err
  done
}
rm -f gpurun_out/g_*.json gpurun_out/g_*.err
run cur A=1
run fc25 GS_FWD_CARVE=25
run fc25_7 GS_FWD_CARVE=25 GS_FWD_PAD=512
run fc25_6 GS_FWD_CARVE=25 GS_FWD_PAD=2000
run fc25_5 GS_FWD_CARVE=25 GS_FWD_PAD=4400
run ch16 GS_LIB_PATH=_ab/ch16/libsplat_b200.so
run ch16_bc72 GS_LIB_PATH=_ab/ch16/libsplat_b200.so GS_BWD_CARVE=72
run ch16_bc58 GS_LIB_PATH=_ab/ch16/libsplat_b200.so GS_BWD_CARVE=58
run ch16_bc72_fc25_7 GS_LIB_PATH=_ab/ch16/libsplat_b200.so GS_BWD_CARVE=72 GS_FWD_CARVE=25 GS_FWD_PAD=512
run bc58 GS_BWD_CARVE=58
python tools/show_bench.py gpurun_out/g_*.json
