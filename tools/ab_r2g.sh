#!/bin/bash
# Round-2g A/B (configs 1, 2, 4): record backward budgeted for 7 CTAs per SM (_ab/bm7) against 8 (in-tree).
mkdir -p gpurun_out
rm -f gpurun_out/g_*.json gpurun_out/g_*.err
for c in 1 2 4; do
  for rep in 1 2; do
    python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/g_c${c}_cur_$rep.json 2>/dev/null
    GS_LIB_PATH=_ab/bm7/libsplat_b200.so python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/g_c${c}_bm7_$rep.json 2>/dev/null
  done
done
python tools/show_bench.py gpurun_out/g_*.json
