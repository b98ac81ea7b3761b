#!/bin/bash
# A/B of library variants: tools/ab_libs.sh <config> <steps> <lib-dir>... (plus the in-tree build as "cur")
c=$1; st=$2; shift 2
for rep in 1 2; do
  python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_c${c}_cur_$rep.json 2>/dev/null
  for d in "$@"; do
    n=$(basename $d)
    GS_LIB_PATH=$d/libsplat_b200.so python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_c${c}_${n}_$rep.json 2>/dev/null
  done
done
python tools/show_bench.py gpurun_out/ab_c${c}_*.json
