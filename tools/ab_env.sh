#!/bin/bash
# A/B of an environment switch: tools/ab_env.sh <config> <steps> "<ENV=a>" "<ENV=b>" ...
c=$1; st=$2; shift 2
for rep in 1 2; do
  i=0
  for e in "$@"; do
    env $e python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abe_c${c}_${i}_$rep.json 2>/dev/null
    i=$((i+1))
  done
done
echo "variants: $*"
python tools/show_bench.py gpurun_out/abe_c${c}_*.json
