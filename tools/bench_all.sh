#!/bin/bash
# Every BASELINE config with its end-to-end leg (results table of DESIGN.md), then the
# default (judged) bench line with its CPU baseline.
for c in 0 1 2 3 4; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/all_c$c.json 2>gpurun_out/all_c$c.err
done
python bench.py > gpurun_out/default.json 2>gpurun_out/default.err
