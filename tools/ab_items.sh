for I in 16 20 24; do
  GS_SORT_ITEMS=$I python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2_i$I.json 2>/dev/null
  GS_SORT_ITEMS=$I python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b4_i$I.json 2>/dev/null
  GS_SORT_ITEMS=$I python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_i$I.json 2>/dev/null
done
