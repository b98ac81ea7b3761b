for M in 8 9 10; do
  GS_FWD_MINB=$M python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b1_m$M.json 2>/dev/null
  GS_FWD_MINB=$M python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2_m$M.json 2>/dev/null
done
