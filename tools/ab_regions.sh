for R in 4 2; do
  GS_BWD_REGIONS=$R GS_FWD_REGIONS=$R python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b1_r$R.json 2>/dev/null
  GS_BWD_REGIONS=$R GS_FWD_REGIONS=$R python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2_r$R.json 2>/dev/null
done
