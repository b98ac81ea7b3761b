for B in 1 2; do
  GS_BINNING=$B python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2_m$B.json 2>/dev/null
  GS_BINNING=$B python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_m$B.json 2>/dev/null
  GS_BINNING=$B python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b4_m$B.json 2>/dev/null
  GS_BINNING=$B python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b1_m$B.json 2>/dev/null
done
