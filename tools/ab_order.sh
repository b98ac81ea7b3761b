for R in 1 2; do
for O in 0 1; do
  GS_TILE_ORDER=$O python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b1_o${O}_$R.json 2>/dev/null
  GS_TILE_ORDER=$O python bench.py --config 0 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b0_o${O}_$R.json 2>/dev/null
  GS_TILE_ORDER=$O python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2_o${O}_$R.json 2>/dev/null
  GS_TILE_ORDER=$O python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_o${O}_$R.json 2>/dev/null
done
done
