timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t.log
for P in 0 1; do
  GS_PDL=$P python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b1_p$P.json 2>/dev/null
  GS_PDL=$P python bench.py --config 0 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b0_p$P.json 2>/dev/null
  GS_PDL=$P python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2_p$P.json 2>/dev/null
done
