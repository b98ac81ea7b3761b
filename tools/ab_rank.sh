timeout 600 python -m pytest tests/test_gpu_frame.py tests/test_gpu_golden.py -x -q > gpurun_out/t.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t.log
for R in match or; do
  GS_SORT_RANK=$R python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b4_$R.json 2>/dev/null
  GS_SORT_RANK=$R python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b1_$R.json 2>/dev/null
done
