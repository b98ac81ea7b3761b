timeout 600 python -m pytest tests/test_gpu_frame.py tests/test_gpu_golden.py -x -q > gpurun_out/t.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t.log
for S in 1 0; do
  GS_SORT_SMALL=$S python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b1_s$S.json 2>/dev/null
done
python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null
python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b4.json 2>/dev/null
