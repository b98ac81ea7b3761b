for M in 8 9 10; do
  GS_FWD_MINB=$M python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b1_m$M.json 2>/dev/null
  GS_FWD_MINB=$M python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2_m$M.json 2>/dev/null
done
timeout 600 python -m pytest tests/test_gpu_frame.py tests/test_gpu_golden.py -x -q > gpurun_out/t.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t.log
