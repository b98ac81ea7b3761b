python -m pytest tests/test_gpu_frame_parity.py tests/test_gpu_engine.py -m gpu -q -x 2>&1 | grep -E "Error|assert |passed|failed" | head -20
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/n$i.json 2>/dev/null; python tools/show_bench.py gpurun_out/n$i.json; done
python bench.py --streams 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3.json 2>/dev/null; python tools/show_bench.py gpurun_out/s3.json
