python -m pytest tests/test_gpu_frame.py tests/test_gpu_frame_parity.py -x -q > gpurun_out/pt_ab.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pt_ab.log
for v in 1 2; do python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bab$v.json 2>gpurun_out/bab.err; python tools/show_bench.py gpurun_out/bab$v.json | cut -c1-330; done
