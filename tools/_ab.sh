python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/pt_ab.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pt_ab.log
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bab.json 2>gpurun_out/bab.err; python tools/show_bench.py gpurun_out/bab.json | cut -c1-330; done
