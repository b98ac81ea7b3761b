python -m pytest tests/test_gpu_frame.py tests/test_gpu_frame_parity.py -m gpu -q -x 2>&1 | grep -E "Error|assert |passed|failed" | head -5
for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/n$i.json 2>/dev/null; python tools/show_bench.py gpurun_out/n$i.json; done
for st in 2 4; do python bench.py --streams $st --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s$st.json 2>/dev/null; python tools/show_bench.py gpurun_out/s$st.json; done
CMD="python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 300 --csv --log-file gpurun_out/launches_c3d.csv $CMD > /dev/null 2>&1; echo ncu=$?
