python -m pytest tests/test_gpu_frame_parity.py tests/test_gpu_api.py -m gpu -q -s > gpurun_out/parity.log 2>&1; echo parity_rc=$?
grep -E "^config|passed|failed|Error|assert" gpurun_out/parity.log | head -40
python tests/parity_report.py --out gpurun_out/parity_r2.json > gpurun_out/parity_report.log 2>&1; echo report_rc=$?
tail -45 gpurun_out/parity_report.log
