python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|Error" gpurun_out/pytest.log | tail -5
python -m pytest tests/test_gpu_frame_parity.py -m gpu -q -s 2>&1 | grep -E "^config|passed|failed" > gpurun_out/parity.log; cat gpurun_out/parity.log
python tests/parity_report.py --out gpurun_out/parity_r2.json > gpurun_out/parity_report.log 2>&1; echo report_rc=$?
grep -v "ok=True img flips 0 viol 0" gpurun_out/parity_report.log | tail -20
