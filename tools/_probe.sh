python -m pytest tests/test_gpu_frame.py tests/test_gpu_engine.py tests/test_gpu_api.py -m gpu -q -x 2>&1 | grep -E "Error|assert |passed|failed|error" | head -20
