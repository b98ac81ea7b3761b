python -m pytest tests -m gpu -q -x 2>&1 | grep -E "Error|assert |passed|failed|error" | head -20
