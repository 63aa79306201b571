timeout 600 python -m pytest tests/test_gpu_comm.py -q -x --timeout 300 2>&1 | grep -E "Error|assert|error" | head -20
