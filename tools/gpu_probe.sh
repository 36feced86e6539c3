timeout 100 python -m pytest tests/test_gpu_chunk.py -q -x -k "paged_k4 and 64-4113-333" 2>&1 | grep -E "Error|assert|error" | head -10
