timeout 900 python -m pytest tests/test_gpu_loop.py -x -q 2>&1 | tail -5
