timeout 900 python -m pytest tests/test_gpu_loop.py tests/test_gpu_operator.py -x -q 2>&1 | tail -3
timeout 120 python tools/loop_rate.py --workload medium --iters 2000 2>&1 | tail -1 | grep -oE '"loop_us_per_iter": [0-9.]+|"graph_us_per_iter": [0-9.]+' | paste - -
NFGPU_LOOP_PROFILE=2 timeout 120 python tools/loop_rate.py --workload medium --iters 400 2>&1 | tail -2 | grep -oE '"(fwd|adj)_end_(min|mean|max)": [0-9.]+|"profile_us.*next_iter_gap": [0-9.]+'
