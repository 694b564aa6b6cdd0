python -m pytest tests/test_gpu_loop.py -x -q 2>&1 | tail -3
python tools/loop_rate.py --workload medium --iters 2000 2>&1 | tail -1
NFGPU_LOOP_PROFILE=1 python tools/loop_rate.py --workload medium --iters 400 2>&1 | tail -1
NFGPU_LOOP_PROFILE=2 python tools/loop_rate.py --workload medium --iters 400 2>&1 | tail -2
