python -m pytest tests/test_gpu_loop.py -x -q 2>&1 | tail -3
for cf in 0 80; do for ca in 0 100 150 200; do echo "COST $cf $ca"; NFGPU_CT_COST_FWD=$cf NFGPU_CT_COST_ADJ=$ca python tools/loop_rate.py --workload medium --iters 2000 2>&1 | tail -1 | grep -oE '"loop_us_per_iter": [0-9.]+|"graph_us_per_iter": [0-9.]+' | paste - -; done; done
NFGPU_LOOP_PROFILE=2 python tools/loop_rate.py --workload medium --iters 400 2>&1 | tail -2 | grep -oE '"(fwd|adj)_end_(min|mean|max)": [0-9.]+|"profile_us.*next_iter_gap": [0-9.]+'
