ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r02_launches_all.csv python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc $?"
wc -l gpurun_out/r02_launches_all.csv
