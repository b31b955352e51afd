set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
tail -c 3000 gpurun_out/r02b_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02b_ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/r02b_launches.csv 2
