#!/bin/bash
# Session-3 baseline: GPU suite, smoke, bench line, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ca_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02ca_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ca_bench.json 2> gpurun_out/r02ca_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02ca_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02ca_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02ca_ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/r02ca_launches.csv 2 > gpurun_out/r02ca_launch_summary.txt 2>&1; head -30 gpurun_out/r02ca_launch_summary.txt
