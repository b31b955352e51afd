#!/bin/bash
# validation after the epilogue L1 prefetch and the two-warp top-k drop loop
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02f_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02f_smoke.log
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02f_bench.json').read().strip().splitlines()[-1]);print('mistral', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['roofline']['attention']['frac'], d['e2e']['ms'], d['e2e'].get('paired_overhead_ms'), d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
CB_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02f_ncu_list.log 2>&1
python tools/launch_summary.py gpurun_out/r02f_launches.csv 2 > gpurun_out/r02f_launch_summary.txt 2>&1; head -12 gpurun_out/r02f_launch_summary.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_reference.json 2>&1; echo "reference rc=$?"; tail -c 300 gpurun_out/r02f_reference.json
