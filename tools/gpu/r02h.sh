#!/bin/bash
# final validation on the final code: GPU suite, smoke, bench line, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02h_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02h_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02h_smoke.log
timeout 900 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02h_bench.json').read().strip().splitlines()[-1]);print('mistral', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['roofline']['attention']['frac'], d['e2e']['ms'], d['e2e'].get('paired_overhead_ms'), d['clocks'])"
CB_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02h_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02h_ncu_list.log 2>&1
python tools/launch_summary.py gpurun_out/r02h_launches.csv 2 > gpurun_out/r02h_launch_summary.txt 2>&1; head -8 gpurun_out/r02h_launch_summary.txt
