#!/bin/bash
# Round-2 final refresh after the multicast default change, the L1 epilogue prefetch and the two-warp top-k
# ncu full captures of layer 14's GEMMs, its attention and two top-k launches.
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02g_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02g_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02g_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02g_bench.json').read().strip().splitlines()[-1]);print('mistral', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['roofline']['attention']['frac'], d['e2e']['ms'], d['e2e'].get('paired_overhead_ms'), d['clocks'])"
CB_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02g_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02g_ncu_list.log 2>&1
python tools/launch_summary.py gpurun_out/r02g_launches.csv 2 > gpurun_out/r02g_launch_summary.txt 2>&1; cat gpurun_out/r02g_launch_summary.txt
CB_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc -s 57 -c 4 \
    -o gpurun_out/r02g_gemm_l14 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02g_ncu_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/r02g_gemm_l14.ncu-rep 6 > gpurun_out/r02g_gemm_l14_summary.txt 2>&1
CB_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_tc5 -s 14 -c 1 \
    -o gpurun_out/r02g_attn_l14 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02g_ncu_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/r02g_attn_l14.ncu-rep 6 > gpurun_out/r02g_attn_l14_summary.txt 2>&1
CB_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:topk -s 1 -c 2 \
    -o gpurun_out/r02g_topk python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02g_ncu_topk.log 2>&1
python tools/ncu_summary.py gpurun_out/r02g_topk.ncu-rep 4 > gpurun_out/r02g_topk_summary.txt 2>&1
rm -f gpurun_out/r02g_*.ncu-rep.tmp
for r in 0.05 0.15 0.30 0.50; do
timeout 900 python bench.py --config yi --ratio $r --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02g_yi_$r.json 2> gpurun_out/r02g_yi_$r.err
python -c "import json;d=json.loads(open('gpurun_out/r02g_yi_$r.json').read().strip().splitlines()[-1]);print('yi r=$r', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['clocks']['sm_mhz'])"
done
timeout 1500 python bench.py --config llama --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02g_llama.json 2> gpurun_out/r02g_llama.err
python -c "import json;d=json.loads(open('gpurun_out/r02g_llama.json').read().strip().splitlines()[-1]);print('llama', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['clocks']['sm_mhz'])"
timeout 1500 python bench.py --config batched --steps 3 --warmup 3 > gpurun_out/r02g_batched.json 2> gpurun_out/r02g_batched.err
tail -c 600 gpurun_out/r02g_batched.json
ls -la gpurun_out | grep r02g
