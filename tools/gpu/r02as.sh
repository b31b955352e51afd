mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r02as_bench.json 2> gpurun_out/r02as_bench.err
tail -c 600 gpurun_out/r02as_bench.json
CB_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02as_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02as_ncu_list.log 2>&1
python tools/launch_summary.py gpurun_out/r02as_launches.csv 2 > gpurun_out/r02as_launch_summary.txt 2>&1; cat gpurun_out/r02as_launch_summary.txt
CB_PROFILE_RANGE=1 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc -s 57 -c 4 \
    -o gpurun_out/r02as_gemm_l14 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02as_ncu_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/r02as_gemm_l14.ncu-rep 6 > gpurun_out/r02as_gemm_l14_summary.txt 2>&1
CB_PROFILE_RANGE=1 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_tc5 -s 14 -c 1 \
    -o gpurun_out/r02as_attn_l14 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02as_ncu_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/r02as_attn_l14.ncu-rep 6 > gpurun_out/r02as_attn_l14_summary.txt 2>&1
CB_PROFILE_RANGE=1 ncu --profile-from-start off --set full --clock-control none -k regex:topk -s 1 -c 2 \
    -o gpurun_out/r02as_topk python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02as_ncu_topk.log 2>&1
python tools/ncu_summary.py gpurun_out/r02as_topk.ncu-rep 4 > gpurun_out/r02as_topk_summary.txt 2>&1
for r in 0.05 0.15 0.30 0.50; do
timeout 900 python bench.py --config yi --ratio $r --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02as_yi_$r.json 2> gpurun_out/r02as_yi_$r.err
python -c "import json;d=json.loads(open('gpurun_out/r02as_yi_$r.json').read().strip().splitlines()[-1]);print('yi r=$r', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['clocks']['sm_mhz'])"
done
timeout 1500 python bench.py --config llama --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02as_llama.json 2> gpurun_out/r02as_llama.err
python -c "import json;d=json.loads(open('gpurun_out/r02as_llama.json').read().strip().splitlines()[-1]);print('llama', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['clocks']['sm_mhz'])"
tail -3 gpurun_out/r02as_llama.err
timeout 1500 python bench.py --config batched --steps 3 --warmup 2 > gpurun_out/r02as_batched.json 2> gpurun_out/r02as_batched.err
tail -c 800 gpurun_out/r02as_batched.json
