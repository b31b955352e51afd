mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "controller or q_after or topk_sort" 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err
tail -c 600 gpurun_out/r02r_bench.json
CB_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02r_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02r_ncu_list.log 2>&1
python tools/launch_summary.py gpurun_out/r02r_launches.csv 2 > gpurun_out/r02r_launch_summary.txt 2>&1; cat gpurun_out/r02r_launch_summary.txt
CB_PROFILE_RANGE=1 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc -s 57 -c 4 \
    -o gpurun_out/r02r_gemm_l14 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02r_ncu_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/r02r_gemm_l14.ncu-rep 6 > gpurun_out/r02r_gemm_l14_summary.txt 2>&1
CB_PROFILE_RANGE=1 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_tc5 -s 14 -c 1 \
    -o gpurun_out/r02r_attn_l14 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02r_ncu_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/r02r_attn_l14.ncu-rep 6 > gpurun_out/r02r_attn_l14_summary.txt 2>&1
CB_PROFILE_RANGE=1 ncu --profile-from-start off --set full --clock-control none -k regex:topk -s 1 -c 2 \
    -o gpurun_out/r02r_topk python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02r_ncu_topk.log 2>&1
python tools/ncu_summary.py gpurun_out/r02r_topk.ncu-rep 4 > gpurun_out/r02r_topk_summary.txt 2>&1
python bench.py --cpu-full > gpurun_out/r02r_cpu_full.json 2> gpurun_out/r02r_cpu_full.err
cat gpurun_out/r02r_cpu_full.json
