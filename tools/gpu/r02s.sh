mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "controller or q_after or ksplit or topk" 2>&1 | tail -3
for ks in 0 2 3; do
CB_OPTS=gemm_ksplit=$ks python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02s_bench_$ks.json 2> gpurun_out/r02s_bench_$ks.err
python -c "import json;d=json.loads(open('gpurun_out/r02s_bench_$ks.json').read().strip().splitlines()[-1]);print('ksplit=$ks', d['ms_per_step'],d['kernel_ms'], d['clocks']['sm_mhz'])"
done
