mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention" 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -m gpu -x -q 2>&1 | tail -4
for pm in 0 1; do
CB_OPTS=attn_pair=$pm python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02i_bench_$pm.json 2> gpurun_out/r02i_bench_$pm.err
python -c "import json;d=json.loads(open('gpurun_out/r02i_bench_$pm.json').read().strip().splitlines()[-1]);print('attn_pair=$pm', d['ms_per_step'],d['kernel_ms'])"
done
