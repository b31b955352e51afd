mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or blend_small" 2>&1 | tail -2
for pf in 0 1 0 1; do
CB_OPTS=gemm_pf=$pf python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02y_bench_$pf.json 2> gpurun_out/r02y_bench_$pf.err
python -c "import json;d=json.loads(open('gpurun_out/r02y_bench_$pf.json').read().strip().splitlines()[-1]);print('gemm_pf=$pf', d['ms_per_step'],d['kernel_ms']['gemm'], d['clocks']['sm_mhz'])"
done
