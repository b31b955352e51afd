mkdir -p gpurun_out
python tools/gemm_swap_ab.py 2>&1 | tail -16
for sw in 0 1; do
CB_OPTS=gemm_swap=$sw python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02o_bench_$sw.json 2> gpurun_out/r02o_bench_$sw.err
python -c "import json;d=json.loads(open('gpurun_out/r02o_bench_$sw.json').read().strip().splitlines()[-1]);print('gemm_swap=$sw', d['ms_per_step'],d['kernel_ms'], d['clocks'])"
done
timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -4
