mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -4
for qs in 0 1; do
CB_OPTS=q_split=$qs python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02q_bench_$qs.json 2> gpurun_out/r02q_bench_$qs.err
python -c "import json;d=json.loads(open('gpurun_out/r02q_bench_$qs.json').read().strip().splitlines()[-1]);print('q_split=$qs', d['ms_per_step'],d['kernel_ms'], d['clocks'])"
done
