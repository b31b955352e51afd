mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk or deviation_topk or blend_small or tiny_fp32" 2>&1 | tail -3
python tools/topk_trace.py
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
python -c "import json;d=json.loads(open('gpurun_out/r02w_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['kernel_ms'], d['clocks']['sm_mhz'])"
done
