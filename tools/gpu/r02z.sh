mkdir -p gpurun_out
for r in 0.05 0.15 0.30 0.50; do
timeout 900 python bench.py --config yi --ratio $r --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02z_yi_$r.json 2> gpurun_out/r02z_yi_$r.err
python -c "import json;d=json.loads(open('gpurun_out/r02z_yi_$r.json').read().strip().splitlines()[-1]);print('yi r=$r', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['clocks']['sm_mhz'])"
done
timeout 1500 python bench.py --config llama --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > gpurun_out/r02z_llama.json 2> gpurun_out/r02z_llama.err
python -c "import json;d=json.loads(open('gpurun_out/r02z_llama.json').read().strip().splitlines()[-1]);print('llama', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['path']['frac'], d['clocks']['sm_mhz'])"
tail -3 gpurun_out/r02z_llama.err
timeout 1500 python bench.py --config batched --steps 3 --warmup 2 > gpurun_out/r02z_batched.json 2> gpurun_out/r02z_batched.err
tail -c 800 gpurun_out/r02z_batched.json
