#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ao_bench.json 2> gpurun_out/r02ao_bench.err
python -c "import json;d=json.loads(open('gpurun_out/r02ao_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['kernel_ms'],d['roofline']['frac'],d['roofline']['path']['frac'],d['clocks'],d['e2e'])"
