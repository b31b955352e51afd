#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/micro/mc_check.py 2>&1 | tail -2
timeout 300 python tools/gemm_micro.py --only qkv_l2,o_l2,down_l2,gu_l2,qkv_l31,o_l31,down_l31,gu_l31,qkv_l1 --mcs 0,2 --iters 30 2>&1 | grep -v "^{" | tee gpurun_out/r02al_micro.txt
timeout 600 python tools/ab.py "gemm_mc=0" "gemm_mc=2" 40 2>&1 | tail -4
for o in 0 2; do CB_OPTS=gemm_mc=$o timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-request-sub > gpurun_out/r02al_bench_$o.json 2> gpurun_out/r02al_bench_$o.err; python -c "import json;d=json.loads(open('gpurun_out/r02al_bench_$o.json').read().strip().splitlines()[-1]);print('mc=$o',d['ms_per_step'],d['kernel_ms'],d['clocks'])"; done
