#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "request or store or controller" 2>&1 | tail -3
L=paper_2405_16444_b200/libcacheblend.so
cp $L /tmp/lib_new.so
for v in new old new old; do
  if [ $v = old ]; then cp tools/gpu/lib_before.so $L; else cp /tmp/lib_new.so $L; fi
  touch $L
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/r02at_bench_$v.json 2> gpurun_out/r02at_bench_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/r02at_bench_$v.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'],d['e2e']['ms'],d['clocks']['sm_mhz'])"
done
cp /tmp/lib_new.so $L
