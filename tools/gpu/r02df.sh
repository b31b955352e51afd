#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -k "attention or config_heads" 2>&1 | tail -1
for i in 1 2 3; do
  for v in new base; do
    cp tools/gpu/libs/lib_$v.so paper_2405_16444_b200/libcacheblend.so
    echo "== $v"; timeout 300 python tools/attn_micro.py --rows 3072,553,460,369 --splits 0 --iters 60 2>&1 | grep rows=
  done
done
cp tools/gpu/libs/lib_new.so paper_2405_16444_b200/libcacheblend.so
