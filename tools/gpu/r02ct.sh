#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk or blend" 2>&1 | tail -2
echo "== new"; for i in 1 2 3; do timeout 120 python tools/topk_trace.py 2>&1 | tail -1; done
cp paper_2405_16444_b200/libcacheblend.so /tmp/lib_new.so
cp tools/gpu/libs/lib_base.so paper_2405_16444_b200/libcacheblend.so
echo "== base"; for i in 1 2 3; do timeout 120 python tools/topk_trace.py 2>&1 | tail -1; done
cp /tmp/lib_new.so paper_2405_16444_b200/libcacheblend.so
