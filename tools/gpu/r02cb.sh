#!/bin/bash
# dual-stream attention: parity tests, micro timing vs attn_tc5
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention" 2>&1 | tail -5
timeout 300 python tools/attn_micro.py --splits 0,1,2,3 --pairs 0 --duals 0,1 2>&1 | grep rows= | tee gpurun_out/r02cb_attn_micro.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
