#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_splits=1" "attn_splits=0" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_splits=0" "attn_splits=1" 40 2>&1 | tail -3
