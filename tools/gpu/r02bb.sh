#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention or attn" 2>&1 | tail -3
timeout 600 python tools/attn_micro.py --splits 0,1,2,3 --pairs 0 --iters 30 2>&1 | tail -16
