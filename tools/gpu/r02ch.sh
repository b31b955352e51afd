#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk or blend" 2>&1 | tail -3
timeout 600 python tools/ab.py "topk_scatter=0,topk_drop2=0" "topk_scatter=1,topk_drop2=1" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "topk_scatter=1,topk_drop2=0" "topk_scatter=1,topk_drop2=1" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_dual=0" "attn_dual=1,attn_dual_f=80,attn_dual_m=15" 40 2>&1 | tail -3
