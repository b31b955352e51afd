#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/attn_dual_debug.py 3072 460 2 0 1 2 3 2>&1 | tail -8
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention" 2>&1 | tail -2
timeout 300 python tools/attn_micro.py --rows 3072,553,369 --splits 0,1,2 --pairs 0 --duals 0,1 --polys 0,1,2 2>&1 | grep rows= | tee gpurun_out/r02ce_attn_micro.txt
timeout 600 python tools/ab.py "attn_dual=0" "attn_dual=1" 30 2>&1 | tail -4
timeout 600 python tools/ab.py "attn_dual=1,attn_poly=0" "attn_dual=1,attn_poly=1" 30 2>&1 | tail -4
