#!/bin/bash
timeout 600 python tools/ab.py "" "gemm_mc=0" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "gemm_mc=0" "" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "" "gemm_mc=0" 40 --e2e 2>&1 | tail -1
timeout 600 python tools/gemm_micro.py --only qkv_l2,o_l2,down_l2,qkv_l31,o_l31,down_l31 --mcs 0,2 --resid --rotate 4 --iters 20 2>&1 | grep -v "^{"
