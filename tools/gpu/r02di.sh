#!/bin/bash
timeout 900 python tools/gemm_micro.py --only down_l2,down_l31,o_l2,o_l31 --resid --rotate 4 --iters 20 --bns 0,128,192,256 --ksplits 0,1,2,3 2>&1 | grep -v "^{"
