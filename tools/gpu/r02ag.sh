#!/bin/bash
mkdir -p gpurun_out
python tools/gemm_micro.py --only o_l31,down_l31,qkv_l31,o_l2 --pairs 1,2 --bns 128,192,256 --iters 30 2>&1 | grep -v "^{" | tee gpurun_out/r02ag_micro.txt
