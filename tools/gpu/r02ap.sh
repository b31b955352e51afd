#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/micro/mc_check.py 2>&1 | tail -9
timeout 300 python tools/gemm_micro.py --only qkv_l2,o_l2,down_l2,qkv_l31,o_l31,down_l31,qkv_l1 --mcs 0,2,3 --iters 30 2>&1 | grep -v "^{" | tee gpurun_out/r02ap_micro.txt
