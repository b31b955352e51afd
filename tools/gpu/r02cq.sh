#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "multicast_clusters_bitwise" 2>&1 | tail -2
timeout 900 python tools/gemm_micro.py --only qkv_l2,o_l2,gu_l2,down_l2,qkv_l31,o_l31,gu_l31,down_l31 --mcs 2 --l2pfs 0,4,8,16 --rotate 4 --iters 20 2>&1 | grep -v "^{" | tee gpurun_out/r02cq_micro.txt
timeout 600 python tools/ab.py "gemm_l2pf=0" "gemm_l2pf=8" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "gemm_l2pf=8" "gemm_l2pf=0" 40 2>&1 | tail -3
