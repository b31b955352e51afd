#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/micro/mc_check.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or blend_small or multicast or ksplit" 2>&1 | tail -3
timeout 300 python tools/gemm_micro.py --only o_l2,down_l2,o_l31,down_l31 --resid --iters 30 2>&1 | grep -v "^{"
for shp in "579 4096 4096 1 1" "401 4096 14336 1 1"; do echo "== trace $shp"; python tools/gemm_trace.py $shp 2>&1 | head -5; done
timeout 600 python tools/ab.py "gemm_mc=2" "gemm_mc=2" 20 2>&1 | tail -3
