#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "gemm or blend or fullsize or mistral" 2>&1 | tail -1
timeout 600 python tools/gemm_micro.py --only down_l2,down_l31,o_l2,o_l31 --resid --rotate 4 --iters 20 --ksplits 0,1 2>&1 | grep -v "^{\|num_sms"
for i in 1 2; do timeout 600 python tools/ab.py "" "gemm_ksplit=1" 40 2>&1 | tail -1; timeout 600 python tools/ab.py "gemm_ksplit=1" "" 40 2>&1 | tail -1; done
