#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "blend or gemm" 2>&1 | tail -1
for b in "gemm_no192=1" "gemm_balance=0" "gemm_mc=2" "realign_overlap=1"; do
  echo "== $b"; timeout 600 python tools/ab.py "" "$b" 40 2>&1 | tail -1; timeout 600 python tools/ab.py "$b" "" 40 2>&1 | tail -1
done
