#!/bin/bash
for b in "gemm_pair=1" "gemm_bn=128" "gemm_bn=192" "gemm_bn=256" "gemm_sched=1"; do
  echo "== $b"
  timeout 600 python tools/ab.py "" "$b" 40 2>&1 | tail -1; timeout 600 python tools/ab.py "$b" "" 40 2>&1 | tail -1
done
