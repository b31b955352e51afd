#!/bin/bash
for b in "gemm_no192=1" "gemm_no224=1" "q_split=0" "attn_splits=1" "gemm_balance=0"; do
  echo "== $b"
  for i in 1 2; do timeout 600 python tools/ab.py "" "$b" 40 2>&1 | tail -1; timeout 600 python tools/ab.py "$b" "" 40 2>&1 | tail -1; done
done
