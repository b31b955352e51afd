#!/bin/bash
timeout 600 python tools/ab.py "" "" 30 2>&1 | tail -1
for b in "gemm_mc=2" "gemm_no192=1" "attn_splits=1"; do
  echo "== $b"
  timeout 600 python tools/ab.py "" "$b" 40 2>&1 | tail -1; timeout 600 python tools/ab.py "$b" "" 40 2>&1 | tail -1
done
