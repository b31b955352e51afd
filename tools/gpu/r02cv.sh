#!/bin/bash
# sweep of existing planner / kernel knobs against the defaults (paired blend A/B, 30 rounds each)
for b in "gemm_balance=0" "gemm_no192=1" "gemm_mc=1" "gemm_mc=0" "topk_threads=512" "realign_overlap=1" "gemm_tail=0" "pdl=0" "topk_drop=0"; do
  echo "== $b"; timeout 600 python tools/ab.py "" "$b" 30 2>&1 | tail -1
done
