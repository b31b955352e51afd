#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/attn_micro.py --splits 0 --pairs 0 --iters 30 2>&1 | tail -4
for o in "attn_poly=1" "attn_poly=2" "attn_wg4=1"; do
  timeout 600 python tools/ab.py "attn_poly=0" "$o" 30 2>&1 | tail -3
done
