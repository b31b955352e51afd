#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/ab.py "realign_copy_ctas=0" "realign_copy_ctas=16" 30 --e2e 2>&1 | tail -3
timeout 600 python tools/ab.py "realign_copy_ctas=0" "realign_copy_ctas=148" 30 --e2e 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_early=0" "attn_early=1" 30 --e2e 2>&1 | tail -3
