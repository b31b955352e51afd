#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ck_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r02ck_pytest_gpu.log
timeout 600 python tools/ab.py "attn_early=0" "attn_early=1" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_early=1" "attn_early=0" 40 2>&1 | tail -3
