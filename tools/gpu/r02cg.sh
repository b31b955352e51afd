#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02cg_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02cg_pytest_gpu.log
timeout 600 python tools/ab.py "attn_dual=0" "attn_dual=1" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_dual=1" "attn_dual=0" 40 2>&1 | tail -3
