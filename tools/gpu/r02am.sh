#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/ab.py "gemm_mc=0" "gemm_mc=2" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "gemm_mc=2" "gemm_mc=0" 40 2>&1 | tail -3
