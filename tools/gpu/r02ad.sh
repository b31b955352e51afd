#!/bin/bash
mkdir -p gpurun_out
python tools/gemm_vs_cublas.py 2>&1 | tee gpurun_out/r02ad_gemm_vs_cublas.txt | tail -14
