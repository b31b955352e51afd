#!/bin/bash
for i in 1 2 3; do timeout 600 python tools/ab.py "" "" 40 2>&1 | tail -1; done
for i in 1 2; do timeout 600 python tools/ab.py "gemm_mc=0" "gemm_mc=2" 40 2>&1 | tail -1; timeout 600 python tools/ab.py "gemm_mc=2" "gemm_mc=0" 40 2>&1 | tail -1; done
